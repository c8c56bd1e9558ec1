// The persistent schedule of the tcgen05 GEMM family, shared by the device
// kernel (gemm_kernel.cuh), the host launcher (gemm.cu) and the CPU protocol
// checker (csrc/check/async_check.cpp): kernel arguments, tile shape constants,
// the tile raster, the per-cluster unit sequence and the launch planner.
// Plain C++ when compiled without nvcc.
#pragma once

#if defined(__CUDACC__)
#define FI_HD __host__ __device__
#else
#define FI_HD
#endif

namespace fireiron::sm100 {

enum class OutType : int { F32 = 0, F16 = 1, BF16 = 2 };

struct GemmArgs {
    void* C = nullptr;
    long ldc = 0;               // elements
    int M = 0, N = 0, K = 0;
    int tiles_m = 0, tiles_n = 0;
    int k_blocks = 0;           // 64-wide K blocks per tile (per split-K rank)
    int ab_format = 0;          // 0 = f16, 1 = bf16 (UMMA a/b format field)
    int a_mn_major = 0;         // A stored M-contiguous (col-major M x K)
    int b_mn_major = 0;         // B stored N-contiguous (row-major K x N)
    int c_row_major = 0;
    int out_type = 0;           // OutType
    int group_m = 8;            // raster band (tile rows) for the default order
    int stages = 0;             // pipeline depth actually used (0 = deepest that fits)
    const int* tile_order = nullptr;  // optional permutation: Fireiron block-swizzle table
    // gated B (all-gather fused into one launch): column chunk j of B -- b_chunk_tiles
    // scheduled tile columns -- may be read once b_ready[j] >= b_epoch (set by the
    // copy engine's stream after the chunk has landed); the raster starts at tile
    // column n_rot so the locally owned chunk comes first
    const unsigned* b_ready = nullptr;
    unsigned b_epoch = 0;
    int b_chunk_tiles = 0;
    int n_rot = 0;
    // stream-K
    int streamk = 0;
    int sk_tile_begin = 0;           // tiles before this index run data-parallel
    int sk_slices = 1;               // K-slices per leftover tile
    // remainder slices (K-slice tail only): main slice s covers K-blocks
    // [s*sk_w, (s+1)*sk_w) and the remainder [sk_slices*sk_w, k_blocks) of
    // leftover tile i runs on extra cluster rest*sk_slices + i % sk_extra as
    // its (i / sk_extra)-th unit; sk_w = 0: even slices, no remainder
    int sk_w = 0;
    int sk_extra = 0;
    int sk_q = 0;
    // 2-slice pull fixup (K-slice tail with S = 2, no remainder): slice 1 runs
    // K-blocks [0, sk_w) and publishes its whole partial; slice 0 runs the longer
    // [sk_w, k_blocks) -- its extra MMA time hides the publish -- then streams
    // the partial in chunk by chunk, adds it and stores C
    int sk_pull = 0;
    // tail units first (sk_pull only): each cluster runs its K-slice unit before
    // its data-parallel tiles, so the fixup's partial exchange and C stores
    // overlap the following main loops instead of ending the kernel exposed
    int sk_head = 0;
    int c_tma = 0;                   // f32 col-major C stored by TMA from smem staging
    int ring_drain = 1;              // the cluster's last unit stages C in the idle operand ring
    int l2_hint = 0;                 // TMA L2 eviction policy: 0 normal, 1 A last / B first, 2 A first / B last
    float* workspace = nullptr;     // [slots][kCtaGroup][BN][128] fp32 partials
    unsigned* flags = nullptr;       // [slots][kCtaGroup] epoch of the published partial
                                     // slots: one per cluster + sk_extra*(sk_q-1)
    unsigned epoch = 0;              // this launch's epoch (> every earlier launch's)
    // device epoch counter [2] = {epoch, CTAs done}: when set, a launch's epoch is
    // counter + 1, read on the device, and the last CTA to finish advances it --
    // so a launch captured in a CUDA graph gets a fresh epoch on every replay
    unsigned* epoch_ctr = nullptr;
    // optional timeline (FI_TC_TRACE): [cta][unit < 16][16] %globaltimer stamps
    // [0..7] and clock64 [8..15] of: producer first load, MMA last commit,
    // epilogue accumulator ready, epilogue done, tail partial published, tail
    // peers staged
    unsigned long long* trace = nullptr;
};

// kSlabs = 2 (CTA pairs, BN = 256 only): each CTA holds two 128-row A slabs and
// the pair computes a 512 x 256 tile with two M = 256 MMAs per K step sharing
// B -- 25% fewer operand bytes per FLOP than the 256 x 256 pair tile, at the
// cost of the whole TMEM (2 x 256 columns): no accumulator double-buffering.
// kNHalves = 2 (same restrictions): the pair computes 256 x 512 with two
// N = 256 MMAs per K step sharing A through the tensor core's A collector
// (read from shared memory once), the B stage holding both N halves.
// kKB = 2: a stage holds two 64-deep K blocks, loaded with one TMA box per
// operand (a 3D/4D view whose outer dimension walks K blocks): half the TMA
// operations of kKB = 1 for the same bytes. Stage layout: A [slab][kb][16 KiB],
// B [N half][kb][b_rows * 128 B].
template <int kCtaGroup, int BN, int kSplitK, int kSlabs = 1, int kNHalves = 1, int kKB = 1>
struct GemmShape {
    static constexpr int BM = 128;                 // rows per CTA and slab (TMEM lanes)
    static constexpr int BM_MMA = 128 * kCtaGroup; // rows of one MMA (a slab across the pair)
    static constexpr int BM_TILE = BM_MMA * kSlabs;
    static constexpr int BK = 64;                  // one 128B swizzle span of 16-bit
    static constexpr int BN_LOCAL = BN / kCtaGroup;  // B rows per CTA and MMA
    static constexpr int BN_TILE = BN * kNHalves;
    static constexpr int SLAB_BYTES = BM * BK * 2;
    static constexpr int A_BYTES = SLAB_BYTES * kSlabs;
    static constexpr int HALF_B_BYTES = BN_LOCAL * BK * 2;
    static constexpr int B_BYTES = HALF_B_BYTES * kNHalves;
    static constexpr int KB_STAGE = kKB;             // K blocks per stage
    static constexpr int A_STAGE_BYTES = A_BYTES * kKB;
    static constexpr int STAGE_BYTES = (A_BYTES + B_BYTES) * kKB;
    // split-K reduction scratch: the fp32 partial tile (rows padded by 16B)
    // reuses the operand ring once the tile's main loop has drained it
    static constexpr int RED_LD = BN + 4;
    static constexpr int RED_BYTES = kSplitK > 1 ? BM * RED_LD * 4 : 0;
    // as deep as 192 KiB allows, up to 12 stages (narrow tiles: short K-blocks need depth)
    static constexpr int kStages = (192 * 1024) / STAGE_BYTES > 12 ? 12 : (192 * 1024) / STAGE_BYTES;
    static_assert(kStages >= 2, "pipeline needs at least two stages");
    static constexpr int kAccBufs = kSlabs * kNHalves == 1 ? 2 : 1;
    static constexpr int ACC_COLS = BN * kSlabs * kNHalves;  // TMEM columns of one accumulator buffer
    static constexpr int TMEM_COLS_RAW = kAccBufs * ACC_COLS;
    static_assert(TMEM_COLS_RAW <= 512, "accumulators exceed the 512 TMEM columns");
    static constexpr int TMEM_COLS = TMEM_COLS_RAW <= 32    ? 32
                                     : TMEM_COLS_RAW <= 64  ? 64
                                     : TMEM_COLS_RAW <= 128 ? 128
                                     : TMEM_COLS_RAW <= 256 ? 256
                                                            : 512;
    static constexpr int RING_BYTES = kStages * STAGE_BYTES;
    static constexpr int BAR_BYTES = 512;  // 2 * kStages + 8 mbarriers + the TMEM slot
    static_assert(RED_BYTES <= RING_BYTES, "split-K scratch must fit in the operand ring");
    // epilogue staging for TMA stores of C: two 32-column x 128-row fp32 chunks
    static constexpr int EPI_CHUNK_BYTES = 32 * BM * 4;
    static constexpr int EPI_BYTES = 2 * EPI_CHUNK_BYTES;
    static constexpr int SMEM_BYTES = RING_BYTES + EPI_BYTES + BAR_BYTES + 1024;  // + align slack
    static_assert(SMEM_BYTES <= 227 * 1024, "exceeds the sm_100a per-CTA shared memory");
    static constexpr int kThreads = 256;
    // transaction bytes one stage's TMA loads credit to the (leader's) full
    // barrier: A slabs + B halves of b_rows rows, from every CTA of the pair
    static constexpr FI_HD int stage_tx_bytes(int b_rows) {
        return (A_BYTES + b_rows * BK * 2 * kNHalves) * kCtaGroup * kKB;
    }
    static constexpr int WS_FLOATS = BN * BM;     // one CTA's partial tile
};

// Tile id -> (tile row, tile col). With an explicit order table (the strategy's
// Block .swizzle) the unit id maps RowMajor as in Fireiron: row = u % tiles_m.
// Otherwise a grouped raster keeps a band of group_m A panels L2-resident while
// sweeping N.
FI_HD inline void tile_coords(const GemmArgs& a, int t, int& tm, int& tn) {
    if (a.tile_order) {
        const int u = a.tile_order[t];
        tm = u % a.tiles_m;
        tn = u / a.tiles_m;
        return;
    }
    const int band = a.group_m * a.tiles_n;
    const int g = t / band;
    const int local = t - g * band;
    int rows = a.tiles_m - g * a.group_m;
    if (rows > a.group_m) rows = a.group_m;
    tm = g * a.group_m + local % rows;
    tn = local / rows + a.n_rot;
    if (tn >= a.tiles_n) tn -= a.tiles_n;
}

// One work unit: K-blocks [k0, k1) of columns [n_off, n_off + width) of tile `tile`.
struct Unit {
    int tile, k0, k1;
    int n_off, width;
    int slice;  // K-slice index of a tail unit (sk_slices for a remainder)
    int slot;   // workspace slot its partial is published in (tail units)
};

// Workspace slot of the remainder partial of leftover tile i.
FI_HD inline int remainder_slot(const GemmArgs& a, int rest, int nclusters, int i) {
    const int e = i % a.sk_extra, j = i / a.sk_extra;
    return j == 0 ? rest * a.sk_slices + e : nclusters + e * (a.sk_q - 1) + j - 1;
}

// The unit sequence of one cluster. Tiles [0, D) run data-parallel (tile
// cluster, cluster+P, ...: consecutive clusters work on neighbouring tiles and
// advance through K in lockstep, so a wave's A/B panels are read once from
// DRAM). The R = T - D leftover tiles (the partial last wave) are split into S
// K-slices at fixed offsets: cluster c < R*S takes slice c / R of tile
// D + c % R. Clusters in the same slice stay in K lockstep (L2 reuse again),
// and slice 0 -- whose cluster also holds the K prefix -- owns the fixup.
// With args.streamk == 2 the leftover tiles are instead split along N into two
// half-width units (tcgen05 MMA with N = BN/2): no partials and no fixup.
template <int BN>
struct UnitIter {
    int t, step, kb, dp_tiles, tail_unit;
    int slices, rest, mode, w;
    int rem_e, rem_j, ncl;
    const GemmArgs* args;

    FI_HD UnitIter(const GemmArgs& a, int cluster, int nclusters) {
        args = &a;
        kb = a.k_blocks;
        const int tiles = a.tiles_m * a.tiles_n;
        mode = a.streamk;
        slices = mode ? a.sk_slices : 1;
        dp_tiles = mode ? a.sk_tile_begin : tiles;
        rest = tiles - dp_tiles;
        w = mode == 1 ? a.sk_w : 0;
        tail_unit = (mode && cluster < rest * slices) ? cluster : -1;
        rem_e = (w > 0 && cluster >= rest * slices && cluster < rest * slices + a.sk_extra)
                    ? cluster - rest * slices : -1;
        rem_j = 0;
        ncl = nclusters;
        t = cluster;
        step = nclusters;
    }
    FI_HD bool next(Unit& u) {
        if (args->sk_head && tail_unit >= 0) return take_tail(u);
        if (t < dp_tiles) {
            u = Unit{t, 0, kb, 0, BN, 0, 0};
            t += step;
            return true;
        }
        if (tail_unit < 0) {
            // remainder units of an extra cluster: tiles rem_e, rem_e + E, ...
            if (rem_e < 0) return false;
            const int i = rem_e + rem_j * args->sk_extra;
            if (i >= rest) return false;
            u = Unit{dp_tiles + i, slices * w, kb, 0, BN, slices, remainder_slot(*args, rest, ncl, i)};
            ++rem_j;
            return true;
        }
        return take_tail(u);
    }
    // the cluster's K-slice / N-split unit of a leftover tile
    FI_HD bool take_tail(Unit& u) {
        const int s = tail_unit / rest;
        u.tile = dp_tiles + tail_unit % rest;
        u.slice = s;
        u.slot = tail_unit;
        if (mode == 2) {  // N-split: half s of the tile's columns, full K
            u.k0 = 0;
            u.k1 = kb;
            u.width = BN / 2;
            u.n_off = s * (BN / 2);
        } else if (args->sk_pull) {  // 2-slice pull fixup: slice 1 publishes [0, w), slice 0 owns [w, kb)
            u.k0 = s == 0 ? w : 0;
            u.k1 = s == 0 ? kb : w;
            u.n_off = 0;
            u.width = BN;
        } else if (w > 0) {  // K-slice s of a tail with a remainder slice
            u.k0 = s * w;
            u.k1 = (s + 1) * w;
            u.n_off = 0;
            u.width = BN;
        } else {          // K-slice s
            u.k0 = kb * s / slices;
            u.k1 = kb * (s + 1) / slices;
            u.n_off = 0;
            u.width = BN;
        }
        tail_unit = -1;
        return true;
    }
};

// ---------------------------------------------------------------- host planner
// The persistent schedule of one launch (host side; also replayed by the CPU
// protocol checker, csrc/check/async_check.cpp). `clusters` is the grid's
// cluster count after the occupancy cap.
struct SchedulePlan {
    int status = 0;        // 0 ok, 1 shape (forced slices exceed the grid)
    int clusters = 0;      // clusters launched
    int mode = 0;          // 0 data-parallel, 1 K-slice tail, 2 N-split tail
    int slices = 1, sk_begin = 0;
    int sk_w = 0, sk_extra = 0, sk_q = 0, sk_pull = 0, sk_head = 0;
    long slots = 0;        // workspace slots (partials + flags), 0 without a tail split
};

template <int kCtaGroup, int BN, int kSplitK>
inline SchedulePlan plan_schedule(int tiles, int kb, int clusters, bool b_mn_major, int streamk,
                                  int force_slices, int remainder, int pull_d = -1, int head = 0) {
    using S = GemmShape<kCtaGroup, BN, kSplitK>;
    SchedulePlan P;
    // Tail split: whole waves data-parallel; the R leftover tiles of the partial
    // last wave are cut into S K-slices so the idle clusters share them.
    // S <= P/R (one unit per cluster), slices of >= 8 K-blocks, S <= 6 (an
    // owner stages S partial chunk ranges of <= ceil(NCH/S) chunks in the ring).
    const int dp_clusters = clusters < tiles ? clusters : tiles;
    const int full_waves = tiles / clusters;
    const int rest = tiles - full_waves * clusters;
    int slices = rest > 0 ? clusters / rest : 1;
    if (slices > kb / 8) slices = kb / 8;
    if (slices > 6) slices = 6;
    // N-split of the partial last wave: two half-width units per leftover tile
    const bool half_ok = BN >= 128 && (!b_mn_major || (BN / 2 / kCtaGroup) % 64 == 0);
    const bool nsplit_ok = half_ok && rest > 0 && rest * 2 <= clusters;
    int mode = 0;
    if (kSplitK == 1) {
        // auto: K-slices when each slice still has >= 24 K-blocks to amortise
        // the (parallel, ~5 us) fixup; otherwise N-split halves; else plain
        // (measured at 4096^3 / 1024^2x32768 / 4096^2x1024, profiles/round1/)
        if (streamk < 0)
            mode = (slices >= 2 && kb / slices >= 24) ? 1 : (full_waves >= 1 && nsplit_ok) ? 2 : 0;
        else if (streamk == 1) mode = slices >= 2 ? 1 : 0;
        else if (streamk == 2) mode = nsplit_ok ? 2 : 0;
    }
    if (mode == 2) slices = 2;
    // explicit split-K of every tile (a .splitk strategy on CTA pairs): all
    // tiles are K-sliced across clusters, partials reduced in shared memory
    int sk_begin = full_waves * clusters;
    if (kSplitK == 1 && force_slices > 1) {
        if (tiles * force_slices > clusters) {
            P.status = 1;
            return P;
        }
        mode = 1;
        slices = force_slices;
        sk_begin = 0;
    }
    // Remainder slice: with E = clusters - R*S extra clusters, main slices
    // get W = ceil(q*kb / (S*q + 1)) K-blocks and the remainder kb - S*W runs
    // on the extra clusters, q = ceil(R/E) remainders each, so every cluster
    // has ~q*kb/(S*q+1) blocks instead of kb/S (C3: 114 vs 128). Only when the
    // remainder units stay long enough (>= 24 blocks) to hide their own
    // epilogue and the owners' staging of S+1 sources fits in the ring.
    if (mode == 1 && remainder != 0) {
        const int rest_tiles = tiles - sk_begin;
        const int extra = clusters - rest_tiles * slices;
        const int e = extra < rest_tiles ? extra : rest_tiles;
        if (e > 0) {
            const int q = (rest_tiles + e - 1) / e;
            const int w = (q * kb + slices * q) / (slices * q + 1);
            const int rk = kb - slices * w;
            constexpr int NCH = BN / 32;
            const int nown = (NCH + slices - 1) / slices;
            const bool fits = (slices + 1) * nown * 32 * S::BM * 4 <= S::RING_BYTES;
            if (fits && rk >= 24 && q * rk <= w && w * 100 <= (kb / slices) * 97) {
                P.sk_w = w;
                P.sk_extra = e;
                P.sk_q = q;
            }
        }
    }
    // pull fixup for 2-slice tails: the publisher's share is shorter by the
    // time its 128 KB/CTA publish takes (~pull_d K-blocks at the per-SM write
    // rate), so the owner's MMA covers it
    // (or, with head >= 1 and data-parallel tiles to follow, equal halves run
    // first so the whole fixup overlaps the next main loops)
    if (mode == 1 && slices == 2 && P.sk_w == 0 && pull_d >= 0 && kb >= 24) {
        const bool head_ok = head > 0 && sk_begin > 0;
        int w = head_ok ? kb / 2 : (kb - pull_d) / 2;
        if (w < 8) w = 8;
        P.sk_pull = 1;
        P.sk_head = head_ok ? 1 : 0;
        P.sk_w = w;
    }
    P.mode = mode;
    P.slices = slices;
    P.sk_begin = sk_begin;
    P.clusters = mode ? clusters : dp_clusters;
    if (P.clusters < 1) P.clusters = 1;
    if (mode) P.slots = static_cast<long>(clusters) + (P.sk_q > 1 ? static_cast<long>(P.sk_extra) * (P.sk_q - 1) : 0);
    return P;
}

}  // namespace fireiron::sm100
