// Warp-specialised, persistent tcgen05 GEMM: the sm_100a lowering of the
// Fireiron tensor-core strategy
//
//   tile BMxBN .to block [.pair]           -> persistent CTA (pair) work loop
//   [split K/S .splitk]                    -> S CTAs of a cluster share a tile
//   epilog tm { init {TMEM_ZERO} store {tile 32 BN .to warp; TMEM_STORE} }
//   split 64 .stages S                     -> S-deep TMA/MMA mbarrier ring
//   load a sh {TMA_LOAD}  load b sh {TMA_LOAD}
//   done                                   -> UMMA leaf (tcgen05.mma kind::f16)
//
// Roles (256 threads): warps 0, 3 and 2 = TMA producers (ring stages s % 3 =
// 0, 1, 2), warp 1 = MMA issuer (leader CTA), warp 2 also allocates TMEM,
// warps 4..7 = epilogue (TMEM -> RF -> GL). The
// producer and MMA warps run their loops with all 32 lanes so every operand is
// warp-uniform (uniform registers); one elected lane issues each TMA / MMA /
// commit (elect.sync inside the asm) -- no per-issue waterfall, measured 3-16 %
// faster on narrow tiles (profiles/round2/ab_warp_issue.log).
// Accumulators are double-buffered in TMEM so the epilogue of one work unit
// overlaps the main loop of the next. With kCtaGroup == 2 a CTA pair (cluster
// of 2) computes a 256xBN tile with tcgen05.mma.cta_group::2: each CTA stages
// its 128 rows of A and BN/2 rows of B; the accumulator rows stay in each
// CTA's TMEM.
//
// Work distribution (which K-blocks of which tile a cluster computes):
//  * data-parallel: whole tiles, round-robin over the persistent clusters;
//  * tail split (args.streamk): whole waves of tiles run data-parallel; the
//    leftover tiles of the partial last wave are split into S K-slices at
//    fixed offsets so the idle clusters share their work (a stream-K variant
//    that keeps clusters in K lockstep: contiguous stream-K ranges measured 5x
//    the DRAM traffic). Slices 1..S-1 publish fp32 partials (global workspace
//    slot + epoch flag); slice 0 stages them into its idle operand ring with
//    bulk copies and adds them in K order, so results are deterministic;
//  * cluster split-K (kSplitK > 1): the S CTAs (pairs) of a cluster own K
//    slices of the same tile; partial accumulators are published in shared
//    memory (reusing the drained operand ring) and reduced through DSMEM in a
//    fixed rank order before the fused epilog store. Cluster rank =
//    split_rank * kCtaGroup + pair_rank.
#pragma once

#ifndef FI_TC_WAITPROF
#define FI_TC_WAITPROF 0  // diagnostic build: per-CTA barrier-wait cycles in trace row 15
#endif


#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "ptx.cuh"
#include "schedule.hpp"

namespace fireiron::sm100 {

__device__ __forceinline__ unsigned long long global_timer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void trace_stamp(const GemmArgs& a, int unit, int ev) {
    if (a.trace && unit < 16) {
        a.trace[(blockIdx.x * 16 + unit) * 16 + ev] = global_timer_ns();
        a.trace[(blockIdx.x * 16 + unit) * 16 + 8 + ev] = clock64();  // SM clock: effective MHz
    }
}

template <typename T>
__device__ __forceinline__ T cvt_out(float v);
template <>
__device__ __forceinline__ float cvt_out<float>(float v) { return v; }
template <>
__device__ __forceinline__ __half cvt_out<__half>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ __nv_bfloat16 cvt_out<__nv_bfloat16>(float v) {
    return __float2bfloat16_rn(v);
}

// Store 32 consecutive columns of one accumulator row. Column-major C (the
// Fireiron default) makes each per-column store a coalesced 32-lane segment.
template <typename T>
__device__ __forceinline__ void store_row32(const GemmArgs& a, int m, int n, const float (&v)[32]) {
    T* C = static_cast<T*>(a.C);
    if (a.c_row_major) {
        T* p = C + static_cast<long>(m) * a.ldc + n;
#pragma unroll
        for (int j = 0; j < 32; ++j) p[j] = cvt_out<T>(v[j]);
    } else {
        T* p = C + static_cast<long>(n) * a.ldc + m;
#pragma unroll
        for (int j = 0; j < 32; ++j) p[static_cast<long>(j) * a.ldc] = cvt_out<T>(v[j]);
    }
}

__device__ __forceinline__ void store_row32_any(const GemmArgs& a, int m, int n,
                                                const float (&v)[32]) {
    switch (static_cast<OutType>(a.out_type)) {
        case OutType::F32: store_row32<float>(a, m, n, v); break;
        case OutType::F16: store_row32<__half>(a, m, n, v); break;
        case OutType::BF16: store_row32<__nv_bfloat16>(a, m, n, v); break;
    }
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Gated B (fused all-gather): spin until tile column tn's chunk is flagged
// ready. Out of line: the producer's loop keeps its code shape when ungated.
__device__ __noinline__ void wait_b_chunk(const unsigned* f, unsigned epoch) {
    if (ld_acquire_gpu(f) < epoch) {
        const unsigned long long t0 = global_timer_ns();
        while (ld_acquire_gpu(f) < epoch) {
            __nanosleep(256);
            if (global_timer_ns() - t0 > 4000000000ull) __trap();  // a lost chunk: fail, not hang
        }
    }
    fence_proxy_async_global();  // copy-engine writes before the TMA reads
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// bar.sync among the 4 epilogue warps only (named barrier 1, 128 threads)
__device__ __forceinline__ void epilogue_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Kernel body; the tensor maps must be __grid_constant__ kernel parameters
// (TMA reads them through their parameter-space address).
template <int kCtaGroup, int BN, int kSplitK, int kSlabs, int kNHalves, int kMcast, int kKB = 1>
__device__ __forceinline__ void fi_sm100_gemm_body(const CUtensorMap& tmA, const CUtensorMap& tmB,
                                                   const CUtensorMap& tmB2, const CUtensorMap& tmC,
                                                   const CUtensorMap& tmC2,
                                                   const GemmArgs& args) {
    using S = GemmShape<kCtaGroup, BN, kSplitK, kSlabs, kNHalves, kKB>;
    static_assert(kKB == 1 || (kKB == 2 && kMcast == 1), "two-K-block stages: not with multicast");
    static_assert(kSlabs * kNHalves == 1 || (kCtaGroup == 2 && kSplitK == 1 && kSlabs * kNHalves == 2),
                  "slab / N-half tiles pair with CTA pairs, one doubling, no cluster split-K");
    constexpr bool kWide = kSlabs * kNHalves > 1;  // whole-TMEM accumulator, whole-tile units only
    // kMcast = 2 (.multicast): a cluster of two CTA pairs computes two tiles that are
    // neighbours along N; each pair's CTA of rank r receives the same A rows, so
    // the two CTAs of rank r load one 64-row half each and multicast it to both.
    // A stage slot is refilled only after both pairs' MMAs released it.
    static_assert(kMcast == 1 || (kCtaGroup == 2 && kSplitK == 1 && !kWide), "multicast pairs tiles of one CTA pair");
    constexpr int kBNTile = S::BN_TILE * kMcast;  // columns of one scheduled unit (both pairs)
    constexpr int kStages = S::kStages;
    constexpr int kClusterSize = kCtaGroup * kSplitK * kMcast;

    extern __shared__ uint8_t smem_raw[];
    // 1024B alignment for the 128B-swizzle atoms
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
    uint8_t* ring = smem;
    float* red = reinterpret_cast<float*>(ring);  // split-K scratch (ring reuse)
    float* epi = reinterpret_cast<float*>(smem + S::RING_BYTES);  // [2][32 cols][128 rows] C staging
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::RING_BYTES + S::EPI_BYTES);
    uint64_t* full_bar = bars;                      // [kStages] TMA -> MMA
    uint64_t* empty_bar = bars + kStages;           // [kStages] MMA -> TMA
    uint64_t* tfull_bar = bars + 2 * kStages;       // [2] MMA -> epilogue
    uint64_t* tempty_bar = bars + 2 * kStages + 2;  // [2] epilogue -> MMA
    uint64_t* rfull_bar = bars + 2 * kStages + 4;   // split-K: all partials published
    uint64_t* rempty_bar = bars + 2 * kStages + 5;  // split-K: all peers done reading
    uint64_t* stage_bar = bars + 2 * kStages + 6;   // [2] stream-K fixup staging
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 8);
    uint64_t* src_bar = bars + 2 * kStages + 10;    // [8] symmetric fixup: one per K-slice source

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint32_t crank = kClusterSize > 1 ? cluster_ctarank() : 0;
    const uint32_t pair_rank = crank % kCtaGroup;   // position inside the CTA pair
    const uint32_t split_rank = kSplitK > 1 ? crank / kCtaGroup : 0;  // K slice owned by this CTA
    const bool mma_leader = pair_rank == 0;
    const uint16_t pair_mask = static_cast<uint16_t>(3u << (crank - pair_rank));
    const uint32_t mc_rank = kMcast > 1 ? crank / kCtaGroup : 0;  // which pair of the multicast cluster
    const uint16_t mc_all = static_cast<uint16_t>((1u << kClusterSize) - 1);  // every CTA of the cluster
    const uint16_t mc_a_mask = static_cast<uint16_t>((1u << pair_rank) | (1u << (kCtaGroup + pair_rank)));

    if (threadIdx.x == 0 && args.trace) {  // kernel entry (event 7 of unit 0)
        args.trace[(blockIdx.x * 16) * 16 + 7] = global_timer_ns();
        args.trace[(blockIdx.x * 16) * 16 + 15] = clock64();
    }
    if (threadIdx.x == 32) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], kMcast);  // a release from every pair that reads the slot
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull_bar[b], 1);
            mbar_init(&tempty_bar[b], 4 * kCtaGroup);
        }
        mbar_init(rfull_bar, 4 * kSplitK);
        mbar_init(rempty_bar, 4 * kSplitK);
        mbar_init(&stage_bar[0], 1);
        mbar_init(&stage_bar[1], 1);
        for (int j = 0; j < 8; ++j) mbar_init(&src_bar[j], 1);
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        tma_prefetch_desc(&tmB2);
    }
    if (warp == 2) tmem_alloc<kCtaGroup>(tmem_slot, S::TMEM_COLS);
    if (threadIdx.x == 64 && args.trace) args.trace[(blockIdx.x * 16 + 1) * 16 + 7] = global_timer_ns();  // alloc done
    tc_fence_before();
    if constexpr (kClusterSize > 1) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0 && args.trace) args.trace[(blockIdx.x * 16 + 2) * 16 + 7] = global_timer_ns();  // prologue synced

    const int nst = (args.stages > 0 && args.stages < kStages) ? args.stages : kStages;
    const int cluster = blockIdx.x / kClusterSize;
    const int nclusters = gridDim.x / kClusterSize;
    const int kb0 = static_cast<int>(split_rank) * args.k_blocks;  // first K block of my slice

    // wide tiles (two A slabs or two B halves per stage: 48 KB, 4 stages) keep one
    // producer -- three cost them 1-7 % (stages issued out of order), and their
    // MMA work per stage hides one warp's issue time (ab_three_producers.log)
    constexpr int kProducers = kSlabs * kNHalves > 1 ? 1 : 3;
    if (warp == 0 || (kProducers == 3 && (warp == 2 || warp == 3))) {
        // ------------------------------------------------------------ TMA producers
        // Three warps share the ring: stage s is filled by warp 0, 3 or 2 for
        // s % 3 = 0, 1, 2 (each waits for its stage's empty barrier, credits the
        // expected bytes and issues that stage's A and B loads; warp 2 allocated
        // TMEM before the prologue sync). A warp spends ~500 SM cycles per stage
        // issuing its loads (FI_TC_WAITPROF builds), so one producer capped narrow
        // tiles (N <= 128: 20-24 KB per K block) at ~400 cycles per K block; two
        // and then three issuers cut that to ~295 (profiles/round2/ab_split_producer.log,
        // ab_three_producers.log). A stage always has the same producer, so no
        // producer can get two fills ahead of a stage's empty barrier and pass its
        // parity wait on a stale phase (ownership by fill count instead broke that
        // with shallow rings -- the CPU protocol checker's find, experiments.txt).
        // Each warp runs its loop with all 32 lanes so every operand is warp-
        // uniform (uniform registers, no per-issue waterfall); one lane issues.
        {
            const bool issuer = lane == 0 && warp == 0;
            int s = 0;
            uint32_t ph = 0;
            int it = 0;
            // L2 policy (args.l2_hint): 1 = A panels evict-last (a raster band re-reads
            // them every wave) and B evict-first; 2 = the opposite
            const uint64_t pol_a = args.l2_hint == 1 ? kL2EvictLast : args.l2_hint == 2 ? kL2EvictFirst : kL2EvictNormal;
            const uint64_t pol_b = args.l2_hint == 1 ? kL2EvictFirst : args.l2_hint == 2 ? kL2EvictLast : kL2EvictNormal;
            UnitIter<BN> units(args, cluster, nclusters);
            Unit u;
#if FI_TC_WAITPROF
            long long w_empty = 0;
            const long long t_loop = clock64();
#endif
            while (units.next(u)) {
                int tm, tn;
                tile_coords(args, u.tile, tm, tn);
                const bool half = u.width != BN;
                const int b_rows = u.width / kCtaGroup;  // B rows staged by this CTA
                const uint32_t tx = static_cast<uint32_t>(S::stage_tx_bytes(b_rows));
                if constexpr (kSplitK > 1) {
                    // the ring doubles as the reduction scratch: wait until every
                    // peer has read my previous partial tile
                    mbar_wait_cluster(rempty_bar, (static_cast<uint32_t>(it) & 1) ^ 1);
                    fence_proxy_async();
                }
                if (args.b_ready)  // gated B: the tile's column chunk has landed
                    wait_b_chunk(args.b_ready + tn / args.b_chunk_tiles, args.b_epoch);
                if (issuer) trace_stamp(args, it, 0);
                ++it;
                const int m0 = tm * S::BM_TILE + static_cast<int>(pair_rank) * S::BM;
                const int n0 = tn * kBNTile + static_cast<int>(mc_rank) * S::BN_TILE + u.n_off +
                               static_cast<int>(pair_rank) * b_rows;
                for (int kb = u.k0; kb < u.k1; kb += kKB) {
                    if (kProducers == 3 && warp != (s % 3 == 0 ? 0 : s % 3 == 1 ? 3 : 2)) {  // another producer's stage
                        if (++s == nst) { s = 0; ph ^= 1; }
                        continue;
                    }
#if FI_TC_WAITPROF
                    {
                        const long long t = clock64();
                        mbar_wait(&empty_bar[s], ph ^ 1);
                        w_empty += clock64() - t;
                    }
#else
                    mbar_wait(&empty_bar[s], ph ^ 1);
#endif
                    uint8_t* sa = ring + s * S::STAGE_BYTES;
                    uint8_t* sb = sa + S::A_STAGE_BYTES;
                    const int k0 = (kb0 + kb) * S::BK;
                    // kKB = 2: the box covers two K blocks even when the unit has one
                    // left (the second is read but not multiplied; past K it is zero-
                    // filled); the transaction count is the full box either way
                    if (mma_leader) mbar_arrive_expect_tx_warp(&full_bar[s], tx);
                    auto load = [&](void* dst, const CUtensorMap* map, int c0, int c1, uint64_t pol) {
                        if (args.l2_hint) {
                            if (lane != 0) return;
                            if constexpr (kCtaGroup == 1) tma_load_2d_hint(dst, map, &full_bar[s], c0, c1, pol);
                            else tma_load_2d_pair_hint(dst, map, &full_bar[s], c0, c1, pol);
                        } else {
                            if constexpr (kCtaGroup == 1) tma_load_2d_warp(dst, map, &full_bar[s], c0, c1);
                            else tma_load_2d_pair_warp(dst, map, &full_bar[s], c0, c1);
                        }
                    };
                    auto load3 = [&](void* dst, const CUtensorMap* map, int c0, int c1, int c2) {
                        if constexpr (kCtaGroup == 1) tma_load_3d_warp(dst, map, &full_bar[s], c0, c1, c2);
                        else tma_load_3d_pair_warp(dst, map, &full_bar[s], c0, c1, c2);
                    };
                    if constexpr (kMcast > 1) {
                        // my 64-row half of the A block, to me and my rank-twin in the other pair
                        const int h = static_cast<int>(mc_rank);
                        if (lane != 0) {
                        } else if (args.a_mn_major)
                            tma_load_2d_pair_mc(sa + h * 8192, &tmA, &full_bar[s], m0 + h * 64, k0, mc_a_mask);
                        else  // tmA box: 64 K x 64 rows for multicast plans
                            tma_load_2d_pair_mc(sa + h * 8192, &tmA, &full_bar[s], k0, m0 + h * 64, mc_a_mask);
                    } else {
#pragma unroll
                        for (int sl = 0; sl < kSlabs; ++sl) {  // slab sl: rows m0 + sl * BM_MMA
                            uint8_t* sas = sa + sl * kKB * S::SLAB_BYTES;
                            const int m0s = m0 + sl * S::BM_MMA;
                            if constexpr (kKB == 2) {
                                // one box for both K blocks: MN-major {64, 64, 2 panels, 2 K blocks},
                                // K-major {64 k, 128 rows, 2 K blocks}
                                if (args.a_mn_major) {
                                    if (lane != 0) {
                                    } else if constexpr (kCtaGroup == 1) tma_load_4d(sas, &tmA, &full_bar[s], 0, 0, m0s / 64, kb0 + kb);
                                    else tma_load_4d_pair(sas, &tmA, &full_bar[s], 0, 0, m0s / 64, kb0 + kb);
                                } else {
                                    load3(sas, &tmA, 0, m0s, kb0 + kb);
                                }
                            } else if (args.a_mn_major) {
                                // one 3D box {64, 64, 2}: both 64-row SW128 panels of the slab
                                // (tmA viewed as 64 rows x K x M/64 panels) -- one TMA op instead
                                // of two (measured +3 % on C2)
                                load3(sas, &tmA, 0, k0, m0s / 64);
                            } else {
                                load(sas, &tmA, k0, m0s, pol_a);
                            }
                        }
                    }
#pragma unroll
                    for (int h = 0; h < kNHalves; ++h) {  // N half h: rows n0 + h * BN
                        uint8_t* sbh = sb + h * kKB * S::HALF_B_BYTES;
                        const int n0h = n0 + h * BN;
                        if (args.b_mn_major) {
                            for (int b = 0; b < kKB; ++b)
                                for (int j = 0; j < b_rows / 64; ++j)
                                    load(sbh + b * b_rows * 128 + j * 8192, &tmB, n0h + j * 64, k0 + b * S::BK, pol_b);
                        } else if constexpr (kKB == 2) {
                            load3(sbh, half ? &tmB2 : &tmB, 0, n0h, kb0 + kb);
                        } else {
                            load(sbh, half ? &tmB2 : &tmB, k0, n0h, pol_b);  // tmB2: box of BN_LOCAL/2 rows
                        }
                    }
                    if (++s == nst) { s = 0; ph ^= 1; }
                }
            }
#if FI_TC_WAITPROF
            if (issuer && args.trace) {
                unsigned long long* row = args.trace + (blockIdx.x * 16 + 15) * 16;
                row[10] = static_cast<unsigned long long>(w_empty);
                row[11] = static_cast<unsigned long long>(clock64() - t_loop);
            }
#endif
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (mma_leader) {
            const bool issuer = lane == 0;
            const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem_base, 0);  // provably warp-uniform
            // instruction descriptor: f32 accumulate, a/b format, majors, N>>3, M>>4
            const uint32_t idesc_base = (1u << 4) | (static_cast<uint32_t>(args.ab_format) << 7) |
                                        (static_cast<uint32_t>(args.ab_format) << 10) |
                                        (static_cast<uint32_t>(args.a_mn_major) << 15) |
                                        (static_cast<uint32_t>(args.b_mn_major) << 16) |
                                        (static_cast<uint32_t>(S::BM_MMA >> 4) << 24);
            // K-major: rows of 128B, 8-row atoms 1024B apart (SBO), K step = 32B.
            // MN-major: 64-element chunks 8KB apart (LBO), 8 k-rows per atom (SBO 1KB),
            //           K step of 16 = two atoms = 2KB.
            const uint32_t a_lbo = args.a_mn_major ? 8192 : 16, a_kstep = args.a_mn_major ? 2048 : 32;
            const uint32_t b_lbo = args.b_mn_major ? 8192 : 16, b_kstep = args.b_mn_major ? 2048 : 32;
            // single-slab, single-N-half tiles issue a K block's four MMAs from one
            // asm statement (umma_f16_kblock_warp): with two producers feeding the
            // ring, the MMA warp's issue time bounds N = 64 tiles (~255 -> ~200 SM
            // cycles per K block, profiles/round2/ab_kblock_mma_issue.log)
            constexpr bool kWholeKBlock = kSlabs == 1 && kNHalves == 1 && S::BK == 64;
            int s = 0;
            uint32_t ph = 0;
            int it = 0;
            UnitIter<BN> units(args, cluster, nclusters);
            Unit u;
#if FI_TC_WAITPROF
            long long w_full = 0, n_kb = 0;
            const long long t_loop = clock64();
#endif
            while (units.next(u)) {
                const int buf = S::kAccBufs == 2 ? (it & 1) : 0;
                const uint32_t use = static_cast<uint32_t>(S::kAccBufs == 2 ? (it >> 1) : it);
                ++it;
                const uint32_t idesc = idesc_base | (static_cast<uint32_t>(u.width >> 3) << 17);
                mbar_wait_cluster(&tempty_bar[buf], (use & 1) ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_u + static_cast<uint32_t>(buf * S::ACC_COLS);
                const uint32_t b_kb_bytes = static_cast<uint32_t>(u.width / kCtaGroup) * 128;  // B rows x 128 B
                for (int kb = u.k0; kb < u.k1; kb += kKB) {
#if FI_TC_WAITPROF
                    {
                        const long long t = clock64();
                        mbar_wait(&full_bar[s], ph);
                        w_full += clock64() - t;
                        ++n_kb;
                    }
#else
                    mbar_wait(&full_bar[s], ph);
#endif
                    tc_fence_after();
                    const uint32_t sa = smem_u32(ring + s * S::STAGE_BYTES);
                    const uint32_t sb = sa + S::A_STAGE_BYTES;
#pragma unroll
                    for (int b = 0; b < kKB; ++b) {
                        if (kKB > 1 && kb + b >= u.k1) break;  // a unit's odd last K block
                        if constexpr (kWholeKBlock) {
                            // the whole K block from one elected lane (see umma_f16_kblock_warp)
                            const uint32_t acc = (kb > u.k0 || b > 0) ? 1u : 0u;
                            umma_f16_kblock_warp<kCtaGroup>(
                                d_tmem, static_cast<uint32_t>(smem_desc_sw128(sa + b * S::SLAB_BYTES, a_lbo, 1024)),
                                a_kstep >> 4,
                                static_cast<uint32_t>(smem_desc_sw128(sb + b * b_kb_bytes, b_lbo, 1024)),
                                b_kstep >> 4, idesc, acc);
                        } else {
#pragma unroll
                        for (int k = 0; k < S::BK / 16; ++k) {
                            const uint32_t acc = (kb > u.k0 || b > 0 || k > 0) ? 1u : 0u;
                            if constexpr (kNHalves == 2) {
                                // two N halves share A: the first MMA fills the A collector,
                                // the second reuses it (A leaves shared memory once)
                                uint64_t ad = smem_desc_sw128(sa + b * S::SLAB_BYTES + k * a_kstep, a_lbo, 1024);
                                uint64_t bd0 = smem_desc_sw128(sb + b * b_kb_bytes + k * b_kstep, b_lbo, 1024);
                                uint64_t bd1 = smem_desc_sw128(sb + kKB * S::HALF_B_BYTES + b * b_kb_bytes + k * b_kstep,
                                                               b_lbo, 1024);
                                umma_f16_collect_warp<kCtaGroup, 1>(d_tmem, ad, bd0, idesc, acc);
                                umma_f16_collect_warp<kCtaGroup, 2>(d_tmem + BN, ad, bd1, idesc, acc);
                            } else {
                                uint64_t bd = smem_desc_sw128(sb + b * b_kb_bytes + k * b_kstep, b_lbo, 1024);
#pragma unroll
                                for (int sl = 0; sl < kSlabs; ++sl) {  // slabs share the B operand
                                    uint64_t ad = smem_desc_sw128(
                                        sa + (sl * kKB + b) * S::SLAB_BYTES + k * a_kstep, a_lbo, 1024);
                                    umma_f16_warp<kCtaGroup>(d_tmem + sl * BN, ad, bd, idesc, acc);
                                }
                            }
                        }
                        }
                    }
                    if constexpr (kCtaGroup == 1) umma_commit_warp(&empty_bar[s]);
                    else umma_commit_pair_warp(&empty_bar[s], kMcast > 1 ? mc_all : pair_mask);
                    if (++s == nst) { s = 0; ph ^= 1; }
                }
                if (issuer) {
                    if constexpr (kCtaGroup == 1) umma_commit(&tfull_bar[buf]);
                    else umma_commit_pair(&tfull_bar[buf], pair_mask);
                    trace_stamp(args, it - 1, 1);
                }
            }
#if FI_TC_WAITPROF
            if (issuer && args.trace) {
                unsigned long long* row = args.trace + (blockIdx.x * 16 + 15) * 16;
                row[8] = static_cast<unsigned long long>(w_full);
                row[9] = static_cast<unsigned long long>(clock64() - t_loop);
                row[12] = static_cast<unsigned long long>(n_kb);
            }
#endif
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue
        const int q = warp - 4;  // TMEM lane quarter owned by this warp
        const int row = q * 32 + lane;
        int it = 0;
        UnitIter<BN> units(args, cluster, nclusters);
        Unit u;
        const int kb = args.k_blocks;
        uint32_t epi_chunk = 0;  // staged C chunks so far (alternating buffers)
        // this launch's epoch for the tail-fixup flags: the device counter + 1 when
        // the workspace carries one (correct under CUDA-graph replay, where a
        // host-side epoch would be frozen at capture), else the host's value. One
        // thread reads it and counts the CTA in; the last CTA in advances the
        // counter for the next launch -- all while the first main loop runs.
        if (q == 0 && lane == 0) {
            unsigned e = args.epoch;
            if (args.epoch_ctr) {
                e = *reinterpret_cast<volatile const unsigned*>(args.epoch_ctr) + 1u;
                __threadfence();  // the read completes before this CTA is counted in
                if (atomicAdd(args.epoch_ctr + 1, 1u) == gridDim.x - 1) {
                    __threadfence();
                    args.epoch_ctr[1] = 0;
                    atomicAdd(args.epoch_ctr, 1u);
                }
            }
            tmem_slot[1] = e;
        }
        epilogue_bar();
        const unsigned epoch = tmem_slot[1];
        // TMEM -> RF -> SMEM for nch 32-column chunks into slot(c) (thread `row`
        // writes bank row % 32: conflict-free), TMEM loads double-buffered; after
        // each chunk pair one proxy fence + barrier, then one thread issues
        // store(c), store(c+1) and commits them as a bulk group.
        auto drain_pairs = [&](uint32_t tb, int nch, auto slot, auto store) {
            uint32_t r0[32], r1[32];
            tmem_ld_32x32b_x32(tb, r0);
#pragma unroll 1
            for (int c = 0; c < nch; c += 2) {
                tmem_ld_wait();
                tmem_ld_32x32b_x32(tb + (c + 1) * 32, r1);
                float* d0 = slot(c) + row;
#pragma unroll
                for (int j = 0; j < 32; ++j) d0[j * S::BM] = __uint_as_float(r0[j]);
                tmem_ld_wait();
                if (c + 2 < nch) tmem_ld_32x32b_x32(tb + (c + 2) * 32, r0);
                float* d1 = slot(c + 1) + row;
#pragma unroll
                for (int j = 0; j < 32; ++j) d1[j * S::BM] = __uint_as_float(r1[j]);
                fence_proxy_async();
                epilogue_bar();
                if (q == 0 && lane == 0) {
                    store(c);
                    store(c + 1);
                    bulk_commit_group();
                }
            }
        };
        // one unit of look-ahead: the cluster's last unit drains through the idle
        // operand ring (no buffer reuse, one fence/barrier per chunk pair)
        Unit nxt;
        bool have = units.next(u);
        while (have) {
            const bool have_next = units.next(nxt);
            const bool last_unit = !have_next;
            int tm, tn;
            tile_coords(args, u.tile, tm, tn);
            const int buf = S::kAccBufs == 2 ? (it & 1) : 0;
            const uint32_t use = static_cast<uint32_t>(S::kAccBufs == 2 ? (it >> 1) : it);
            const uint32_t tile_use = static_cast<uint32_t>(it);
            ++it;
            mbar_wait(&tfull_bar[buf], use & 1);
            if (q == 0 && lane == 0) trace_stamp(args, it - 1, 2);
            tc_fence_after();
            const int m = tm * S::BM_TILE + static_cast<int>(pair_rank) * S::BM + row;
            const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                                   static_cast<uint32_t>(buf * S::ACC_COLS);
            // whole-K units: TMEM chunk c (columns c * 32) of accumulator c / nchu --
            // A slab (rows + slab * BM_MMA) or N half (columns + half * BN)
            const int nchu = u.width / 32;
            const int nch_all = kSlabs * kNHalves * nchu;
            auto chunk_row = [&](int c) { return kSlabs > 1 ? (c / nchu) * S::BM_MMA : 0; };
            auto chunk_col = [&](int c) {
                return tn * kBNTile + static_cast<int>(mc_rank) * S::BN_TILE + u.n_off +
                       (kNHalves > 1 ? (c / nchu) * BN : 0) + (c % nchu) * 32;
            };
            if constexpr (kSplitK == 1) {
                auto release_tmem = [&] {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (kCtaGroup == 1) mbar_arrive(&tempty_bar[buf]);
                        else mbar_arrive_cluster(&tempty_bar[buf], crank - pair_rank);
                    }
                    __syncwarp();
                };
                if (u.k0 == 0 && u.k1 == kb && args.c_tma && last_unit && args.ring_drain &&
                    nch_all * 32 * S::BM * 4 <= S::RING_BYTES) {
                    // the cluster's last unit: stage all chunks in the idle ring, TMA
                    // store them pairwise; TMEM loads double-buffered
                    const int m_cta = tm * S::BM_TILE + static_cast<int>(pair_rank) * S::BM;
                    float* stage0 = reinterpret_cast<float*>(ring);
                    drain_pairs(tbase, nch_all, [&](int c) { return stage0 + c * (32 * S::BM); },
                                [&](int c) {  // chunks c, c+1 are adjacent in smem and in C: one 64-column box
                                    if ((c & 1) == 0)
                                        tma_store_2d(&tmC2, stage0 + c * (32 * S::BM), m_cta + chunk_row(c), chunk_col(c));
                                });
                    release_tmem();
                } else if (u.k0 == 0 && u.k1 == kb && args.c_tma) {
                    // whole K range, f32 col-major C: TMEM -> RF -> SMEM chunk -> TMA store.
                    // Column j of a chunk is 128 contiguous rows (512 B): thread `row`
                    // writes bank row % 32, conflict-free; one thread stores the chunk.
                    const int m_cta = tm * S::BM_TILE + static_cast<int>(pair_rank) * S::BM;
                    // chunk pairs fill both epi buffers, then ONE 64-column TMA store
                    // (half the store ops: the SM's TMA unit also feeds the next main loop)
#pragma unroll 1
                    for (int c = 0; c < nch_all; ++c) {
                        uint32_t r[32];
                        tmem_ld_32x32b_x32(tbase + c * 32, r);
                        float* stage = epi + (c & 1) * (32 * S::BM);
                        if ((c & 1) == 0) {
                            if (q == 0 && lane == 0) bulk_wait_group_read<0>();  // the previous pair's store left epi
                            epilogue_bar();
                        }
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 32; ++j) stage[j * S::BM + row] = __uint_as_float(r[j]);
                        if (c & 1) {
                            fence_proxy_async();
                            epilogue_bar();
                            if (q == 0 && lane == 0) {
                                tma_store_2d(&tmC2, epi, m_cta + chunk_row(c - 1), chunk_col(c - 1));
                                bulk_commit_group();
                            }
                            __syncwarp();
                        }
                    }
                    // leave the epi buffers free for the next unit's path (each starts
                    // behind an epilogue barrier this thread also reaches)
                    if (q == 0 && lane == 0) bulk_wait_group_read<0>();
                    release_tmem();
                } else if (u.k0 == 0 && u.k1 == kb) {
                    // whole K range (a tile or an N-split half): TMEM -> RF -> GL
#pragma unroll 1
                    for (int c = 0; c < nch_all; ++c) {
                        uint32_t r[32];
                        tmem_ld_32x32b_x32(tbase + c * 32, r);
                        tmem_ld_wait();
                        float v[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                        store_row32_any(args, m + chunk_row(c), chunk_col(c), v);
                    }
                    release_tmem();
                } else if (kWide || kMcast > 1) {
                    // slab / N-half / multicast tiles run whole-K units only (never split)
                } else if (args.sk_pull) {
                    // 2-slice pull fixup. Slice 1 (K-blocks [0, w)) publishes its whole
                    // partial; slice 0 ([w, kb)) streams it back chunk by chunk into
                    // the epi buffers, adds it and stores C. As the cluster's last
                    // unit (ring idle) slice 0 is longer by the publish time and
                    // both stage through the ring; as its first unit (args.sk_head:
                    // the ring feeds the next main loop) the halves are equal, the
                    // publisher stages through the epi buffers and the owner stores
                    // C from registers -- the exchange overlaps the next tiles.
                    constexpr int NCH = BN / 32;
                    constexpr uint32_t kChunkFloats = 32 * S::BM;
                    constexpr uint32_t kChunkBytes = kChunkFloats * 4;
                    const int rest = args.tiles_m * args.tiles_n - args.sk_tile_begin;
                    const int tile_idx = u.tile - args.sk_tile_begin;
                    float* stage0 = reinterpret_cast<float*>(ring);
                    if (u.slice == 1) {
                        float* slot_ws = args.workspace + static_cast<long>(u.slot * kCtaGroup + pair_rank) * S::WS_FLOATS;
                        if (!args.sk_head) {
                            drain_pairs(tbase, NCH, [&](int c) { return stage0 + c * kChunkFloats; },
                                        [&](int c) { bulk_copy_s2g(slot_ws + c * kChunkFloats, stage0 + c * kChunkFloats, kChunkBytes); });
                        } else {
#pragma unroll 1
                            for (int c = 0; c < NCH; ++c) {
                                uint32_t r[32];
                                tmem_ld_32x32b_x32(tbase + c * 32, r);
                                float* stage = epi + (epi_chunk++ & 1) * kChunkFloats;
                                if (q == 0 && lane == 0) bulk_wait_group_read<1>();
                                epilogue_bar();
                                tmem_ld_wait();
#pragma unroll
                                for (int j = 0; j < 32; ++j) stage[j * S::BM + row] = __uint_as_float(r[j]);
                                fence_proxy_async();
                                epilogue_bar();
                                if (q == 0 && lane == 0) {
                                    bulk_copy_s2g(slot_ws + c * kChunkFloats, stage, kChunkBytes);
                                    bulk_commit_group();
                                }
                            }
                        }
                        release_tmem();
                        if (q == 0 && lane == 0) {
                            bulk_wait_group<0>();
                            fence_proxy_async_global();
                            trace_stamp(args, it - 1, 4);
                            st_release_gpu(args.flags + (u.slot * kCtaGroup + pair_rank), epoch);
                        }
                        __syncwarp();
                    } else {
                        const int ps = tile_idx + rest;  // slot of slice 1
                        const float* peer_ws = args.workspace + static_cast<long>(ps * kCtaGroup + pair_rank) * S::WS_FLOATS;
                        const int m_cta = tm * S::BM_TILE + static_cast<int>(pair_rank) * S::BM;
                        if (q == 0 && lane == 0) {
                            while (ld_acquire_gpu(args.flags + (ps * kCtaGroup + pair_rank)) < epoch) __nanosleep(64);
                            fence_proxy_async_global();
                            trace_stamp(args, it - 1, 4);
                            bulk_wait_group_read<0>();  // earlier units' C stores have left the epi buffers
                            for (int c = 0; c < 2; ++c) {  // prefetch chunks 0, 1 into the epi buffers
                                mbar_arrive_expect_tx(&stage_bar[c], kChunkBytes);
                                bulk_copy_g2s(epi + c * kChunkFloats, peer_ws + c * kChunkFloats, kChunkBytes, &stage_bar[c]);
                            }
                        }
                        __syncwarp();
#pragma unroll 1
                        for (int c = 0; c < NCH; ++c) {
                            uint32_t r[32];
                            tmem_ld_32x32b_x32(tbase + c * 32, r);
                            const int b = c & 1;
                            mbar_wait(&stage_bar[b], static_cast<uint32_t>(c >> 1) & 1);
                            tmem_ld_wait();
                            const float* pp = epi + b * kChunkFloats + row;
                            float v[32];
#pragma unroll
                            for (int j = 0; j < 32; ++j) v[j] = pp[j * S::BM] + __uint_as_float(r[j]);
                            epilogue_bar();  // every thread has read epi[b]: refill it with chunk c + 2
                            if (q == 0 && lane == 0 && c + 2 < NCH) {
                                fence_proxy_async();
                                mbar_arrive_expect_tx(&stage_bar[b], kChunkBytes);
                                bulk_copy_g2s(epi + b * kChunkFloats, peer_ws + (c + 2) * kChunkFloats, kChunkBytes,
                                              &stage_bar[b]);
                            }
                            if (args.c_tma && !args.sk_head) {
                                float* dst = stage0 + c * kChunkFloats + row;
#pragma unroll
                                for (int j = 0; j < 32; ++j) dst[j * S::BM] = v[j];
                                fence_proxy_async();
                                epilogue_bar();
                                if (q == 0 && lane == 0) {
                                    tma_store_2d(&tmC, stage0 + c * kChunkFloats, m_cta, tn * BN + c * 32);
                                    bulk_commit_group();
                                }
                            } else {
                                store_row32_any(args, m, tn * BN + c * 32, v);
                            }
                        }
                        release_tmem();
                        if (q == 0 && lane == 0) trace_stamp(args, it - 1, 5);
                    }
                } else {
                    // K-slice tail unit. Symmetric fixup: main slice s owns 32-column
                    // chunks [c_lo, c_hi) and keeps those in smem (a main slice is the
                    // cluster's last unit: its operand ring is idle); every other chunk
                    // is published in its workspace slot. A remainder slice owns no
                    // columns and publishes all of them (through the epi buffers while
                    // its ring is still in use by a next remainder unit). Each owner then sums its range over all
                    // sources in K order (slices 0..S-1, then the remainder) and
                    // stores it: deterministic, and the S fixups run in parallel.
                    const int nslc = args.sk_slices, s = u.slice;
                    const bool remainder = s == nslc;
                    const int nsrc = nslc + (args.sk_w > 0 ? 1 : 0);
                    const int rest = args.tiles_m * args.tiles_n - args.sk_tile_begin;
                    const int tile_idx = u.tile - args.sk_tile_begin;
                    constexpr int NCH = BN / 32;
                    const int c_lo = remainder ? 0 : NCH * s / nslc;
                    const int c_hi = remainder ? 0 : NCH * (s + 1) / nslc;
                    const int nown = c_hi - c_lo;
                    constexpr uint32_t kChunkFloats = 32 * S::BM;
                    constexpr uint32_t kChunkBytes = kChunkFloats * 4;
                    // main slice: the ring holds [own chunks][published chunks], the
                    // latter reused for the peers' partials once they are stored
                    float* own = reinterpret_cast<float*>(ring);  // [nown][32][128]
                    float* peer = own + nown * kChunkFloats;       // [nsrc-1][nown][32][128]
                    float* slot_ws = args.workspace + static_cast<long>(u.slot * kCtaGroup + pair_rank) * S::WS_FLOATS;
                    // publish: every chunk that is not mine goes to the workspace slot
                    // as one 16 KB bulk copy out of shared memory. A remainder unit
                    // that is its cluster's last unit drains through the idle ring too
                    // (all copies in flight at once instead of two epi buffers)
                    if (!remainder || (last_unit && args.ring_drain)) {
                        auto slot = [&](int c) {
                            const bool mine = c >= c_lo && c < c_hi;
                            return mine ? own + (c - c_lo) * kChunkFloats
                                        : peer + (c < c_lo ? c : c - nown) * kChunkFloats;
                        };
                        drain_pairs(tbase, NCH, slot, [&](int c) {
                            if (c < c_lo || c >= c_hi)
                                bulk_copy_s2g(slot_ws + c * kChunkFloats, slot(c), kChunkBytes);
                        });
                    } else {
                        // the ring is busy with the next unit: double-buffered epi staging
#pragma unroll 1
                        for (int c = 0; c < NCH; ++c) {
                            uint32_t r[32];
                            tmem_ld_32x32b_x32(tbase + c * 32, r);
                            float* stage = epi + (epi_chunk++ & 1) * kChunkFloats;
                            if (q == 0 && lane == 0) bulk_wait_group_read<1>();
                            epilogue_bar();
                            tmem_ld_wait();
#pragma unroll
                            for (int j = 0; j < 32; ++j) stage[j * S::BM + row] = __uint_as_float(r[j]);
                            fence_proxy_async();
                            epilogue_bar();
                            if (q == 0 && lane == 0) {
                                bulk_copy_s2g(slot_ws + c * kChunkFloats, stage, kChunkBytes);
                                bulk_commit_group();
                            }
                        }
                    }
                    release_tmem();
                    if (q == 0 && lane == 0) {
                        trace_stamp(args, it - 1, 6);
                        bulk_wait_group<0>();        // my partial chunks are in global memory
                        fence_proxy_async_global();  // async-proxy writes before the release
                        trace_stamp(args, it - 1, 4);
                        st_release_gpu(args.flags + (u.slot * kCtaGroup + pair_rank), epoch);
                        if (nown > 0) {
                            // fetch each source's chunks of my range as soon as its flag is
                            // set (arrival order), each completing on its own barrier
                            uint32_t pending = ((1u << nsrc) - 1u) & ~(1u << s);
                            while (pending) {
                                for (uint32_t rest_mask = pending; rest_mask; rest_mask &= rest_mask - 1) {
                                    const int j = __ffs(rest_mask) - 1;
                                    const int ps = j < nslc ? tile_idx + j * rest  // slot of source j
                                                            : remainder_slot(args, rest, nclusters, tile_idx);
                                    if (ld_acquire_gpu(args.flags + (ps * kCtaGroup + pair_rank)) < epoch) continue;
                                    fence_proxy_async_global();
                                    mbar_arrive_expect_tx(&src_bar[j], nown * kChunkBytes);
                                    bulk_copy_g2s(peer + (j < s ? j : j - 1) * nown * kChunkFloats,
                                                  args.workspace +
                                                      static_cast<long>(ps * kCtaGroup + pair_rank) * S::WS_FLOATS +
                                                      static_cast<long>(c_lo) * kChunkFloats,
                                                  nown * kChunkBytes, &src_bar[j]);
                                    pending &= ~(1u << j);
                                }
                                if (pending) __nanosleep(32);
                            }
                        }
                    }
                    __syncwarp();
                    if (nown > 0) {
                        // sum in slice order (deterministic) as the sources land; with a TMA
                        // C the chunk is stored as soon as it is summed
                        const int m_cta = tm * S::BM_TILE + static_cast<int>(pair_rank) * S::BM;
#pragma unroll 1
                        for (int c = c_lo; c < c_hi; ++c) {
                            float v[32];
#pragma unroll 1
                            for (int j = 0; j < nsrc; ++j) {
                                if (j != s && c == c_lo) mbar_wait(&src_bar[j], 0);
                                const float* src = (j == s ? own : peer + (j < s ? j : j - 1) * nown * kChunkFloats) +
                                                   (c - c_lo) * kChunkFloats + row;
                                if (j == 0) {
#pragma unroll
                                    for (int x = 0; x < 32; ++x) v[x] = src[x * S::BM];
                                } else {
#pragma unroll
                                    for (int x = 0; x < 32; ++x) v[x] += src[x * S::BM];
                                }
                            }
                            if (c == c_lo && q == 0 && lane == 0) trace_stamp(args, it - 1, 5);
                            if (args.c_tma) {  // sum in place, TMA-store the chunk
                                float* dst = own + (c - c_lo) * kChunkFloats + row;
#pragma unroll
                                for (int x = 0; x < 32; ++x) dst[x * S::BM] = v[x];
                                fence_proxy_async();
                                epilogue_bar();
                                if (q == 0 && lane == 0) {
                                    tma_store_2d(&tmC, own + (c - c_lo) * kChunkFloats, m_cta, tn * BN + c * 32);
                                    bulk_commit_group();
                                }
                            } else {
                                store_row32_any(args, m, tn * BN + c * 32, v);
                            }
                        }
                    }
                }
                if (q == 0 && lane == 0) trace_stamp(args, it - 1, 3);
            } else {
                // The producer only refills the ring after rempty completes, and
                // tfull implies this tile's operands are consumed: the ring is free.
                float* my_row = red + row * S::RED_LD;
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    uint32_t r[32];
                    tmem_ld_32x32b_x32(tbase + c * 32, r);
                    tmem_ld_wait();
                    float4* dst = reinterpret_cast<float4*>(my_row + c * 32);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        dst[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                             __uint_as_float(r[4 * j + 2]),
                                             __uint_as_float(r[4 * j + 3]));
                }
                tc_fence_before();
                fence_acq_rel_cluster();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (kCtaGroup == 1) mbar_arrive(&tempty_bar[buf]);
                    else mbar_arrive_cluster(&tempty_bar[buf], crank - pair_rank);
#pragma unroll 1
                    for (int r = 0; r < kSplitK; ++r)
                        mbar_arrive_cluster(rfull_bar, static_cast<uint32_t>(r * kCtaGroup) + pair_rank);
                }
                mbar_wait_cluster(rfull_bar, tile_use & 1);
                // reduce the column slice owned by this split rank, rank order 0..S-1
                constexpr int kCols = BN / kSplitK;
                const int c0 = static_cast<int>(split_rank) * kCols;
                const uint32_t my_addr = smem_u32(my_row + c0);
#pragma unroll 1
                for (int cc = 0; cc < kCols; cc += 32) {
                    float v[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = 0.0f;
#pragma unroll 1
                    for (int r = 0; r < kSplitK; ++r) {
                        const uint32_t peer = static_cast<uint32_t>(r * kCtaGroup) + pair_rank;
                        const uint32_t base = map_shared_rank(my_addr + cc * 4, peer);
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            float4 x = ld_dsmem_f4(base + j * 16);
                            v[4 * j + 0] += x.x;
                            v[4 * j + 1] += x.y;
                            v[4 * j + 2] += x.z;
                            v[4 * j + 3] += x.w;
                        }
                    }
                    store_row32_any(args, m, tn * BN + c0 + cc, v);
                }
                fence_proxy_async();
                fence_acq_rel_cluster();
                __syncwarp();
                if (lane == 0)
                    for (int r = 0; r < kSplitK; ++r)
                        mbar_arrive_cluster(rempty_bar, static_cast<uint32_t>(r * kCtaGroup) + pair_rank);
                __syncwarp();
                if (q == 0 && lane == 0) trace_stamp(args, it - 1, 3);
            }
            u = nxt;
            have = have_next;
        }
        if (q == 0 && lane == 0) bulk_wait_group<0>();  // TMA stores of C complete
        if (q == 0 && lane == 0 && args.trace) args.trace[(blockIdx.x * 16 + 3) * 16 + 7] = global_timer_ns();
        __syncwarp();
    }

    tc_fence_before();
    if constexpr (kClusterSize > 1) cluster_sync(); else __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<kCtaGroup>(tmem_base, S::TMEM_COLS);
        if (lane == 0 && args.trace) args.trace[(blockIdx.x * 16 + 4) * 16 + 7] = global_timer_ns();
    }
}

template <int kCtaGroup, int BN, int kSplitK, int kSlabs, int kNHalves, int kMcast = 1, int kKB = 1>
__global__ void __launch_bounds__(256, 1)
    fi_sm100_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmC,
                  const __grid_constant__ CUtensorMap tmC2,
                  const __grid_constant__ GemmArgs args) {
    fi_sm100_gemm_body<kCtaGroup, BN, kSplitK, kSlabs, kNHalves, kMcast, kKB>(tmA, tmB, tmB2, tmC, tmC2, args);
}

}  // namespace fireiron::sm100
