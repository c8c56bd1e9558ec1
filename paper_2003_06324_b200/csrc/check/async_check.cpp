// CPU checker for the asynchronous protocol of the tcgen05 GEMM family
// (include/fireiron/async_check.hpp). Every role below restates one branch of
// sm100/gemm_kernel.cuh with its synchronisation and its memory footprint;
// the unit sequence and the launch schedule are the kernel's own
// (sm100/schedule.hpp: UnitIter, plan_schedule), so the checker exercises
// exactly what the GPU runs.
//
// Model. Agents per simulated CTA: P, P2, P3 (the three TMA producer warps, ring
// stages s % 3 = 0, 1, 2), M (MMA issuer),
// E (the four epilogue warps, which move in lockstep through named
// barriers), and the asynchronous engines they drive: TMA (tensor loads, one per producer), MMA
// (tcgen05.mma, completion via tcgen05.commit), BR/BW (bulk and TMA stores:
// their shared-memory reads and global writes complete separately,
// cp.async.bulk.wait_group.read vs wait_group), G2S (bulk loads completing on
// an mbarrier). Happens-before is tracked with vector clocks; an mbarrier
// phase carries the join of its arrivals' clocks to every waiter of that
// phase, an epoch flag carries its releaser's clock to acquirers. A CTA pair
// is simulated through its rank-0 CTA (both halves follow the same schedule);
// cluster split-K simulates each split rank.
#include <coroutine>
#include <cstdint>
#include <deque>
#include <exception>
#include <functional>
#include <memory>
#include <sstream>
#include <unordered_map>
#include <vector>

#include "../sm100/schedule.hpp"
#include "fireiron/async_check.hpp"
#include "fireiron/backend.hpp"
#include "fireiron/error.hpp"

namespace fireiron {

std::string AsyncReport::to_string() const {
    std::ostringstream os;
    os << "async protocol check: " << (ok() ? "ok" : "VIOLATIONS") << "\n"
       << "  schedule: " << clusters << " clusters x " << cluster_size << " CTAs, " << tiles << " tiles, " << units
       << " units, mode " << mode << ", slices " << slices << (remainder ? " + remainder" : "")
       << (pull ? (head ? " (pull fixup, first)" : " (pull fixup)") : "") << ", split-k "
       << split_k << ", stages " << stages
       << (gated_chunks ? ", B gated in " + std::to_string(gated_chunks) + " copy-engine chunks" : std::string()) << "\n"
       << "  events " << events << ", races " << races << ", capacity " << capacity_errors << ", coverage "
       << coverage_errors << ", deadlocks " << deadlocks << "\n";
    for (const auto& r : records)
        os << "  " << r.kind << " " << r.resource << "[" << r.index << "] cluster " << r.cluster << ": " << r.first
           << (r.second.empty() ? "" : " vs " + r.second) << "\n";
    return os.str();
}

namespace {

using namespace sm100;

// ------------------------------------------------------------------ coroutines
struct Task {
    struct promise_type {
        std::function<bool()> ready;  // predicate the task waits on while suspended
        std::exception_ptr error;
        Task get_return_object() { return Task{std::coroutine_handle<promise_type>::from_promise(*this)}; }
        std::suspend_always initial_suspend() noexcept { return {}; }
        std::suspend_always final_suspend() noexcept { return {}; }
        void return_void() {}
        void unhandled_exception() { error = std::current_exception(); }
    };
    std::coroutine_handle<promise_type> h;
};

struct WaitUntil {
    std::function<bool()> pred;
    bool await_ready() { return pred(); }
    void await_suspend(std::coroutine_handle<Task::promise_type> h) { h.promise().ready = pred; }
    void await_resume() {}
};

// ------------------------------------------------------------------ clocks, cells, barriers
using Clock = std::vector<uint32_t>;

void join(Clock& dst, const Clock& src) {
    for (size_t i = 0; i < dst.size(); ++i)
        if (src[i] > dst[i]) dst[i] = src[i];
}

enum Space : uint64_t { kRing = 1, kEpi, kTmem, kWs, kC, kB };
const char* space_name(uint64_t s) {
    switch (s) {
        case kRing: return "ring";
        case kEpi: return "epi";
        case kTmem: return "tmem";
        case kWs: return "workspace";
        case kC: return "C";
        case kB: return "B chunk";
    }
    return "?";
}
uint64_t cell_key(uint64_t space, uint64_t owner, uint64_t index) { return (space << 56) | (owner << 32) | index; }

struct Cell {
    int w_agent = -1;
    uint32_t w_time = 0;
    std::vector<std::pair<int, uint32_t>> reads;  // since the last write, max time per agent
};

struct Barrier {
    int count = 1;      // arrivals per phase
    int arrivals = 0;
    long tx = 0;        // outstanding transaction bytes
    uint64_t completed = 0;
    Clock pending, last[2];
};

struct Flag {
    unsigned value = 0;
    Clock clock;
};

// kP / kTMA, kP2 / kTMA2, kP3 / kTMA3: the three producer warps (ring stages
// s % 3 = 0, 1, 2) and their loads
enum Role { kP = 0, kM, kE, kTMA, kMMA, kBR, kBW, kG2S, kP2, kTMA2, kP3, kTMA3, kRoles };
const char* role_name(int r) {
    static const char* n[] = {"producer", "mma-issuer", "epilogue",   "tma-load",   "tcgen05.mma", "bulk-read",
                              "bulk-write", "bulk-load", "producer-2", "tma-load-2", "producer-3",  "tma-load-3"};
    return n[r];
}

template <int kCtaGroup, int BN, int kSplitK, int kSlabs = 1, int kNHalves = 1, int kMcast = 1>
class Checker {
    // simulated CTAs per cluster: split-K ranks, or the two pairs of a multicast cluster
    static constexpr int kRanks = kSplitK * kMcast;
    using S = GemmShape<kCtaGroup, BN, kSplitK, kSlabs, kNHalves>;
    static constexpr int kStages = S::kStages;
    static constexpr int NCH = BN / 32;
    static constexpr int NCH_ALL = NCH * kSlabs * kNHalves;  // 32-column chunks of a tile's CTA rows, all accumulators
    static constexpr int kChunkBytes = 32 * S::BM * 4;
    static constexpr int kGran = 1024;  // shared-memory cell granularity (bytes)
    static constexpr int kProducers = kSlabs * kNHalves > 1 ? 1 : 3;  // as gemm_kernel.cuh

public:
    Checker(const GemmArgs& args, int clusters, long slots, const AsyncCheckOptions& o, AsyncReport& rep)
        : a_(args), ncl_(clusters), slots_(slots), opt_(o), rep_(rep) {
        nctas_ = ncl_ * kRanks;
        nagents_ = nctas_ * kRoles + 1;  // + the copy engine that lands gated B chunks
        ce_ = nagents_ - 1;
        vc_.assign(static_cast<size_t>(nagents_), Clock(static_cast<size_t>(nagents_), 0));
        ctas_.resize(static_cast<size_t>(nctas_));
        for (auto& c : ctas_) {
            c.full.resize(kStages);
            c.empty.resize(kStages);
            for (auto* b : {&c.tfull[0], &c.tfull[1], &c.tempty[0], &c.tempty[1], &c.rfull, &c.rempty, &c.stage,
                            &c.pstage[0], &c.pstage[1]})
                init_bar(*b, 1);
            for (auto& b : c.src) init_bar(b, 1);
            for (auto& b : c.full) init_bar(b, 1);
            for (auto& b : c.empty)  // a release from every pair reading the slot
                init_bar(b, opt_.mutation == kMutMcastSingleRelease ? 1 : kMcast);
            init_bar(c.tempty[0], 1);
            init_bar(c.tempty[1], 1);
            init_bar(c.rfull, kSplitK);
            init_bar(c.rempty, kSplitK);
        }
        flags_.resize(static_cast<size_t>(slots_ > 0 ? slots_ : 1));
        nst_ = (a_.stages > 0 && a_.stages < kStages) ? a_.stages : kStages;
    }

    void run() {
        if (opt_.gated_chunks > 0) {  // the copy engine lands chunk j, then its stream writes flag j
            b_flags_.resize(static_cast<size_t>(opt_.gated_chunks));
            for (int i = 0; i < opt_.gated_chunks; ++i) {
                const int j = (opt_.gated_first + i) % opt_.gated_chunks;
                access(ce_, kB, 0, static_cast<uint64_t>(j), true);
                ++vc_[static_cast<size_t>(ce_)][static_cast<size_t>(ce_)];
                b_flags_[static_cast<size_t>(j)].value = a_.epoch;
                b_flags_[static_cast<size_t>(j)].clock = vc_[static_cast<size_t>(ce_)];
            }
        }
        std::vector<Task> tasks;
        for (int c = 0; c < ncl_; ++c)
            for (int r = 0; r < kRanks; ++r) {
                for (int pw = 0; pw < kProducers; ++pw) tasks.push_back(producer(c, r, pw));
                tasks.push_back(mma(c, r));
                tasks.push_back(epilogue(c, r));
            }
        // round-robin over runnable tasks until all finish or none can move
        std::vector<bool> done(tasks.size(), false);
        size_t left = tasks.size();
        while (left > 0) {
            bool progress = false;
            for (size_t i = 0; i < tasks.size(); ++i) {
                if (done[i]) continue;
                auto& p = tasks[i].h.promise();
                if (p.ready && !p.ready()) continue;
                p.ready = nullptr;
                tasks[i].h.resume();
                if (p.error) std::rethrow_exception(p.error);
                progress = true;
                if (tasks[i].h.done()) {
                    done[i] = true;
                    --left;
                }
            }
            if (!progress) {
                ++rep_.deadlocks;
                record("deadlock", "barrier", static_cast<long>(left), "tasks blocked with no pending arrival", "",
                       -1);
                break;
            }
        }
        for (auto& t : tasks) t.h.destroy();
        // coverage: every 32-column chunk of every tile's CTA rows stored exactly once
        const long tiles = static_cast<long>(a_.tiles_m) * a_.tiles_n * kMcast;  // per pair of a multicast unit
        for (long t = 0; t < tiles; ++t)
            for (int ch = 0; ch < NCH_ALL; ++ch) {
                auto it = stores_.find(t * NCH_ALL + ch);
                const int n = it == stores_.end() ? 0 : it->second;
                if (n != 1) {
                    ++rep_.coverage_errors;
                    record("coverage", "C", t * NCH_ALL + ch, "tile " + std::to_string(t) + " chunk " +
                           std::to_string(ch) + " stored " + std::to_string(n) + " times", "", -1);
                }
            }
    }

private:
    struct Cta {
        std::vector<Barrier> full, empty;
        Barrier tfull[2], tempty[2], rfull, rempty, stage, pstage[2], src[8];
        std::deque<std::pair<Clock, Clock>> groups;  // committed bulk groups: (read clock, write clock)
        long committed = 0, waited_r = 0, waited_w = 0;
    };

    const GemmArgs a_;
    const int ncl_;
    const long slots_;
    const AsyncCheckOptions opt_;
    AsyncReport& rep_;
    int nctas_ = 0, nagents_ = 0, nst_ = 0;
    std::vector<Clock> vc_;
    std::vector<Cta> ctas_;
    std::vector<Flag> flags_;
    std::unordered_map<uint64_t, Cell> cells_;
    std::unordered_map<long, int> stores_;  // (tile*NCH_ALL + chunk) -> times stored

    int agent(int cta, int role) const { return cta * kRoles + role; }
    int ce_ = 0;
    std::vector<Flag> b_flags_;  // gated B: ready flag of each column chunk
    int cta_of(int c, int r) const { return c * kRanks + r; }

    void init_bar(Barrier& b, int count) {
        b.count = count;
        b.pending.assign(static_cast<size_t>(nagents_), 0);
        b.last[0].assign(static_cast<size_t>(nagents_), 0);
        b.last[1].assign(static_cast<size_t>(nagents_), 0);
    }

    void record(const char* kind, const char* res, long index, std::string first, std::string second, int cluster) {
        if (rep_.records.size() < 256) rep_.records.push_back({kind, res, index, std::move(first), std::move(second), cluster});
    }
    std::string who(int ag) const {
        if (ag == ce_) return "copy-engine";
        return std::string(role_name(ag % kRoles)) + "@cta" + std::to_string(ag / kRoles);
    }

    // ---- memory accesses
    void access(int ag, uint64_t space, uint64_t owner, uint64_t index, bool write) {
        ++rep_.events;
        Clock& v = vc_[static_cast<size_t>(ag)];
        ++v[static_cast<size_t>(ag)];
        Cell& c = cells_[cell_key(space, owner, index)];
        auto ordered = [&](int other, uint32_t t) { return other == ag || v[static_cast<size_t>(other)] >= t; };
        bool race = false;
        int other = -1;
        if (c.w_agent >= 0 && !ordered(c.w_agent, c.w_time)) {
            race = true;
            other = c.w_agent;
        }
        if (write && !race)
            for (auto& [ra, rt] : c.reads)
                if (!ordered(ra, rt)) {
                    race = true;
                    other = ra;
                    break;
                }
        if (race) {
            ++rep_.races;
            record("race", space_name(space), static_cast<long>(index),
                   who(other) + (c.w_agent == other ? " (write)" : " (read)"),
                   who(ag) + (write ? " (write)" : " (read)"), static_cast<int>(owner));
        }
        if (write) {
            c.w_agent = ag;
            c.w_time = v[static_cast<size_t>(ag)];
            c.reads.clear();
        } else {
            bool found = false;
            for (auto& [ra, rt] : c.reads)
                if (ra == ag) {
                    rt = v[static_cast<size_t>(ag)];
                    found = true;
                }
            if (!found) c.reads.push_back({ag, v[static_cast<size_t>(ag)]});
        }
    }
    // shared-memory byte range [off, off + bytes) of the CTA's operand ring / epilogue buffers
    void smem(int ag, int cta, uint64_t space, long off, long bytes, bool write) {
        const long cap = space == kRing ? S::RING_BYTES : S::EPI_BYTES;
        if (off < 0 || off + bytes > cap) {
            ++rep_.capacity_errors;
            record("capacity", space_name(space), off, "bytes [" + std::to_string(off) + ", " +
                   std::to_string(off + bytes) + ") beyond " + std::to_string(cap), who(ag), cta);
            return;
        }
        for (long x = off / kGran; x < (off + bytes + kGran - 1) / kGran; ++x) access(ag, space, cta, x, write);
    }
    void tmem(int ag, int cta, int buf, int col0, int cols, bool write) {
        if (col0 < 0 || col0 + cols > S::ACC_COLS || buf >= S::kAccBufs) {
            ++rep_.capacity_errors;
            record("capacity", "tmem", col0, "columns beyond the accumulator", who(ag), cta);
            return;
        }
        for (int ch = col0 / 32; ch < (col0 + cols) / 32; ++ch) access(ag, kTmem, cta, buf * NCH_ALL + ch, write);
    }
    void workspace(int ag, long slot, int ch0, int nch, bool write) {
        if (slot < 0 || slot >= slots_) {
            ++rep_.capacity_errors;
            record("capacity", "workspace", slot, "slot beyond the " + std::to_string(slots_) + " allocated", who(ag), -1);
            return;
        }
        for (int ch = ch0; ch < ch0 + nch; ++ch) access(ag, kWs, 0, static_cast<uint64_t>(slot) * NCH + ch, write);
    }
    void store_c(int ag, int tile, int ch) {
        access(ag, kC, 0, static_cast<uint64_t>(tile) * NCH_ALL + ch, true);
        ++stores_[static_cast<long>(tile) * NCH_ALL + ch];
    }

    // ---- synchronisation
    void arrive(Barrier& b, const Clock& v) {
        join(b.pending, v);
        if (++b.arrivals >= b.count && b.tx == 0) complete(b);
    }
    void complete(Barrier& b) {
        b.last[b.completed & 1] = b.pending;
        ++b.completed;
        b.arrivals = 0;
        std::fill(b.pending.begin(), b.pending.end(), 0);
    }
    void expect_tx(Barrier& b, long bytes) { b.tx += bytes; }
    // phase = the barrier phase the issuer meant to credit. Bytes may arrive before
    // that phase's expect_tx (the tx-count goes transiently negative, as on the
    // hardware), but bytes for a phase that already completed spill into the next
    // one: an expect_tx that under-counts its loads.
    void complete_tx(Barrier& b, long bytes, const Clock& v, uint64_t phase = ~0ull) {
        if (phase != ~0ull && phase < b.completed) {
            ++rep_.deadlocks;
            record("tx-mismatch", "barrier", static_cast<long>(bytes), "transaction bytes after their phase completed",
                   "", -1);
        }
        join(b.pending, v);
        b.tx -= bytes;
        if (b.arrivals >= b.count && b.tx == 0) complete(b);
    }
    // try_wait.parity(p) succeeds once a phase of parity p completed after the
    // last one of parity !p, i.e. (completed & 1) != p; it acquires that phase
    static bool passed(const Barrier& b, uint32_t parity) { return (b.completed & 1) != parity; }
    void acquire(int ag, const Barrier& b, uint32_t parity) {
        (void)parity;  // a passing wait(p) always observes the last completed phase (parity p)
        if (b.completed == 0) return;  // the initial "previous phase": nothing to acquire
        join(vc_[static_cast<size_t>(ag)], b.last[(b.completed - 1) & 1]);
    }
    WaitUntil wait(Barrier& b, uint32_t parity) {
        return WaitUntil{[&b, parity] { return passed(b, parity); }};
    }

    // async engine op: issued by `issuer`, its accesses ordered after the issue point
    void issue(int eng, int issuer) {
        join(vc_[static_cast<size_t>(eng)], vc_[static_cast<size_t>(issuer)]);
        ++vc_[static_cast<size_t>(eng)][static_cast<size_t>(eng)];
    }
    // bulk groups of the epilogue: the group's read and write clocks
    void commit_group(int cta) {
        Cta& C = ctas_[static_cast<size_t>(cta)];
        C.groups.push_back({vc_[static_cast<size_t>(agent(cta, kBR))], vc_[static_cast<size_t>(agent(cta, kBW))]});
        ++C.committed;
    }
    // cp.async.bulk.wait_group[.read] N: all but the N most recent groups done
    void wait_groups(int cta, long n, bool writes) {
        Cta& C = ctas_[static_cast<size_t>(cta)];
        const long upto = C.committed - n;  // groups [0, upto) complete
        long& w = writes ? C.waited_w : C.waited_r;
        Clock& e = vc_[static_cast<size_t>(agent(cta, kE))];
        for (long g = 0; g < upto; ++g) {
            const auto& gr = C.groups[static_cast<size_t>(g)];
            join(e, gr.first);
            if (writes) join(e, gr.second);
        }
        if (upto > w) w = upto;
    }

    // ------------------------------------------------------------------ roles
    // warps 0, 3, 2: gemm_kernel.cuh "TMA producers" -- producer pw fills the
    // ring stages s with s % 3 == pw; all walk the same unit and stage sequence
    Task producer(int cl, int rank, int pw) {
        const int cta = cta_of(cl, rank), P = agent(cta, pw == 0 ? kP : pw == 1 ? kP2 : kP3),
                  T = agent(cta, pw == 0 ? kTMA : pw == 1 ? kTMA2 : kTMA3);
        Cta& C = ctas_[static_cast<size_t>(cta)];
        int s = 0;
        uint32_t ph = 0;
        uint64_t lap = 0;  // ring wraps so far: the full-barrier phase this stage's loads credit
        int it = 0;
        UnitIter<BN> units(a_, cl, ncl_);
        Unit u;
        while (units.next(u)) {
            if constexpr (kSplitK > 1) {
                co_await wait(C.rempty, (static_cast<uint32_t>(it) & 1) ^ 1);
                acquire(P, C.rempty, (static_cast<uint32_t>(it) & 1) ^ 1);
            }
            ++it;
            const int b_rows = u.width / kCtaGroup;
            // the kernel's expect_tx (per CTA of the pair) vs the bytes its loads deliver
            const long expect = opt_.mutation == kMutTxUndercount
                                    ? S::A_BYTES + static_cast<long>(b_rows) * S::BK * 2  // the first N-half kernel's bug
                                    : S::stage_tx_bytes(b_rows) / kCtaGroup;
            const long a_bytes = S::A_BYTES, b_bytes = static_cast<long>(b_rows) * S::BK * 2 * kNHalves;
            int chunk = -1;  // gated B: wait_b_chunk (ld.acquire of the chunk's ready flag) before the loads
            if (!b_flags_.empty()) {
                int tm, tn;
                tile_coords(a_, u.tile, tm, tn);
                chunk = tn / a_.b_chunk_tiles;
                Flag& f = b_flags_[static_cast<size_t>(chunk)];
                co_await WaitUntil{[&f, this] { return f.value >= a_.epoch; }};
                if (opt_.mutation != kMutGateSkipAcquire) join(vc_[static_cast<size_t>(P)], f.clock);
            }
            for (int kb = u.k0; kb < u.k1; ++kb) {
                if (s % kProducers != pw) {  // another producer's stage
                    if (++s == nst_) {
                        s = 0;
                        ph ^= 1;
                        ++lap;
                    }
                    continue;
                }
                if (opt_.mutation != kMutSkipEmptyWait) {
                    co_await wait(C.empty[static_cast<size_t>(s)], ph ^ 1);
                    acquire(P, C.empty[static_cast<size_t>(s)], ph ^ 1);
                }
                ++vc_[static_cast<size_t>(P)][static_cast<size_t>(P)];
                Barrier& full = C.full[static_cast<size_t>(s)];
                expect_tx(full, expect);
                arrive(full, vc_[static_cast<size_t>(P)]);
                issue(T, P);
                const long st = static_cast<long>(s) * S::STAGE_BYTES;
                if constexpr (kMcast > 1) {
                    // my 64-row half of A, multicast to me and my rank-twin in the other pair
                    for (int r2 = 0; r2 < kMcast; ++r2) {
                        const int dst = cta_of(cl, r2);
                        smem(T, dst, kRing, st + static_cast<long>(rank) * (a_bytes / 2), a_bytes / 2, true);
                        complete_tx(ctas_[static_cast<size_t>(dst)].full[static_cast<size_t>(s)], a_bytes / 2,
                                    vc_[static_cast<size_t>(T)], lap);
                    }
                } else {
                    smem(T, cta, kRing, st, a_bytes, true);  // A slab(s)
                    complete_tx(full, a_bytes, vc_[static_cast<size_t>(T)], lap);
                }
                if (chunk >= 0) access(T, kB, 0, static_cast<uint64_t>(chunk), false);  // TMA reads the landed chunk
                smem(T, cta, kRing, st + S::A_BYTES, b_bytes, true);  // B half (halves)
                complete_tx(full, b_bytes, vc_[static_cast<size_t>(T)], lap);
                if (++s == nst_) {
                    s = 0;
                    ph ^= 1;
                    ++lap;
                }
            }
        }
    }

    // warp 1: "MMA issuer"
    Task mma(int cl, int rank) {
        const int cta = cta_of(cl, rank), M = agent(cta, kM), X = agent(cta, kMMA);
        Cta& C = ctas_[static_cast<size_t>(cta)];
        int s = 0;
        uint32_t ph = 0;
        int it = 0;
        UnitIter<BN> units(a_, cl, ncl_);
        Unit u;
        while (units.next(u)) {
            const int buf = S::kAccBufs == 2 ? (it & 1) : 0;
            const uint32_t use = static_cast<uint32_t>(S::kAccBufs == 2 ? (it >> 1) : it);
            ++it;
            if (opt_.mutation != kMutSkipTmemEmptyWait) {
                co_await wait(C.tempty[buf], (use & 1) ^ 1);
                acquire(M, C.tempty[buf], (use & 1) ^ 1);
            }
            const long bytes = S::A_BYTES + static_cast<long>(u.width / kCtaGroup) * S::BK * 2 * kNHalves;
            for (int kb = u.k0; kb < u.k1; ++kb) {
                co_await wait(C.full[static_cast<size_t>(s)], ph);
                acquire(M, C.full[static_cast<size_t>(s)], ph);
                ++vc_[static_cast<size_t>(M)][static_cast<size_t>(M)];
                issue(X, M);
                smem(X, cta, kRing, static_cast<long>(s) * S::STAGE_BYTES, bytes, false);
                tmem(X, cta, buf, 0, u.width * kSlabs * kNHalves, true);
                if constexpr (kMcast > 1) {  // commit multicast to every CTA of the cluster
                    for (int r2 = 0; r2 < kMcast; ++r2)
                        arrive(ctas_[static_cast<size_t>(cta_of(cl, r2))].empty[static_cast<size_t>(s)],
                               vc_[static_cast<size_t>(X)]);
                } else {
                    arrive(C.empty[static_cast<size_t>(s)], vc_[static_cast<size_t>(X)]);  // tcgen05.commit
                }
                if (++s == nst_) {
                    s = 0;
                    ph ^= 1;
                }
            }
            arrive(C.tfull[buf], vc_[static_cast<size_t>(X)]);
        }
    }

    // warps 4..7: "epilogue"
    Task epilogue(int cl, int rank) {
        const int cta = cta_of(cl, rank), E = agent(cta, kE), BR = agent(cta, kBR), BW = agent(cta, kBW),
                  G = agent(cta, kG2S);
        Cta& C = ctas_[static_cast<size_t>(cta)];
        Clock& ve = vc_[static_cast<size_t>(E)];
        const int kb = a_.k_blocks;
        int it = 0;
        uint32_t epi_chunk = 0;
        UnitIter<BN> units(a_, cl, ncl_);
        Unit u, nxt;
        bool have = units.next(u);
        auto tick = [&] { ++ve[static_cast<size_t>(E)]; };
        // bulk / TMA store of one 16 KB chunk from shared memory
        auto bulk_store = [&](uint64_t space, long off, auto&& write_global) {
            issue(BR, E);
            smem(BR, cta, space, off, kChunkBytes, false);
            issue(BW, E);
            write_global(BW);
        };
        while (have) {
            const bool have_next = units.next(nxt);
            const bool last_unit = !have_next || opt_.mutation == kMutRingDrainEveryUnit;
            const int buf = S::kAccBufs == 2 ? (it & 1) : 0;
            const uint32_t use = static_cast<uint32_t>(S::kAccBufs == 2 ? (it >> 1) : it);
            const uint32_t tile_use = static_cast<uint32_t>(it);
            ++it;
            co_await wait(C.tfull[buf], use & 1);
            acquire(E, C.tfull[buf], use & 1);
            const int tile = u.tile * kMcast + (kMcast > 1 ? rank : 0);  // a multicast unit = two pair tiles
            const int ch_off = u.n_off / 32;
            const int nchu = u.width / 32, nch_all = nchu * kSlabs * kNHalves;
            auto cchunk = [&](int c) { return (c / nchu) * NCH + ch_off + c % nchu; };  // C chunk id of TMEM chunk c
            auto release_tmem = [&] {
                tick();
                arrive(C.tempty[buf], ve);
            };
            if constexpr (kSplitK == 1) {
                const bool whole = u.k0 == 0 && u.k1 == kb;
                if (whole && a_.c_tma && last_unit && a_.ring_drain &&
                    static_cast<long>(nch_all) * kChunkBytes <= S::RING_BYTES) {
                    // ring-staged last unit: chunks at ring + c*16KB, TMA-stored pairwise
                    for (int c = 0; c < nch_all; ++c) {
                        tmem(E, cta, buf, c * 32, 32, false);
                        smem(E, cta, kRing, static_cast<long>(c) * kChunkBytes, kChunkBytes, true);
                        if (c & 1) {
                            for (int x = c - 1; x <= c; ++x)
                                bulk_store(kRing, static_cast<long>(x) * kChunkBytes,
                                           [&](int bw) { store_c(bw, tile, cchunk(x)); });
                            commit_group(cta);
                        }
                    }
                    release_tmem();
                } else if (whole && a_.c_tma) {
                    // chunk pairs staged in both epi buffers, one 64-column TMA store per pair
                    for (int c = 0; c < nch_all; ++c) {
                        tmem(E, cta, buf, c * 32, 32, false);
                        const long off = static_cast<long>(c & 1) * kChunkBytes;
                        if ((c & 1) == 0) wait_groups(cta, 0, false);  // bulk_wait_group_read<0> + epilogue_bar
                        smem(E, cta, kEpi, off, kChunkBytes, true);
                        if (c & 1) {
                            bulk_store(kEpi, 0, [&](int bw) { store_c(bw, tile, cchunk(c - 1)); });
                            bulk_store(kEpi, kChunkBytes, [&](int bw) { store_c(bw, tile, cchunk(c)); });
                            commit_group(cta);
                        }
                    }
                    wait_groups(cta, 0, false);  // the epi buffers are free for the next unit
                    release_tmem();
                } else if (whole) {
                    for (int c = 0; c < nch_all; ++c) {
                        tmem(E, cta, buf, c * 32, 32, false);
                        store_c(E, tile, cchunk(c));
                    }
                    release_tmem();
                } else if (a_.sk_pull) {
                    // 2-slice pull fixup
                    const int rest = a_.tiles_m * a_.tiles_n - a_.sk_tile_begin;
                    const int tile_idx = u.tile - a_.sk_tile_begin;
                    if (u.slice == 1) {
                        for (int c = 0; c < NCH; ++c) {
                            tmem(E, cta, buf, c * 32, 32, false);
                            if (a_.sk_head) {  // ring busy: double-buffered epi staging
                                const long off = static_cast<long>(epi_chunk++ & 1) * kChunkBytes;
                                wait_groups(cta, 1, false);
                                smem(E, cta, kEpi, off, kChunkBytes, true);
                                bulk_store(kEpi, off, [&](int bw) { workspace(bw, u.slot, c, 1, true); });
                                commit_group(cta);
                                continue;
                            }
                            smem(E, cta, kRing, static_cast<long>(c) * kChunkBytes, kChunkBytes, true);
                            if (c & 1) {
                                for (int x = c - 1; x <= c; ++x)
                                    bulk_store(kRing, static_cast<long>(x) * kChunkBytes,
                                               [&](int bw) { workspace(bw, u.slot, x, 1, true); });
                                commit_group(cta);
                            }
                        }
                        release_tmem();
                        if (opt_.mutation != kMutFlagBeforeBulkWait) wait_groups(cta, 0, true);
                        tick();
                        Flag& f = flags_[static_cast<size_t>(u.slot)];
                        f.value = a_.epoch;
                        f.clock = ve;
                        if (opt_.mutation == kMutFlagBeforeBulkWait) wait_groups(cta, 0, true);
                    } else {
                        const long ps = tile_idx + static_cast<long>(rest);
                        Flag& pf = flags_[static_cast<size_t>(ps)];
                        co_await WaitUntil{[&pf, this] { return pf.value >= a_.epoch; }};
                        join(ve, pf.clock);
                        wait_groups(cta, 0, false);  // bulk_wait_group_read<0>
                        auto fetch = [&](int c) {    // bulk g2s of peer chunk c into epi[c & 1]
                            Barrier& sb = C.pstage[c & 1];
                            expect_tx(sb, kChunkBytes);
                            tick();
                            arrive(sb, ve);
                            issue(G, E);
                            workspace(G, ps, c, 1, false);
                            smem(G, cta, kEpi, static_cast<long>(c & 1) * kChunkBytes, kChunkBytes, true);
                            complete_tx(sb, kChunkBytes, vc_[static_cast<size_t>(G)]);
                        };
                        fetch(0);
                        fetch(1);
                        for (int c = 0; c < NCH; ++c) {
                            tmem(E, cta, buf, c * 32, 32, false);
                            Barrier& sb = C.pstage[c & 1];
                            co_await wait(sb, static_cast<uint32_t>(c >> 1) & 1);
                            acquire(E, sb, static_cast<uint32_t>(c >> 1) & 1);
                            smem(E, cta, kEpi, static_cast<long>(c & 1) * kChunkBytes, kChunkBytes, false);
                            if (c + 2 < NCH) fetch(c + 2);
                            if (a_.c_tma && !a_.sk_head) {
                                smem(E, cta, kRing, static_cast<long>(c) * kChunkBytes, kChunkBytes, true);
                                bulk_store(kRing, static_cast<long>(c) * kChunkBytes, [&](int bw) { store_c(bw, tile, c); });
                                commit_group(cta);
                            } else {
                                store_c(E, tile, c);
                            }
                        }
                        release_tmem();
                    }
                } else {
                    // K-slice tail unit: symmetric fixup
                    const int nslc = a_.sk_slices, s = u.slice;
                    const bool remainder = s == nslc;
                    const int nsrc = nslc + (a_.sk_w > 0 ? 1 : 0);
                    const int rest = a_.tiles_m * a_.tiles_n - a_.sk_tile_begin;
                    const int tile_idx = u.tile - a_.sk_tile_begin;
                    const int c_lo = remainder ? 0 : NCH * s / nslc, c_hi = remainder ? 0 : NCH * (s + 1) / nslc;
                    const int nown = c_hi - c_lo;
                    long slot = u.slot;
                    if (remainder && opt_.mutation == kMutRemainderSlotCollision) slot = ncl_ - 1;
                    const long peer0 = static_cast<long>(nown) * kChunkBytes;  // ring offset of the peer region
                    if (!remainder || (last_unit && a_.ring_drain)) {
                        auto slot_off = [&](int c) {
                            const bool mine = c >= c_lo && c < c_hi;
                            return mine ? static_cast<long>(c - c_lo) * kChunkBytes
                                        : peer0 + static_cast<long>(c < c_lo ? c : c - nown) * kChunkBytes;
                        };
                        for (int c = 0; c < NCH; ++c) {
                            tmem(E, cta, buf, c * 32, 32, false);
                            smem(E, cta, kRing, slot_off(c), kChunkBytes, true);
                            if (c & 1) {
                                for (int x = c - 1; x <= c; ++x)
                                    if (x < c_lo || x >= c_hi)
                                        bulk_store(kRing, slot_off(x), [&](int bw) { workspace(bw, slot, x, 1, true); });
                                commit_group(cta);
                            }
                        }
                    } else {
                        for (int c = 0; c < NCH; ++c) {
                            tmem(E, cta, buf, c * 32, 32, false);
                            const long off = static_cast<long>(epi_chunk++ & 1) * kChunkBytes;
                            wait_groups(cta, 1, false);
                            smem(E, cta, kEpi, off, kChunkBytes, true);
                            bulk_store(kEpi, off, [&](int bw) { workspace(bw, slot, c, 1, true); });
                            commit_group(cta);
                        }
                    }
                    release_tmem();
                    if (opt_.mutation != kMutFlagBeforeBulkWait) wait_groups(cta, 0, true);  // bulk_wait_group<0>
                    tick();
                    Flag& f = flags_[static_cast<size_t>(slot < static_cast<long>(flags_.size()) ? slot : 0)];
                    f.value = a_.epoch;
                    f.clock = ve;  // st.release.gpu
                    if (opt_.mutation == kMutFlagBeforeBulkWait) wait_groups(cta, 0, true);
                    if (nown > 0) {
                        // every source's chunks of my range land on their own barrier
                        // (the kernel issues them in arrival order; each copy follows
                        // the acquire of its source's flag either way)
                        for (int j = 0; j < nsrc; ++j) {
                            if (j == s) continue;
                            const long ps = j < nslc ? tile_idx + static_cast<long>(j) * rest
                                                     : remainder_slot(a_, rest, ncl_, tile_idx);
                            if (ps < 0 || ps >= static_cast<long>(flags_.size())) {
                                ++rep_.capacity_errors;
                                record("capacity", "flag", ps, "flag slot out of range", who(E), cl);
                                continue;
                            }
                            Flag& pf = flags_[static_cast<size_t>(ps)];
                            co_await WaitUntil{[&pf, this] { return pf.value >= a_.epoch; }};
                            join(ve, pf.clock);  // ld.acquire.gpu
                            tick();
                            Barrier& sb = C.src[j];
                            expect_tx(sb, static_cast<long>(nown) * kChunkBytes);
                            arrive(sb, ve);
                            issue(G, E);
                            workspace(G, ps, c_lo, nown, false);
                            const int pj = opt_.mutation == kMutUnpackedPeerStaging ? j : (j < s ? j : j - 1);
                            smem(G, cta, kRing, peer0 + static_cast<long>(pj) * nown * kChunkBytes,
                                 static_cast<long>(nown) * kChunkBytes, true);
                            complete_tx(sb, static_cast<long>(nown) * kChunkBytes, vc_[static_cast<size_t>(G)]);
                        }
                        // sum in slice order as the sources land; a TMA C stores each
                        // chunk as soon as it is summed
                        for (int c = c_lo; c < c_hi; ++c) {
                            for (int j = 0; j < nsrc; ++j) {
                                if (j != s && c == c_lo) {
                                    co_await wait(C.src[j], 0);
                                    acquire(E, C.src[j], 0);
                                }
                                const int pj = opt_.mutation == kMutUnpackedPeerStaging ? j : (j < s ? j : j - 1);
                                const long off = j == s ? static_cast<long>(c - c_lo) * kChunkBytes
                                                        : peer0 + (static_cast<long>(pj) * nown + (c - c_lo)) * kChunkBytes;
                                smem(E, cta, kRing, off, kChunkBytes, false);
                            }
                            if (a_.c_tma) {
                                smem(E, cta, kRing, static_cast<long>(c - c_lo) * kChunkBytes, kChunkBytes, true);
                                bulk_store(kRing, static_cast<long>(c - c_lo) * kChunkBytes,
                                           [&](int bw) { store_c(bw, tile, c); });
                                commit_group(cta);
                            } else {
                                store_c(E, tile, c);
                            }
                        }
                    }
                }
            } else {
                // cluster split-K: the partial tile goes to the (drained) ring, every
                // rank reduces its column slice over DSMEM in rank order
                (void)tile_use;
                const long red_bytes = static_cast<long>(S::BM) * S::RED_LD * 4;
                tmem(E, cta, buf, 0, BN, false);
                smem(E, cta, kRing, 0, red_bytes, true);
                release_tmem();
                for (int r = 0; r < kSplitK; ++r) arrive(ctas_[static_cast<size_t>(cta_of(cl, r))].rfull, ve);
                co_await wait(C.rfull, tile_use & 1);
                acquire(E, C.rfull, tile_use & 1);
                constexpr int kCols = BN / kSplitK;
                const int c0 = rank * kCols;
                for (int r = 0; r < kSplitK; ++r)  // ld.shared::cluster of every rank's rows
                    smem(E, cta_of(cl, r), kRing, 0, red_bytes, false);
                for (int cc = 0; cc < kCols; cc += 32) store_c(E, tile, (c0 + cc) / 32);
                tick();
                for (int r = 0; r < kSplitK; ++r) arrive(ctas_[static_cast<size_t>(cta_of(cl, r))].rempty, ve);
            }
            u = nxt;
            have = have_next;
        }
        wait_groups(cta, 0, true);
    }
};

template <int kCtaGroup, int BN, int kSplitK, int kSlabs = 1, int kNHalves = 1, int kMcast = 1>
void run_checker(GemmArgs args, int sms, int force_slices, const AsyncCheckOptions& o, AsyncReport& rep) {
    using S = GemmShape<kCtaGroup, BN, kSplitK, kSlabs, kNHalves>;
    constexpr int kCluster = kCtaGroup * kSplitK * kMcast;
    const int tiles = args.tiles_m * args.tiles_n;
    int clusters = sms / kCluster;
    if (o.max_active_clusters > 0 && o.max_active_clusters < clusters) clusters = o.max_active_clusters;
    // as the launcher: slab tiles (512-row pair tiles) run whole tiles only
    const SchedulePlan plan =
        kSlabs * kNHalves * kMcast > 1 ? plan_schedule<kCtaGroup, BN, kSplitK>(tiles, args.k_blocks, clusters, args.b_mn_major != 0, 0, 0,
                                                           0, -1, 0)
                   : plan_schedule<kCtaGroup, BN, kSplitK>(tiles, args.k_blocks, clusters, args.b_mn_major != 0,
                                                           o.streamk, force_slices, o.remainder,
                                                           o.pull_d == -2 ? BN / 32 : o.pull_d, o.head);
    rep.tiles = tiles;
    rep.cluster_size = kCluster;
    rep.split_k = kSplitK > 1 ? kSplitK : (force_slices > 1 ? force_slices : 1);
    rep.stages = (args.stages > 0 && args.stages < S::kStages) ? args.stages : S::kStages;
    if (plan.status != 0) {
        ++rep.capacity_errors;
        rep.records.push_back({"capacity", "grid", tiles, "forced K slices exceed the persistent grid", "", -1});
        return;
    }
    if (plan.mode) {
        args.streamk = plan.mode;
        args.sk_tile_begin = plan.sk_begin;
        args.sk_slices = plan.slices;
        args.sk_w = plan.sk_w;
        args.sk_extra = plan.sk_extra;
        args.sk_q = plan.sk_q;
        args.sk_pull = plan.sk_pull;
        args.sk_head = plan.sk_head;
    }
    args.epoch = 1;
    if (o.gated_chunks > 0) {  // as fi_plan_launch_gated: chunk tiles, raster rotated to the first chunk
        if (args.tiles_n % o.gated_chunks != 0 || o.gated_first < 0 || o.gated_first >= o.gated_chunks) {
            ++rep.capacity_errors;
            rep.records.push_back({"capacity", "B chunk", o.gated_chunks, "chunks must split the tile columns evenly", "", -1});
            return;
        }
        args.b_chunk_tiles = args.tiles_n / o.gated_chunks;
        rep.gated_chunks = o.gated_chunks;
        args.n_rot = o.gated_first * args.b_chunk_tiles;
        args.b_epoch = 1;
    }
    rep.clusters = plan.clusters;
    rep.mode = plan.mode;
    rep.slices = plan.slices;
    rep.remainder = plan.sk_w > 0 && !plan.sk_pull ? 1 : 0;
    rep.pull = plan.sk_pull;
    rep.head = plan.sk_head;
    for (int c = 0; c < plan.clusters; ++c) {
        UnitIter<BN> it(args, c, plan.clusters);
        Unit u;
        while (it.next(u)) ++rep.units;
    }
    Checker<kCtaGroup, BN, kSplitK, kSlabs, kNHalves, kMcast> chk(args, plan.clusters, plan.slots, o, rep);
    chk.run();
}

}  // namespace

AsyncReport check_async(const Spec& root, const NodePtr& tree, const AsyncCheckOptions& opts,
                        const MicroKernelSet& mks) {
    TcStrategy tc = match_tc_strategy(root, tree, mks);
    if (!tc.matched) fail(ErrorKind::InvalidTree, "not a tcgen05 strategy: " + tc.why_not);
    const auto& mm = root.mm();
    // the launcher's configuration (runtime/plan.cpp Plan::create)
    const int bm = tc.tile_m;  // 128, 256 (pair) or 512 (pair, two A slabs)
    const long M = root.m(), N = root.n(), K = root.k();
    int split_k = tc.split_k, force_slices = 0;
    if (M % bm || N % tc.tile_n || K % (64 * split_k))
        fail(ErrorKind::ShapeMismatch, "problem is not a multiple of the block tile");
    const long tiles = (M / bm) * (N / tc.tile_n);
    if (split_k > 1 && tc.cta_group == 2 && tiles * split_k <= opts.num_sms / 2) {
        force_slices = split_k;
        split_k = 1;
    }
    sm100::GemmArgs a;
    a.M = static_cast<int>(M);
    a.N = static_cast<int>(N);
    a.K = static_cast<int>(K);
    a.tiles_m = static_cast<int>(M / bm);
    a.tiles_n = static_cast<int>(N / (tc.tile_n * tc.mcast));
    a.k_blocks = static_cast<int>(K / 64 / split_k);
    a.b_mn_major = mm.b.layout.major == Major::RowMajor ? 1 : 0;
    a.c_row_major = mm.c.layout.major == Major::RowMajor ? 1 : 0;
    a.out_type = mm.c.elem == ElemType::F32 ? 0 : mm.c.elem == ElemType::F16 ? 1 : 2;
    a.stages = tc.stages;
    a.c_tma = opts.c_tma >= 0 ? opts.c_tma : (split_k == 1 && a.out_type == 0 && !a.c_row_major ? 1 : 0);
    a.ring_drain = opts.ring_drain;
    AsyncReport rep;
    if (tc.tile_m == 512) {
        run_checker<2, 256, 1, 2>(a, opts.num_sms, force_slices, opts, rep);
        return rep;
    }
    if (tc.tile_n == 512) {
        run_checker<2, 256, 1, 1, 2>(a, opts.num_sms, force_slices, opts, rep);
        return rep;
    }
    if (tc.mcast == 2) {
        if (tc.tile_n == 64) run_checker<2, 64, 1, 1, 1, 2>(a, opts.num_sms, force_slices, opts, rep);
        else if (tc.tile_n == 128) run_checker<2, 128, 1, 1, 1, 2>(a, opts.num_sms, force_slices, opts, rep);
        else run_checker<2, 256, 1, 1, 1, 2>(a, opts.num_sms, force_slices, opts, rep);
        return rep;
    }
#define FI_CHECK(CG, BN_, SK)                                                        \
    if (tc.cta_group == CG && tc.tile_n == BN_ && split_k == SK) {                 \
        run_checker<CG, BN_, SK>(a, opts.num_sms, force_slices, opts, rep);        \
        return rep;                                                                \
    }
    FI_CHECK(1, 64, 1) FI_CHECK(1, 128, 1) FI_CHECK(1, 256, 1) FI_CHECK(2, 64, 1) FI_CHECK(2, 128, 1) FI_CHECK(2, 256, 1)
    FI_CHECK(1, 64, 2) FI_CHECK(1, 128, 2) FI_CHECK(1, 128, 4) FI_CHECK(1, 256, 2) FI_CHECK(1, 256, 4)
    FI_CHECK(2, 256, 2) FI_CHECK(2, 256, 4) FI_CHECK(2, 128, 2) FI_CHECK(2, 128, 4)
#undef FI_CHECK
    fail(ErrorKind::InvalidTree, "no tcgen05 kernel instance for this tile configuration");
}

}  // namespace fireiron
