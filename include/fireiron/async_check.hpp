// CPU checker for the asynchronous protocol of the tcgen05 GEMM family
// (SURVEY.md 8(f) rank 4).
//
// The reference validates its strategies on the CPU with a same-phase race
// detector over shared memory and a register-ownership check
// (proj/include/anvil/sim.hpp:63-104 detect_races, :268-312 note_sh_access /
// check_owner, :546-561 check_ownership). The B200 lowering has no barrier
// phases a thread-level model could use: its synchronisation is mbarrier
// phases completed by TMA transactions and tcgen05.commit, async-proxy bulk
// copies, TMEM accumulator hand-off and release/acquire epoch flags between
// clusters. check_async replays the launch exactly as the kernel schedules it
// (the same UnitIter and launch planner, sm100/schedule.hpp) with one agent
// per role (TMA producer, MMA issuer, epilogue) and per asynchronous engine
// (TMA loads, tcgen05.mma, bulk stores, bulk loads) of every cluster, tracks
// happens-before with vector clocks, and reports
//   * races: two accesses to one shared-memory / TMEM / workspace / C cell,
//     at least one a write, not ordered by the protocol;
//   * capacity violations: staging outside the operand ring, epilogue
//     buffers, TMEM columns or workspace slots the launch allocates;
//   * coverage errors: an output chunk stored zero or several times;
//   * deadlocks: a wait no arrival can complete.
// Mutations inject known protocol faults so the checker's own tests can show
// each class is caught (the reference's noSync race tests play that role).
#pragma once

#include <string>
#include <vector>

#include "fireiron/program.hpp"
#include "fireiron/script.hpp"

namespace fireiron {

enum AsyncMutation : int {
    kMutNone = 0,
    kMutSkipEmptyWait = 1,          // producer refills a stage without waiting for the MMA to free it
    kMutRingDrainEveryUnit = 2,     // every unit (not only the last) stages C in the operand ring
    kMutFlagBeforeBulkWait = 3,     // a tail slice publishes its flag before its bulk stores completed
    kMutSkipTmemEmptyWait = 4,      // the MMA reuses an accumulator before the epilogue drained it
    kMutRemainderSlotCollision = 5, // remainder partials all written to one workspace slot
    kMutUnpackedPeerStaging = 6,    // owners stage peers at j*nown chunks (the pre-remainder layout)
    kMutTxUndercount = 7,           // expect_tx without the second B half of an N-half tile
    kMutMcastSingleRelease = 8,     // multicast: a stage refilled after one pair's release, not both
    kMutGateSkipAcquire = 9,        // gated B: the producer loads a chunk without acquiring its ready flag
};

struct AsyncCheckOptions {
    int num_sms = 148;
    int max_active_clusters = 0;  // occupancy cap; 0 = num_sms / cluster size
    int streamk = -1;             // as FI_STREAMK: -1 auto, 0 data-parallel, 1 K-slice, 2 N-split
    int remainder = 1;            // as FI_REMAINDER
    int c_tma = -1;               // -1 as the launcher decides (f32 column-major C), 0/1 force
    int ring_drain = 1;           // as FI_TC_RING_DRAIN
    int pull_d = -2;              // as FI_TC_PULL_D: -2 the launcher's default, -1 no pull fixup
    int head = 1;                 // as FI_TC_HEAD: 2-slice pull tails run before the data-parallel tiles
    int mutation = kMutNone;
    int gated_chunks = 0;         // > 0: a gated launch (fi_plan_launch_gated) with B in this many column chunks,
    int gated_first = 0;          //      each written by a copy engine and released by its ready flag
};

struct AsyncRecord {
    std::string kind;      // race | capacity | coverage | deadlock
    std::string resource;  // ring / epi / tmem / workspace / C / flag / barrier
    long index = 0;
    std::string first, second;  // the two agents (race), or a description
    int cluster = -1;
};

struct AsyncReport {
    long events = 0;  // checked accesses
    long races = 0, capacity_errors = 0, coverage_errors = 0, deadlocks = 0;
    // the schedule that was checked
    int clusters = 0, cluster_size = 1, mode = 0, slices = 1, remainder = 0, pull = 0, head = 0, split_k = 1, stages = 0;
    int gated_chunks = 0;  // > 0: a gated launch was modelled (B in this many copy-engine chunks)
    long units = 0, tiles = 0;
    std::vector<AsyncRecord> records;  // first 256
    bool ok() const { return races == 0 && capacity_errors == 0 && coverage_errors == 0 && deadlocks == 0; }
    std::string to_string() const;
};

// Checks the launch a tcgen05 strategy lowers to (throws fireiron::Error for
// trees without a tcgen05 lowering, like Plan::create).
AsyncReport check_async(const Spec& root, const NodePtr& tree, const AsyncCheckOptions& opts = AsyncCheckOptions{},
                        const MicroKernelSet& mks = MicroKernelSet{});

}  // namespace fireiron
