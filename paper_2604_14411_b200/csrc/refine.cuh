// refine.cuh — one refinement level on device.
#pragma once
#include <functional>

#include "graph.cuh"

namespace dhgp {

// host-side view of one round for the observer hook (refine.py:295-307)
struct RoundRecord {
    int32_t level, round, num_parts, k;
    double total_gain;
    std::vector<int32_t> assign, node, from, to;
    std::vector<double> gain_iso, gain_seq;
    std::vector<int64_t> active;
};
using RoundObserver = std::function<void(const RoundRecord &)>;

// Refinement state carried across rounds and levels (uncoarsening).
//
// The per-h-edge run lists (sparse replacement of the dense pins/pins_in
// matrices) live at the level-0 pin offsets, which bound every level's pin
// count, so h-edge e keeps its slot on every level.  In incremental mode a
// round recomputes only what changed since the previous proposal:
//   - run lists of h-edges touched by applied moves (their pins' proposals
//     are then stale) or by a split cluster during projection (counts only;
//     no other node's proposal changes, see refine.cu);
//   - proposals of dirty nodes, and of nodes whose choice depends on a part
//     size that changed (target part grew, or a size-filtered better part
//     may have become eligible: `fsens`);
//   - sequence gains and inbound events over the movers' h-edges only.
// Every other value equals what a full recomputation gives (bit-exact).
struct RefineState {
    bool inc = false;     // incremental mode (else every round is recomputed)
    bool fresh = true;    // no valid proposals yet (coarsest level)
    bool moved = false;   // moves applied since the last proposal pass
    int32_t K = 0, E = 0;
    int64_t ncap = 0;
    const int64_t *roff = nullptr;                         // [E+1] run base (level-0 pin offsets)
    int32_t *rpc = nullptr, *rcin = nullptr, *rlen = nullptr;  // runs: (part, count) pairs [2U], count_in [U], lambda [E]
    int64_t *psizes = nullptr, *pinbound = nullptr;        // [K]
    uint8_t *pflags = nullptr;                             // [K] bit 1: part shrank
    unsigned long long *conn = nullptr;                    // connectivity of the current runs
    int32_t *target = nullptr, *target2 = nullptr;         // [ncap] per node (double-buffered for projection)
    int64_t *gain = nullptr, *gain2 = nullptr;
    uint8_t *fsens = nullptr, *fsens2 = nullptr;           // filtered positive parts: count (3 = more)
    int32_t *fpart = nullptr, *fpart2 = nullptr;           // [2 ncap] the first two of them
    int32_t *ndirty = nullptr, *ndirty2 = nullptr;         // [N0] dirty-node flags
    int32_t *nlist = nullptr, *ccount = nullptr;  // [N0]
    int32_t *splist = nullptr;   // [N0] split clusters' halves as (min, max) pairs
    int32_t *spfirst = nullptr;  // [N0] per coarse node: the first half seen (pairing)
    int32_t *edirty = nullptr, *elist = nullptr;           // [E] dirty h-edges (bit 0 split, bit 1 moved)
    int32_t *emflag = nullptr, *mlist = nullptr;           // [E] h-edges of the round's movers
    int32_t *wide = nullptr;                               // [E] dirty h-edges over 128 pins (block update)
    int32_t *ctr = nullptr;                                // [8] list counters
    int32_t hub_max = 0;                                   // propose hub tier capacity
    long long *hacc = nullptr, *htot = nullptr;            // [hub_max x K], [2 hub_max]
    int32_t *hdone = nullptr, *hlist = nullptr;            // [hub_max]
    int32_t *hpref = nullptr;                              // [hub_max + 1] work-item prefix
};
void refine_state_init(Ctx &c, RefineState &st, const DLevel &level0, int32_t K, bool incremental);
void refine_state_release(Ctx &c, RefineState &st);
// Projection to the next finer level (refine.py:257-259): assign, the
// carried proposals and dirty flags follow gamma; split clusters mark their
// halves and incident h-edges dirty.  Swaps assign/assign2.
void refine_project(Ctx &c, RefineState &st, const DLevel &fine, int32_t coarse_n, int32_t *&assign,
                    int32_t *&assign2);

// refine_level (refine.py:262-318) with sparse per-edge part counters in
// place of the dense (E x K) pins matrices.  `assign` (device, L.N) is
// refined in place; connectivity values are appended to `conns`.
void refine_level(Ctx &c, const DLevel &L, const DWeights &W, RefineState &st, int32_t *assign, int32_t K,
                  int64_t omega, int64_t delta, int32_t max_rounds, int32_t level, std::vector<double> &conns,
                  const RoundObserver *obs, int32_t max_edge_pins);

// connectivity (A12) and per-part sizes / distinct inbound (A13/A16) of an
// assignment; any of the outputs may be null.
void evaluate_assign(Ctx &c, const DLevel &L, const DWeights &W, const int32_t *assign, int32_t K,
                     int64_t *d_sizes, int64_t *d_inbound, double *h_conn);

}  // namespace dhgp
