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

// refine_level (refine.py:262-318) with sparse per-edge part counters in
// place of the dense (E x K) pins matrices.  `assign` (device, L.N) is
// refined in place; connectivity values are appended to `conns`.
void refine_level(Ctx &c, const DLevel &L, const DWeights &W, int32_t *assign, int32_t K, int64_t omega,
                  int64_t delta, int32_t max_rounds, int32_t level, std::vector<double> &conns,
                  const RoundObserver *obs, int32_t max_edge_pins);

// connectivity (A12) and per-part sizes / distinct inbound (A13/A16) of an
// assignment; any of the outputs may be null.
void evaluate_assign(Ctx &c, const DLevel &L, const DWeights &W, const int32_t *assign, int32_t K,
                     int64_t *d_sizes, int64_t *d_inbound, double *h_conn);

}  // namespace dhgp
