// coarsen.cuh — one coarsening level on device.
#pragma once
#include "graph.cuh"

namespace dhgp {

// A4+A5+A6 fused: per node, shared-edge-weight histogram over the pins of
// its incident h-edges (never written to HBM), candidates in (hist desc,
// id desc) order, first one passing the size and inbound-union checks.
// coarsen.py:93-132, _kernels.pyx:47-103.  Requires exact-integer weights.
void score_select(Ctx &c, const DLevel &L, const DWeights &W, int64_t omega, int64_t delta, int32_t *pair,
                  double *score);

// A7: pseudo-forest -> involution (_kernels.pyx:106-181).  Returns the number
// of matched pairs (PairingForest.matched_pairs, coarsen.py:54-58); throws
// DHGP_ERR_MATCHING on a pairing cycle of length != 2.
int64_t resolve_matching(Ctx &c, int32_t N, const int32_t *pair, const double *score, int32_t *match,
                         uint8_t *isrep);

// A9: contraction (coarsen.py:141-173).  Fills fine.gamma and builds coarse.
void contract(Ctx &c, DLevel &fine, const int32_t *match, const uint8_t *isrep, DLevel &coarse);

}  // namespace dhgp
