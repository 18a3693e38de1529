// ordered.cuh — the reference-order f64 path.
//
// Weights that are not multiples of one power of two (e.g. 0.1 steps) make
// the reference's f64 sums round at every step, so only its own summation
// order reproduces them: hist in ascending h-edge order
// (_kernels.pyx:65-70), saving / total / present[p] likewise (270-297),
// gain_seq's per-edge nets (330-362), the prefix cumsum (refine.py:244) and
// connectivity (_kernels.pyx:199-213).  This path keeps every one of those
// sums sequential in that order — one thread or one warp per sum, the sums
// of different nodes / moves / h-edges in parallel — and the phase structure
// of the reference (dense pins matrices, sorted candidate lists), so it is
// slower and needs E x K x 8 bytes, like the reference.  Everything
// weight-independent (incidence, matching, contraction, part sizes) is the
// production code.
#pragma once
#include "graph.cuh"
#include "refine.cuh"

namespace dhgp {

// 𝒩(n) as device CSR (coarsen.py:78-85): *nb_off [N+1], *nb_dat [nnz]; the
// caller frees both
void ord_neighbors(Ctx &c, const DLevel &L, int64_t **nb_off, int32_t **nb_dat, int64_t *nnz);
// hist (fill_histograms) in ascending h-edge order per neighbour slot
void ord_fill_hist(Ctx &c, const DLevel &L, const double *w, const int64_t *nb_off, const int32_t *nb_dat,
                   double *hist);
// first valid candidate in (hist desc, id desc) order (coarsen.py:118-132)
void ord_select(Ctx &c, const DLevel &L, const int64_t *nb_off, const int32_t *nb_dat, const double *hist,
                int64_t nnz, int64_t omega, int64_t delta, int32_t *pair, double *score);
// dense pins / pins_in [E x K] (compute_pins, _kernels.pyx:216-231)
void ord_dense_pins(Ctx &c, const DLevel &L, const int32_t *assign, int32_t K, int32_t *pins, int32_t *pins_in);
// propose_moves (_kernels.pyx:234-311): target [N] (-1 none), gain [N]
void ord_propose(Ctx &c, const DLevel &L, const double *w, const int32_t *pins, int32_t K, const int32_t *assign,
                 const int64_t *psizes, int64_t omega, int32_t *target, double *gain);
// sequence_gains (_kernels.pyx:314-364)
void ord_seq_gains(Ctx &c, const DLevel &L, const double *w, const int32_t *pins, int32_t K, int32_t M,
                   const int32_t *node, const int32_t *from, const int32_t *to, const double *giso,
                   const int64_t *pos, double *gseq);
// distinct_inbound_sizes from the dense pins_in (hgraph.py:324-339)
void ord_pinbound(Ctx &c, int32_t E, int32_t K, const int32_t *pins_in, int64_t *pinb);
// build_events_and_select (refine.py:178-247); pins_in is consumed (mutated)
void ord_select_prefix(Ctx &c, const DLevel &L, int32_t K, int32_t M, const int32_t *node, const int32_t *from,
                       const int32_t *to, const double *gseq, int32_t *pins_in, int64_t *psizes, int64_t *pinb,
                       int64_t omega, int64_t delta, int64_t *active, int64_t *k_out, double *total);
// connectivity_value in ascending h-edge order (host result)
double ord_connectivity(Ctx &c, const DLevel &L, const double *w, const int32_t *assign);

// One level's candidate scoring: neighbours, histogram, ordered walk.
void ord_score(Ctx &c, const DLevel &L, const double *w, int64_t omega, int64_t delta, int32_t *pair,
               double *score);
// refine_level (refine.py:262-318) of one level in reference order; appends
// the level's connectivity values to `conns`
void ord_refine_level(Ctx &c, const DLevel &L, const double *w, int32_t *assign, int32_t K, int64_t omega,
                      int64_t delta, int32_t max_rounds, int32_t level, std::vector<double> &conns,
                      const RoundObserver *obs);
// fine assign = coarse assign o gamma (refine.py:257-259)
void ord_project(Ctx &c, int32_t N, const int32_t *gamma, const int32_t *coarse, int32_t *fine);

}  // namespace dhgp
