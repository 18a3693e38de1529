// graph.cuh — device-resident hypergraph levels.
//
// HBM layout per level (all CSR offsets int64, ids int32):
//   src_off/src_dat, dst_off/dst_dat : per h-edge source / destination pins
//   pin_off/pin_dat                  : per h-edge sorted unique src ∪ dst
//   in_off/in_dat                    : per node ascending inbound h-edges
//   inc_off/inc_dat                  : per node ascending incident h-edges
//   size                             : per node level-0 node count
// Weights are level-independent (h-edges are never merged, coarsen.py:146).
#pragma once
#include "common.cuh"

namespace dhgp {

struct DLevel {
    int32_t N = 0, E = 0;
    int64_t Ps = 0, Pd = 0, U = 0, Sin = 0;
    int64_t *src_off = nullptr, *dst_off = nullptr, *pin_off = nullptr, *in_off = nullptr, *inc_off = nullptr;
    int32_t *src_dat = nullptr, *dst_dat = nullptr, *pin_dat = nullptr, *in_dat = nullptr, *inc_dat = nullptr;
    int32_t *size = nullptr;
    // Per-node lists may live in a shared pool (node_pool): node n's list is
    // [in_off[n], in_end[n]) of in_dat.  in_end == nullptr means plain CSR
    // (end = in_off + 1); in_e() / inc_e() give the end array either way.
    int64_t *in_end = nullptr, *inc_end = nullptr;
    bool pooled = false;       // in_dat / inc_dat belong to the partition's node pool
    const int64_t *in_e() const { return in_end ? in_end : in_off + 1; }
    const int64_t *inc_e() const { return inc_end ? inc_end : inc_off + 1; }
    int32_t *gamma = nullptr;  // fine -> coarse map once this level has been contracted
    int32_t maxp = 0;          // bound on any h-edge's pin slots (src + dst) at this level
    bool borrowed = false;     // src/dst/size belong to a resident input (level 0)
    bool stub = false;         // lists dropped (only gamma kept); rebuilt on demand
    void release(Ctx &c) {
        if (!borrowed) {
            c.free(src_off); c.free(dst_off); c.free(src_dat); c.free(dst_dat); c.free(size);
        }
        c.free(pin_off); c.free(in_off); c.free(inc_off);
        c.free(in_end); c.free(inc_end);
        c.free(pin_dat);
        if (!pooled) {
            c.free(in_dat);
            c.free(inc_dat);
        }
        c.free(gamma);
        *this = DLevel();
    }
};

// Shared storage of the per-node lists (in, inc) of every level: level 0's
// lists, then each contraction's merged-cluster unions appended; an unmerged
// node keeps pointing at its list where it is, so a contraction writes only
// the unions and a kept level costs only its (begin, end) arrays.  Offsets
// are relative to dat[f]; growing the pool moves the data and keeps them.
struct NodePool {
    int32_t *dat[2] = {nullptr, nullptr};  // [0] in lists, [1] inc lists
    int64_t cap[2] = {0, 0};
    int64_t *top = nullptr;                // device [2]: next free slot of each family
    void release(Ctx &c) {
        c.free(dat[0]);
        c.free(dat[1]);
        c.free(top);
        *this = NodePool();
    }
};

struct DWeights {
    int32_t E = 0;
    const double *w = nullptr;  // [E] as given (borrowed from the input)
    int64_t *wi = nullptr;      // [E] w * 2^scale_bits as integers (exact-integer mode)
    int64_t wsum = 0;           // sum of wi
    int scale_bits = 0;         // S: every weight is a multiple of 2^-S (0 when integral)
    double unit = 1.0;          // 2^-S: a sum of wi times unit is the reference's f64 value
    bool integral = true;       // wi exact and wsum < 2^53: the exact-integer device path applies
    void release(Ctx &c) {
        c.free(wi);
        *this = DWeights();
    }
};

// Primary hypergraph fields resident in HBM (the inputs of partition()).
struct DInput {
    int32_t N = 0, E = 0;
    int64_t Ps = 0, Pd = 0;
    int64_t *src_off = nullptr, *dst_off = nullptr;
    int32_t *src_dat = nullptr, *dst_dat = nullptr;
    double *w = nullptr;
    int32_t *size = nullptr;
    int32_t max_edge_pins = 0;
    void release(Ctx &c) {
        c.free(src_off); c.free(dst_off); c.free(src_dat); c.free(dst_dat); c.free(w); c.free(size);
        *this = DInput();
    }
};
// host -> HBM copy of the primary fields (offsets rebased to 0)
void upload_input(Ctx &c, const dhgp_graph &g, DInput &in);
// Validates the weights (finite, >= 0) and derives the exact-integer copy:
// dyadic weights (multiples of 2^-S, e.g. 0.5 steps) are scaled by 2^S.
void prepare_weights(Ctx &c, const DInput &in, DWeights &W);
// Level 0 over a resident input (Hypergraph._from_csr, hgraph.py:212-238).
void build_level0(Ctx &c, const DInput &in, DLevel &L);
// Derived families from device-resident src/dst (used at level 0).
void derive_incidence(Ctx &c, DLevel &L);
// node_out (only for the incidence API / observer)
void derive_out(Ctx &c, const DLevel &L, int64_t *out_off, int32_t *out_dat);

// check_feasibility (hgraph.py:376-401): returns first offending node or -1
// for each of (size > omega, |in| > delta).
void feasibility(Ctx &c, const DLevel &L, int64_t omega, int64_t delta, int32_t *bad_size, int32_t *bad_in);
// The same check straight from the resident input (in-degree = occurrences in
// the destination lists), so that it runs before anything that could reject
// the input as unsupported — the reference checks feasibility first
// (driver.py:89 -> hgraph.py:376-401).  *size_val / *indeg_val receive the
// offending values.
void feasibility_input(Ctx &c, const DInput &in, int64_t omega, int64_t delta, int32_t *bad_size, int32_t *bad_in,
                       int32_t *size_val, int32_t *indeg_val);

}  // namespace dhgp
