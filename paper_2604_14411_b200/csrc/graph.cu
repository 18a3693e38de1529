// graph.cu — level-0 upload and incidence materialisation.
#include <cmath>

#include "graph.cuh"
#include "prims.cuh"

namespace dhgp {

namespace {
// weights: finite, >= 0; exact-integer mode needs integral values with a
// total < 2^53 so every partial sum in any order is exact.
// Weights w = m * 2^e are all multiples of 2^-S, S = the most fractional
// bits of any weight (0 for integral weights).  With the scaled integers
// w * 2^S summing below 2^53, every partial sum the reference forms in its
// fixed order is an exactly representable multiple of 2^-S, so
// integer accumulation in any order followed by one multiplication by 2^-S
// is bit-identical to it.
__device__ __forceinline__ int weight_frac_bits(double x) {
    if (x == 0.0) return 0;
    int e;
    const double m = frexp(x, &e);
    const unsigned long long mant = (unsigned long long)ldexp(m, 53);
    const int fb = 53 - (__ffsll((long long)mant) - 1) - e;
    return fb > 0 ? fb : 0;
}
__global__ void k_check_weights(const double *w, int64_t E, int32_t *flags, int32_t *maxbits) {
    pdl_entry();
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int mb = 0;
    if (e < E) {
        double x = w[e];
        if (!(x >= 0.0) || !isfinite(x)) atomicOr(&flags[0], 1);  // invalid weight
        else mb = weight_frac_bits(x);
    }
    for (int o = 16; o; o >>= 1) mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
    if ((threadIdx.x & 31) == 0 && mb) atomicMax(maxbits, mb);
}
__global__ void k_scale_weights(const double *w, int64_t E, const int32_t *maxbits, int64_t *wi,
                                unsigned long long *sum, int32_t *flags) {
    pdl_entry();
    __shared__ int64_t sh[33];
    const int S = *maxbits;
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t v = 0;
    if (e < E && S <= 62) {
        const double x = ldexp(w[e], S);
        if (x >= 9007199254740992.0) atomicOr(&flags[0], 2);  // a scaled weight alone reaches 2^53
        else v = (int64_t)x;
        wi[e] = v;
    }
    int64_t t = block_sum<int64_t>(v, sh);
    if (threadIdx.x == 0) atomicAdd(sum, (unsigned long long)t);
}

__global__ void k_rebase(int64_t *off, int64_t n, int64_t base) {
    pdl_entry();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) off[i] -= base;
}

__global__ void k_max_edge(int64_t E, const int64_t *so, const int64_t *dof, int32_t *mx) {
    pdl_entry();
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < E) atomicMax(mx, (int32_t)(so[e + 1] - so[e] + dof[e + 1] - dof[e]));
}

__global__ void k_comb(int64_t E, const int64_t *so, const int32_t *sd, const int64_t *dof, const int32_t *dd,
                       int64_t *co, int32_t *cd) {
    pdl_entry();
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e > E) return;
    co[e] = so[e] + dof[e];
    if (e == E) return;
    int64_t o = so[e] + dof[e];
    for (int64_t p = so[e]; p < so[e + 1]; p++) cd[o++] = sd[p];
    for (int64_t p = dof[e]; p < dof[e + 1]; p++) cd[o++] = dd[p];
}

__global__ void k_feasible(int32_t N, const int32_t *size, const int64_t *in_off, int64_t omega, int64_t delta,
                           int32_t *bad) {
    pdl_entry();
    int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    if ((int64_t)size[n] > omega) atomicMin(&bad[0], (int32_t)n);
    if (in_off[n + 1] - in_off[n] > delta) atomicMin(&bad[1], (int32_t)n);
}
__global__ void k_indegree(int64_t Pd, const int32_t *dst_dat, int32_t *deg) {
    pdl_entry();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < Pd; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&deg[dst_dat[i]], 1);
}
__global__ void k_feasible_deg(int32_t N, const int32_t *size, const int32_t *deg, int64_t omega, int64_t delta,
                               int32_t *bad) {
    pdl_entry();
    int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    if ((int64_t)size[n] > omega) atomicMin(&bad[0], (int32_t)n);
    if ((int64_t)deg[n] > delta) atomicMin(&bad[1], (int32_t)n);
}
}  // namespace

void upload_input(Ctx &c, const dhgp_graph &g, DInput &in) {
    const int64_t E = g.num_edges;
    in.N = g.num_nodes;
    in.E = g.num_edges;
    const int64_t sb = g.src_off[0], db = g.dst_off[0];
    in.Ps = g.src_off[E] - sb;
    in.Pd = g.dst_off[E] - db;
    in.src_off = c.alloc<int64_t>(E + 1);
    in.dst_off = c.alloc<int64_t>(E + 1);
    in.src_dat = c.alloc<int32_t>(in.Ps);
    in.dst_dat = c.alloc<int32_t>(in.Pd);
    in.w = c.alloc<double>(E);
    c.h2d(in.src_off, g.src_off, E + 1);
    c.h2d(in.dst_off, g.dst_off, E + 1);
    c.h2d(in.src_dat, g.src_dat + sb, in.Ps);
    c.h2d(in.dst_dat, g.dst_dat + db, in.Pd);
    c.h2d(in.w, g.edge_weight, E);
    if (sb) {
        pdl_launch(k_rebase, (unsigned)cdiv(E + 1, 256), 256, 0, c.stream, in.src_off, E + 1, sb);
        DHGP_LAUNCHED(c);
    }
    if (db) {
        pdl_launch(k_rebase, (unsigned)cdiv(E + 1, 256), 256, 0, c.stream, in.dst_off, E + 1, db);
        DHGP_LAUNCHED(c);
    }
    in.size = c.alloc<int32_t>(in.N);
    if (g.node_size)
        c.h2d(in.size, g.node_size, in.N);
    else
        fill_i32(c, in.size, 1, in.N);
    // largest h-edge (bounds every per-edge sort at every level)
    int32_t *mx = c.alloc<int32_t>(1);
    c.zero(mx, 1);
    if (E > 0) {
        pdl_launch(k_max_edge, (unsigned)cdiv(E, 256), 256, 0, c.stream, E, in.src_off, in.dst_off, mx);
        DHGP_LAUNCHED(c);
    }
    c.d2h(&in.max_edge_pins, mx, 1);
    c.sync();
    c.free(mx);
}

void prepare_weights(Ctx &c, const DInput &in, DWeights &W) {
    W.E = in.E;
    W.w = in.w;
    W.wi = c.alloc<int64_t>(W.E);
    unsigned long long *sum = c.alloc<unsigned long long>(1);
    int32_t *flags = c.alloc<int32_t>(2);
    c.zero(sum, 1);
    c.zero(flags, 2);
    if (W.E > 0) {
        pdl_launch(k_check_weights, (unsigned)cdiv(W.E, 256), 256, 0, c.stream, W.w, W.E, flags, flags + 1);
        DHGP_LAUNCHED(c);
        pdl_launch(k_scale_weights, (unsigned)cdiv(W.E, 256), 256, 0, c.stream, W.w, W.E, flags + 1, W.wi, sum, flags);
        DHGP_LAUNCHED(c);
    }
    unsigned long long hs = 0;
    int32_t hf[2] = {0, 0};
    c.d2h(&hs, sum, 1);
    c.d2h(hf, flags, 2);
    c.sync();
    c.free(sum);
    c.free(flags);
    if (hf[0] & 1) throw Error{DHGP_ERR_ARG, "edge weights must be finite and >= 0"};
    W.scale_bits = hf[1];
    W.unit = ldexp(1.0, -hf[1]);
    W.integral = !(hf[0] & 2) && hf[1] <= 62 && hs < (1ull << 53);
    W.wsum = (int64_t)hs;
}

void build_level0(Ctx &c, const DInput &in, DLevel &L) {
    L.N = in.N;
    L.E = in.E;
    L.Ps = in.Ps;
    L.Pd = in.Pd;
    L.src_off = in.src_off;
    L.dst_off = in.dst_off;
    L.src_dat = in.src_dat;
    L.dst_dat = in.dst_dat;
    L.size = in.size;
    L.borrowed = true;
    L.maxp = in.max_edge_pins;
    // Sides in ascending order.  The reference keeps level-0 sides as given
    // but every coarse side is sorted unique (coarsen.py:163-166) and no
    // result depends on the level-0 order; sorted sides
    // let contraction keep an h-edge's gamma image as is whenever no absorbed
    // member sits in it (gamma is increasing on the cluster minima).
    {
        int32_t *tmp = c.alloc<int32_t>(std::max<int64_t>(std::max(in.Ps, in.Pd), 1));
        seg_sort(c, in.E, in.src_off, in.src_dat, nullptr, tmp);
        c.d2d(in.src_dat, tmp, in.Ps);
        seg_sort(c, in.E, in.dst_off, in.dst_dat, nullptr, tmp);
        c.d2d(in.dst_dat, tmp, in.Pd);
        c.free(tmp);
    }
    derive_incidence(c, L);
}

void derive_incidence(Ctx &c, DLevel &L) {
    // algorithmic bytes: the sides read twice (combine, transpose: 8 B per
    // pin slot each), the pin lists written and read back (8 B per pin), the
    // two transposes' outputs (4 B per entry) and the offsets
    KScope ks(c, "incidence", (double)(16.0 * (L.Ps + L.Pd) + 12.0 * L.U + 4.0 * L.Pd + 32.0 * L.E + 16.0 * L.N));
    const int64_t E = L.E;
    // edge_pins = sorted unique (src ∪ dst) per h-edge  (hgraph.py:219-221)
    const int64_t cap = L.Ps + L.Pd;
    int64_t *co = c.alloc<int64_t>(E + 1);
    int32_t *cd = c.alloc<int32_t>(cap);
    int32_t *tmp = c.alloc<int32_t>(cap);
    pdl_launch(k_comb, (unsigned)cdiv(E + 1, 256), 256, 0, c.stream, E, L.src_off, L.src_dat, L.dst_off, L.dst_dat, co, cd);
    DHGP_LAUNCHED(c);
    seg_sort(c, E, co, cd, nullptr, tmp);
    int64_t *cnt = c.alloc<int64_t>(E);
    seg_unique_count(c, E, co, tmp, cnt);
    L.pin_off = c.alloc<int64_t>(E + 1);
    scan_excl<int64_t>(c, cnt, L.pin_off, E);
    c.d2h(&L.U, L.pin_off + E, 1);
    c.sync();
    L.pin_dat = c.alloc<int32_t>(L.U);
    seg_unique_write(c, E, co, tmp, L.pin_off, L.pin_dat);
    c.free(co);
    c.free(cd);
    c.free(tmp);
    c.free(cnt);
    // node_in = transpose(edge_dst), node_inc = transpose(edge_pins)  (hgraph.py:218, 222)
    L.Sin = L.Pd;
    L.in_off = c.alloc<int64_t>((int64_t)L.N + 1);
    L.in_dat = c.alloc<int32_t>(L.Pd);
    transpose_csr(c, E, L.N, L.dst_off, L.dst_dat, L.Pd, L.in_off, L.in_dat);
    L.inc_off = c.alloc<int64_t>((int64_t)L.N + 1);
    L.inc_dat = c.alloc<int32_t>(L.U);
    transpose_csr(c, E, L.N, L.pin_off, L.pin_dat, L.U, L.inc_off, L.inc_dat);
}

void derive_out(Ctx &c, const DLevel &L, int64_t *out_off, int32_t *out_dat) {
    transpose_csr(c, L.E, L.N, L.src_off, L.src_dat, L.Ps, out_off, out_dat);
}

void feasibility(Ctx &c, const DLevel &L, int64_t omega, int64_t delta, int32_t *bad_size, int32_t *bad_in) {
    int32_t *bad = c.alloc<int32_t>(2);
    fill_i32(c, bad, 0x7fffffff, 2);
    if (L.N > 0) {
        pdl_launch(k_feasible, (unsigned)cdiv(L.N, 256), 256, 0, c.stream, L.N, L.size, L.in_off, omega, delta, bad);
        DHGP_LAUNCHED(c);
    }
    int32_t h[2];
    c.d2h(h, bad, 2);
    c.sync();
    c.free(bad);
    *bad_size = h[0] == 0x7fffffff ? -1 : h[0];
    *bad_in = h[1] == 0x7fffffff ? -1 : h[1];
}

void feasibility_input(Ctx &c, const DInput &in, int64_t omega, int64_t delta, int32_t *bad_size, int32_t *bad_in,
                       int32_t *size_val, int32_t *indeg_val) {
    *bad_size = *bad_in = -1;
    if (in.N <= 0) return;
    int32_t *deg = c.alloc<int32_t>((int64_t)in.N + 2);
    int32_t *bad = deg + in.N;
    c.zero(deg, in.N);
    fill_i32(c, bad, 0x7fffffff, 2);
    if (in.Pd > 0) {
        pdl_launch(k_indegree, (unsigned)std::min<int64_t>(cdiv(in.Pd, 256), (int64_t)c.num_sms * 16), 256, 0,
                   c.stream, in.Pd, in.dst_dat, deg);
        DHGP_LAUNCHED(c);
    }
    pdl_launch(k_feasible_deg, (unsigned)cdiv(in.N, 256), 256, 0, c.stream, in.N, in.size, deg, omega, delta, bad);
    DHGP_LAUNCHED(c);
    int32_t h[2];
    c.d2h(h, bad, 2);
    c.sync();
    *bad_size = h[0] == 0x7fffffff ? -1 : h[0];
    *bad_in = h[1] == 0x7fffffff ? -1 : h[1];
    if (*bad_size >= 0) c.d2h(size_val, in.size + *bad_size, 1);
    if (*bad_in >= 0) c.d2h(indeg_val, deg + *bad_in, 1);
    c.sync();
    c.free(deg);
}

}  // namespace dhgp
