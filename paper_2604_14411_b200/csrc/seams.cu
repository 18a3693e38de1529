// seams.cu — data-model entry points (hgraph.py) and the kernel-level seams
// that mirror dhgpart.kernels (kernels.py:58-103) one call each.
//
// The seams take the reference's exact argument lists (explicit neighbour
// sets, candidate order, dense pins matrices) and are written to follow the
// reference's accumulation order, so they are bit-exact for any finite
// non-negative weights.  The production path (driver.cu) uses the fused,
// sparse kernels instead.
#include <mutex>

#include "coarsen.cuh"
#include "prims.cuh"
#include "refine.cuh"

namespace dhgp {
void seams_setup(Ctx &c, int device);
std::recursive_mutex &device_mutex(int device);
}

using namespace dhgp;

namespace {

template <class T>
struct DevBuf {
    Ctx *c = nullptr;
    T *p = nullptr;
    int64_t n = 0;
    DevBuf(Ctx &ctx, int64_t count) : c(&ctx), p(ctx.alloc<T>(count)), n(count) {}
    DevBuf(Ctx &ctx, const T *host, int64_t count) : c(&ctx), p(ctx.alloc<T>(count)), n(count) {
        if (host) ctx.h2d(p, host, count);
    }
    ~DevBuf() {
        try {
            c->free(p);
        } catch (...) {
        }
    }
    void get(T *host) {
        c->d2h(host, p, n);
    }
};

// ---- fill_histograms (_kernels.pyx:47-72): warp per node, incident h-edges in
// ascending order, lanes over the pins of one h-edge (distinct slots) -------
__global__ void k_fill_hist(int32_t N, const int64_t *inc_off, const int32_t *inc_dat, const int64_t *pin_off,
                            const int32_t *pin_dat, const double *w, const int64_t *nbr_off, const int32_t *nbr_dat,
                            double *hist) {
    pdl_entry();
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int lane = lane_id();
    for (int64_t n = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id(); n < N; n += nw) {
        const int64_t lo = nbr_off[n], hi = nbr_off[n + 1];
        if (lo == hi) continue;
        for (int64_t ii = inc_off[n]; ii < inc_off[n + 1]; ii++) {
            const int32_t e = inc_dat[ii];
            const double we = w[e];
            for (int64_t p = pin_off[e] + lane; p < pin_off[e + 1]; p += 32) {
                int64_t j = bsearch_dev(nbr_dat, lo, hi, pin_dat[p]);
                if (j >= 0) hist[j] += we;
            }
            __syncwarp();
        }
    }
}

// ---- select_first_valid (_kernels.pyx:75-103): thread per node ------------
__global__ void k_select_first_valid(int32_t N, const int64_t *order, const int64_t *nbr_off, const int32_t *nbr_dat,
                                     const double *hist, const int32_t *size, const int64_t *in_off,
                                     const int32_t *in_dat, int64_t omega, int64_t delta, int32_t *pair,
                                     double *score) {
    pdl_entry();
    int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    pair[n] = -1;
    score[n] = 0.0;
    for (int64_t t = nbr_off[n]; t < nbr_off[n + 1]; t++) {
        const int64_t pos = order[t];
        const int32_t m = nbr_dat[pos];
        if ((int64_t)size[n] + size[m] > omega) continue;
        int64_t cnt = in_off[n + 1] - in_off[n];
        for (int64_t k = in_off[m]; k < in_off[m + 1]; k++)
            if (bsearch_dev(in_dat, in_off[n], in_off[n + 1], in_dat[k]) < 0) cnt++;
        if (cnt > delta) continue;
        pair[n] = m;
        score[n] = hist[pos];
        break;
    }
}

// ---- connectivity_value (_kernels.pyx:184-213) -----------------------------
__global__ void k_edge_lambda(int32_t E, const int64_t *pin_off, const int32_t *sorted_parts, const double *w,
                              double *contrib) {
    pdl_entry();
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    int64_t lam = 0;
    for (int64_t p = pin_off[e]; p < pin_off[e + 1]; p++) lam += (p == pin_off[e]) || sorted_parts[p] != sorted_parts[p - 1];
    contrib[e] = lam > 0 ? w[e] * (double)(lam - 1) : 0.0;
}
// Sum of x[0..n) equal to the reference's sequential f64 sum in ascending
// order (connectivity_value, _kernels.pyx:199-213).  Every x is a multiple
// of 2^-S for S = the most fractional bits of any element; when
// sum|x| * 2^S < 2^53, every partial sum of any order is an exactly
// representable multiple of 2^-S, so an int64 reduction of x * 2^S in any
// order is bit-identical to the sequential f64 sum.  Pass 1 finds S and
// sum|x|; pass 2 reduces in parallel when that holds, else one thread walks
// the elements in order.
__device__ __forceinline__ int frac_bits(double x) {
    if (x == 0.0 || !isfinite(x)) return 0;
    int e;
    const double m = frexp(fabs(x), &e);  // x = m * 2^e, m in [0.5, 1)
    const unsigned long long mant = (unsigned long long)ldexp(m, 53);
    const int tz = __ffsll((long long)mant) - 1;  // trailing zero bits of the 53-bit mantissa
    const int fb = 53 - tz - e;                     // bits after the binary point
    return fb > 0 ? fb : 0;
}
__global__ void k_sum_probe(int64_t n, const double *x, int *maxbits, double *abssum) {
    pdl_entry();
    int mb = 0;
    double a = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        mb = max(mb, frac_bits(x[i]));
        a += fabs(x[i]);
    }
    for (int o = 16; o; o >>= 1) {
        mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
        a += __shfl_xor_sync(0xffffffffu, a, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(maxbits, mb);
        atomicAdd(abssum, a);
    }
}
__global__ void k_sum_exact(int64_t n, const double *x, const int *maxbits, const double *abssum,
                            unsigned long long *acc, double *out) {
    pdl_entry();
    const int S = *maxbits;
    // margin: the probe's own f64 sum of |x| may round by a relative 2^-40
    const bool parallel = S <= 60 && ldexp(*abssum, S) < 0x1p52;
    if (!parallel) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            double t = 0.0;
            for (int64_t i = 0; i < n; i++) t += x[i];
            *out = t;
        }
        return;
    }
    long long v = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v += (long long)ldexp(x[i], S);
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(acc, (unsigned long long)v);
}
__global__ void k_sum_finish(const int *maxbits, const double *abssum, const unsigned long long *acc, double *out) {
    pdl_entry();
    const int S = *maxbits;
    if (S <= 60 && ldexp(*abssum, S) < 0x1p52) *out = ldexp((double)(long long)*acc, -S);
}
// scratch: 32 bytes
void exact_sum(Ctx &c, int64_t n, const double *x, double *out, void *scratch) {
    int *mb = (int *)scratch;
    double *as = (double *)((char *)scratch + 8);
    unsigned long long *acc = (unsigned long long *)((char *)scratch + 16);
    c.zero((char *)scratch, 24);
    c.zero(out, 1);
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), (int64_t)c.num_sms * 8));
    pdl_launch(k_sum_probe, g, 256, 0, c.stream, n, x, mb, as);
    DHGP_LAUNCHED(c);
    pdl_launch(k_sum_exact, g, 256, 0, c.stream, n, x, mb, as, acc, out);
    DHGP_LAUNCHED(c);
    pdl_launch(k_sum_finish, 1, 32, 0, c.stream, mb, as, acc, out);
    DHGP_LAUNCHED(c);
}

// ---- compute_pins (_kernels.pyx:216-231): thread per h-edge row -----------
__global__ void k_dense_pins(int32_t E, const int64_t *off, const int32_t *dat, const int32_t *assign, int32_t K,
                             int32_t *pins) {
    pdl_entry();
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    for (int64_t p = off[e]; p < off[e + 1]; p++) pins[e * (int64_t)K + assign[dat[p]]]++;
}

// ---- propose_moves (_kernels.pyx:234-311): thread per node ----------------
__global__ void k_node_work(int32_t N, const int64_t *inc_off, const int32_t *inc_dat, const int64_t *pin_off,
                            int64_t *work) {
    pdl_entry();
    int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    int64_t acc = 0;
    for (int64_t i = inc_off[n]; i < inc_off[n + 1]; i++) acc += pin_off[inc_dat[i] + 1] - pin_off[inc_dat[i]];
    work[n] = acc;
}
__global__ void k_propose_dense(int32_t N, const int64_t *inc_off, const int32_t *inc_dat, const int64_t *pin_off,
                                const int32_t *pin_dat, const double *w, const int32_t *pins, int32_t K,
                                const int32_t *assign, const int64_t *psizes, const int32_t *size, int64_t omega,
                                const int64_t *scratch_off, int32_t *cand, double *pres, int32_t *eparts,
                                int32_t *target, double *gain) {
    pdl_entry();
    int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    target[n] = -1;
    gain[n] = 0.0;
    if (inc_off[n + 1] == inc_off[n] || K < 2) return;
    int32_t *cd = cand + scratch_off[n];
    double *pr = pres + scratch_off[n];
    int32_t *ep = eparts + scratch_off[n];
    const int32_t ps = assign[n];
    double saving = 0.0, total = 0.0;
    int64_t nc = 0;
    for (int64_t ii = inc_off[n]; ii < inc_off[n + 1]; ii++) {
        const int32_t e = inc_dat[ii];
        const double we = w[e];
        total += we;
        if (pins[(int64_t)e * K + ps] == 1) saving += we;
        int64_t ne = 0;
        for (int64_t pp = pin_off[e]; pp < pin_off[e + 1]; pp++) {
            const int32_t part = assign[pin_dat[pp]];
            bool seen = false;
            for (int64_t j = 0; j < ne && !seen; j++) seen = ep[j] == part;
            if (!seen) ep[ne++] = part;
        }
        for (int64_t j = 0; j < ne; j++) {
            bool seen = false;
            for (int64_t q = 0; q < nc; q++)
                if (cd[q] == ep[j]) {
                    pr[q] += we;
                    seen = true;
                    break;
                }
            if (!seen) {
                cd[nc] = ep[j];
                pr[nc] = we;
                nc++;
            }
        }
    }
    int32_t best = -1;
    double best_gain = 0.0;
    for (int64_t j = 0; j < nc; j++) {
        const int32_t part = cd[j];
        if (part == ps || psizes[part] + size[n] > omega) continue;
        const double g = saving - (total - pr[j]);
        if (best < 0 || g > best_gain || (g == best_gain && part < best)) {
            best = part;
            best_gain = g;
        }
    }
    if (best >= 0 && best_gain > 0.0) {
        target[n] = best;
        gain[n] = best_gain;
    }
}

// ---- sequence_gains (_kernels.pyx:314-364): thread per move ---------------
__global__ void k_seq_dense(int32_t M, const int64_t *inc_off, const int32_t *inc_dat, const int64_t *pin_off,
                            const int32_t *pin_dat, const double *w, const int32_t *pins, int32_t K,
                            const int32_t *node, const int32_t *from, const int32_t *to, const double *giso,
                            const int64_t *pos, double *out) {
    pdl_entry();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M) return;
    const int32_t n = node[i], ps = from[i], pd = to[i];
    double g = giso[i];
    for (int64_t ii = inc_off[n]; ii < inc_off[n + 1]; ii++) {
        const int32_t e = inc_dat[ii];
        const int64_t base_ps = pins[(int64_t)e * K + ps], base_pd = pins[(int64_t)e * K + pd];
        int64_t leav_pd = 0, ent_pd = 0, leav_ps = 0, ent_ps = 0;
        for (int64_t pp = pin_off[e]; pp < pin_off[e + 1]; pp++) {
            const int64_t j = pos[pin_dat[pp]];
            if (j < 0 || j >= i) continue;
            leav_pd += from[j] == pd;
            ent_pd += to[j] == pd;
            leav_ps += from[j] == ps;
            ent_ps += to[j] == ps;
        }
        double net = 0.0;
        if (base_pd > 0) {
            if (leav_pd - ent_pd == base_pd) net -= w[e];
        } else if (ent_pd > 0) {
            net += w[e];
        }
        if (base_ps == 1) {
            if (ent_ps > 0) net -= w[e];
        } else if (base_ps - 1 > 0 && leav_ps - ent_ps == base_ps - 1) {
            net += w[e];
        }
        g += net;
    }
    out[i] = g;
}

__global__ void k_union_size(const int32_t *a, int64_t na, const int32_t *b, int64_t nb, unsigned long long *out) {
    pdl_entry();
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < nb && bsearch_dev(a, 0, na, b[k]) < 0) atomicAdd(out, 1ull);
}

// ---- neighbours (coarsen.py:78-85): (node, pin) keys, radix-sorted ---------
__global__ void k_nbr_count(int32_t N, const int64_t *inc_off, const int32_t *inc_dat, const int64_t *pin_off,
                            int64_t *cnt) {
    pdl_entry();
    int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    int64_t acc = 0;
    for (int64_t i = inc_off[n]; i < inc_off[n + 1]; i++) acc += pin_off[inc_dat[i] + 1] - pin_off[inc_dat[i]];
    cnt[n] = acc;
}
__global__ void k_nbr_expand(int32_t N, const int64_t *inc_off, const int32_t *inc_dat, const int64_t *pin_off,
                             const int32_t *pin_dat, const int64_t *xoff, uint64_t *keys, uint32_t *vals) {
    pdl_entry();
    int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    int64_t o = xoff[n];
    for (int64_t i = inc_off[n]; i < inc_off[n + 1]; i++) {
        const int32_t e = inc_dat[i];
        for (int64_t p = pin_off[e]; p < pin_off[e + 1]; p++) {
            keys[o] = ((uint64_t)n << 32) | (uint32_t)pin_dat[p];
            vals[o] = 0;
            o++;
        }
    }
}
__global__ void k_nbr_keep(int64_t X, const uint64_t *keys, uint8_t *keep, int64_t *node_cnt) {
    pdl_entry();
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= X) return;
    const uint64_t key = keys[k];
    const uint32_t n = (uint32_t)(key >> 32), m = (uint32_t)key;
    const bool kp = m != n && (k == 0 || keys[k - 1] != key);
    keep[k] = kp;
    if (kp) atomicAdd((unsigned long long *)&node_cnt[n], 1ull);
}
__global__ void k_nbr_write(int64_t X, const uint64_t *keys, const uint8_t *keep, const int64_t *kpos, int32_t *out) {
    pdl_entry();
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < X && keep[k]) out[kpos[k]] = (int32_t)(uint32_t)keys[k];
}

}  // namespace

#define SEAM_BEGIN                           \
    std::lock_guard<std::recursive_mutex> _lk(device_mutex(device));   \
    try {                                    \
        Ctx c;                               \
        seams_setup(c, device);
#define SEAM_END                            \
    c.sync();                               \
    }                                       \
    catch (const Error &e) {                \
        set_error(e.code, e.msg);           \
        return e.code;                      \
    }                                       \
    catch (const std::exception &e) {       \
        set_error(DHGP_ERR_CUDA, e.what()); \
        return DHGP_ERR_CUDA;               \
    }                                       \
    return DHGP_OK;

namespace {
// build_events_and_select (refine.py:178-247) for the seam, as one
// sequential walk in move order: the running per-(part, h-edge) destination
// counts (a working copy of the dense pins_in), the per-part size and
// distinct-inbound values and their violation flags are exactly the groups
// _track_violations forms — every (part, move) group of both tracks sits at
// the move's source or target part, and each part's groups are visited in
// move order.  Then active = cumsum(delta) and the smallest argmax of the
// sequential f64 prefix gain among active == 0 prefixes.
__global__ void k_seam_select(int32_t M, int32_t K, const int64_t *in_off, const int32_t *in_dat,
                              const int32_t *node_size, const int32_t *node, const int32_t *from, const int32_t *to,
                              const double *gain_seq, int32_t *pins_in, int64_t *psize, int64_t *pinb, int64_t omega,
                              int64_t delta, int64_t *active, int64_t *k_out, double *total) {
    pdl_entry();
    if (threadIdx.x || blockIdx.x) return;
    int64_t act = 0;
    active[0] = 0;
    for (int32_t i = 0; i < M; i++) {
        const int32_t n = node[i], f = from[i], t = to[i];
        int64_t tog = 0;
        // size track: (f, i, -size), (t, i, +size)
        const int64_t s = node_size[n];
        {
            const bool b0 = psize[f] > omega, b1 = psize[t] > omega;
            psize[f] -= s;
            psize[t] += s;
            const bool a0 = psize[f] > omega, a1 = psize[t] > omega;
            tog += (a0 != b0 ? (a0 ? 1 : -1) : 0) + (a1 != b1 ? (a1 ? 1 : -1) : 0);
        }
        // inbound track: per inbound h-edge, 1 -> 0 at f and 0 -> 1 at t
        int64_t df = 0, dt = 0;
        for (int64_t j = in_off[n]; j < in_off[n + 1]; j++) {
            const int64_t e = in_dat[j];
            if (--pins_in[e * K + f] == 0) df--;
            if (++pins_in[e * K + t] == 1) dt++;
        }
        {
            const bool b0 = pinb[f] > delta, b1 = pinb[t] > delta;
            pinb[f] += df;
            pinb[t] += dt;
            const bool a0 = pinb[f] > delta, a1 = pinb[t] > delta;
            tog += (a0 != b0 ? (a0 ? 1 : -1) : 0) + (a1 != b1 ? (a1 ? 1 : -1) : 0);
        }
        act += tog;
        active[i + 1] = act;
    }
    double cum = 0.0, best = 0.0;
    int64_t k = 0;  // the empty prefix (active[0] == 0) always competes
    for (int32_t j = 1; j <= M; j++) {
        cum += gain_seq[j - 1];
        if (active[j] == 0 && cum > best) {
            best = cum;
            k = j;
        }
    }
    *k_out = k;
    *total = best;
}

}  // namespace

extern "C" {

int dhgp_incidence(const dhgp_graph *g, int32_t device, int64_t *in_off, int32_t *in_dat, int64_t *out_off,
                   int32_t *out_dat, int64_t *pin_off, int32_t *pin_dat, int64_t *inc_off, int32_t *inc_dat,
                   int64_t *num_pins_out) {
    SEAM_BEGIN
    DInput in;
    upload_input(c, *g, in);
    DLevel L;
    build_level0(c, in, L);
    const int64_t N = L.N, E = L.E;
    if (num_pins_out) *num_pins_out = L.U;
    if (in_off) c.d2h(in_off, L.in_off, N + 1);
    if (in_dat) c.d2h(in_dat, L.in_dat, L.Pd);
    if (pin_off) c.d2h(pin_off, L.pin_off, E + 1);
    if (pin_dat) c.d2h(pin_dat, L.pin_dat, L.U);
    if (inc_off) c.d2h(inc_off, L.inc_off, N + 1);
    if (inc_dat) c.d2h(inc_dat, L.inc_dat, L.U);
    if (out_off || out_dat) {
        int64_t *oo = c.alloc<int64_t>(N + 1);
        int32_t *od = c.alloc<int32_t>(L.Ps);
        derive_out(c, L, oo, od);
        if (out_off) c.d2h(out_off, oo, N + 1);
        if (out_dat) c.d2h(out_dat, od, L.Ps);
        c.sync();
        c.free(oo);
        c.free(od);
    }
    c.sync();
    L.release(c);
    in.release(c);
    SEAM_END
}

int dhgp_neighbors(const dhgp_graph *g, int32_t device, int64_t *nb_off, int32_t **nb_dat, int64_t *nnz_out) {
    SEAM_BEGIN
    DInput in;
    upload_input(c, *g, in);
    DLevel L;
    build_level0(c, in, L);
    const int32_t N = L.N;
    int64_t *cnt = c.alloc<int64_t>(N), *xoff = c.alloc<int64_t>((int64_t)N + 1);
    int64_t X = 0;
    if (N > 0) {
        pdl_launch(k_nbr_count, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, L.inc_off, L.inc_dat, L.pin_off, cnt);
        DHGP_LAUNCHED(c);
    }
    scan_excl<int64_t>(c, cnt, xoff, N);
    c.d2h(&X, xoff + N, 1);
    c.sync();
    uint64_t *k = c.alloc<uint64_t>(X), *kt = c.alloc<uint64_t>(X);
    uint32_t *v = c.alloc<uint32_t>(X), *vt = c.alloc<uint32_t>(X);
    if (N > 0) {
        pdl_launch(k_nbr_expand, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, L.inc_off, L.inc_dat, L.pin_off, L.pin_dat,
                                                                  xoff, k, v);
        DHGP_LAUNCHED(c);
    }
    radix_sort_pairs(c, k, v, kt, vt, X, nullptr, 32 + bitlen((uint64_t)(N > 0 ? N - 1 : 0)));
    uint8_t *keep = c.alloc<uint8_t>(X);
    int64_t *kpos = c.alloc<int64_t>(X + 1);
    c.zero(cnt, N);
    if (X > 0) {
        pdl_launch(k_nbr_keep, (unsigned)cdiv(X, 256), 256, 0, c.stream, X, k, keep, cnt);
        DHGP_LAUNCHED(c);
    }
    scan_excl<uint8_t>(c, keep, kpos, X);
    int64_t nnz = 0;
    c.d2h(&nnz, kpos + X, 1);
    c.sync();
    int32_t *out = c.alloc<int32_t>(nnz);
    if (X > 0) {
        pdl_launch(k_nbr_write, (unsigned)cdiv(X, 256), 256, 0, c.stream, X, k, keep, kpos, out);
        DHGP_LAUNCHED(c);
    }
    scan_excl<int64_t>(c, cnt, xoff, N);
    c.d2h(nb_off, xoff, (int64_t)N + 1);
    int32_t *h = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nnz ? nnz : 1));
    c.d2h(h, out, nnz);
    c.sync();
    *nb_dat = h;
    *nnz_out = nnz;
    for (void *p : {(void *)cnt, (void *)xoff, (void *)k, (void *)kt, (void *)v, (void *)vt, (void *)keep,
                    (void *)kpos, (void *)out})
        c.free(p);
    L.release(c);
    in.release(c);
    SEAM_END
}

int dhgp_check_feasibility(const dhgp_graph *g, int64_t max_size, int64_t max_inbound, int32_t device) {
    SEAM_BEGIN
    if (max_size < 1) throw Error{DHGP_ERR_INFEASIBLE, "max_size must be >= 1, got " + std::to_string(max_size)};
    if (max_inbound < 0)
        throw Error{DHGP_ERR_INFEASIBLE, "max_inbound must be >= 0, got " + std::to_string(max_inbound)};
    DInput in;
    upload_input(c, *g, in);
    DLevel L;
    build_level0(c, in, L);
    int32_t bs = -1, bi = -1;
    if (L.N > 0) feasibility(c, L, max_size, max_inbound, &bs, &bi);
    std::string msg;
    if (bs >= 0) {
        int32_t sz;
        c.d2h(&sz, L.size + bs, 1);
        c.sync();
        msg = "node " + std::to_string(bs) + " has size " + std::to_string(sz) + " > max_size " +
              std::to_string(max_size);
    } else if (bi >= 0) {
        int64_t o[2];
        c.d2h(o, L.in_off + bi, 2);
        c.sync();
        msg = "node " + std::to_string(bi) + " has " + std::to_string(o[1] - o[0]) + " inbound edges > max_inbound " +
              std::to_string(max_inbound);
    }
    L.release(c);
    in.release(c);
    c.sync();
    if (!msg.empty()) throw Error{DHGP_ERR_INFEASIBLE, msg};
    SEAM_END
}

int dhgp_evaluate(const dhgp_graph *g, const int32_t *assign, int32_t num_parts, int32_t device, int64_t *sizes_out,
                  int64_t *inbound_out, double *connectivity_out) {
    SEAM_BEGIN
    DInput in;
    upload_input(c, *g, in);
    DLevel L;
    build_level0(c, in, L);
    DevBuf<int32_t> da(c, assign, L.N);
    DevBuf<int64_t> ds(c, num_parts), di(c, num_parts);
    // per-part sizes and distinct inbound (integer, exact)
    DWeights W;
    W.E = in.E;
    W.w = in.w;
    W.wi = c.alloc<int64_t>(in.E);
    c.zero(W.wi, in.E);
    evaluate_assign(c, L, W, da.p, num_parts, ds.p, di.p, nullptr);
    if (sizes_out) ds.get(sizes_out);
    if (inbound_out) di.get(inbound_out);
    // connectivity with the reference's ascending-edge f64 summation
    if (connectivity_out) {
        int32_t *tmp = c.alloc<int32_t>(L.U);
        double *contrib = c.alloc<double>(L.E), *res = c.alloc<double>(5);
        seg_sort(c, L.E, L.pin_off, L.pin_dat, da.p, tmp);
        if (L.E > 0) {
            pdl_launch(k_edge_lambda, (unsigned)cdiv(L.E, 256), 256, 0, c.stream, L.E, L.pin_off, tmp, in.w, contrib);
            DHGP_LAUNCHED(c);
        }
        exact_sum(c, L.E, contrib, res, res + 1);
        c.d2h(connectivity_out, res, 1);
        c.sync();
        c.free(tmp);
        c.free(contrib);
        c.free(res);
    }
    c.sync();
    W.release(c);
    L.release(c);
    in.release(c);
    SEAM_END
}

int dhgp_union_size_sorted(const int32_t *a, int64_t na, const int32_t *b, int64_t nb, int32_t device, int64_t *out) {
    SEAM_BEGIN
    DevBuf<int32_t> da(c, a, na), db(c, b, nb);
    DevBuf<unsigned long long> r(c, 1);
    c.zero(r.p, 1);
    if (nb > 0) {
        pdl_launch(k_union_size, (unsigned)cdiv(nb, 256), 256, 0, c.stream, da.p, na, db.p, nb, r.p);
        DHGP_LAUNCHED(c);
    }
    unsigned long long h = 0;
    r.get(&h);
    c.sync();
    *out = na + (int64_t)h;
    SEAM_END
}

int dhgp_fill_histograms(int32_t N, const int64_t *inc_off, const int32_t *inc_dat, int32_t E, const int64_t *pin_off,
                         const int32_t *pin_dat, const double *w, const int64_t *nbr_off, const int32_t *nbr_dat,
                         int64_t batch, int32_t device, double *hist) {
    SEAM_BEGIN
    if (batch < 1) throw Error{DHGP_ERR_ARG, "batch_size must be >= 1, got " + std::to_string(batch)};
    DevBuf<int64_t> io(c, inc_off, (int64_t)N + 1), po(c, pin_off, (int64_t)E + 1), no(c, nbr_off, (int64_t)N + 1);
    DevBuf<int32_t> id(c, inc_dat, inc_off[N]), pd(c, pin_dat, pin_off[E]), nd(c, nbr_dat, nbr_off[N]);
    DevBuf<double> dw(c, w, E), dh(c, nbr_off[N]);
    c.zero(dh.p, nbr_off[N]);
    if (N > 0) {
        pdl_launch(k_fill_hist, (unsigned)std::min<int64_t>(cdiv(N, 8), 4096), 256, 0, c.stream, N, io.p, id.p, po.p, pd.p,
                                                                                      dw.p, no.p, nd.p, dh.p);
        DHGP_LAUNCHED(c);
    }
    dh.get(hist);
    SEAM_END
}

int dhgp_select_first_valid(int32_t N, const int64_t *order, const int64_t *nbr_off, const int32_t *nbr_dat,
                            const double *hist, const int32_t *node_size, const int64_t *in_off, const int32_t *in_dat,
                            int64_t max_size, int64_t max_inbound, int32_t device, int32_t *pair, double *score) {
    SEAM_BEGIN
    const int64_t NB = nbr_off[N];
    DevBuf<int64_t> dord(c, order, NB), no(c, nbr_off, (int64_t)N + 1), io(c, in_off, (int64_t)N + 1);
    DevBuf<int32_t> nd(c, nbr_dat, NB), sz(c, node_size, N), id(c, in_dat, in_off[N]), dp(c, N);
    DevBuf<double> dh(c, hist, NB), ds(c, N);
    if (N > 0) {
        pdl_launch(k_select_first_valid, (unsigned)cdiv(N, 128), 128, 0, c.stream, N, dord.p, no.p, nd.p, dh.p, sz.p, io.p,
                                                                          id.p, max_size, max_inbound, dp.p, ds.p);
        DHGP_LAUNCHED(c);
    }
    dp.get(pair);
    ds.get(score);
    SEAM_END
}

int dhgp_resolve_matching(int32_t N, const int32_t *pair, const double *score, int32_t device, int32_t *match) {
    SEAM_BEGIN
    DevBuf<int32_t> dp(c, pair, N), dm(c, N);
    DevBuf<double> ds(c, score, N);
    DevBuf<uint8_t> rep(c, N);
    resolve_matching(c, N, dp.p, ds.p, dm.p, rep.p);
    if (N > 0) dm.get(match);
    SEAM_END
}

int dhgp_connectivity_value(int32_t E, const int64_t *pin_off, const int32_t *pin_dat, const double *w, int32_t N,
                            const int32_t *assign, int32_t device, double *out) {
    SEAM_BEGIN
    DevBuf<int64_t> po(c, pin_off, (int64_t)E + 1);
    DevBuf<int32_t> pd(c, pin_dat, pin_off[E]), da(c, assign, N), tmp(c, pin_off[E]);
    DevBuf<double> dw(c, w, E), contrib(c, E), res(c, 5);
    seg_sort(c, E, po.p, pd.p, da.p, tmp.p);
    if (E > 0) {
        pdl_launch(k_edge_lambda, (unsigned)cdiv(E, 256), 256, 0, c.stream, E, po.p, tmp.p, dw.p, contrib.p);
        DHGP_LAUNCHED(c);
    }
    exact_sum(c, E, contrib.p, res.p, res.p + 1);
    c.d2h(out, res.p, 1);
    SEAM_END
}

int dhgp_compute_pins(int32_t E, const int64_t *pin_off, const int32_t *pin_dat, const int64_t *dst_off,
                      const int32_t *dst_dat, int32_t N, const int32_t *assign, int32_t K, int32_t device, int32_t *pins,
                      int32_t *pins_in) {
    SEAM_BEGIN
    DevBuf<int64_t> po(c, pin_off, (int64_t)E + 1), dof(c, dst_off, (int64_t)E + 1);
    DevBuf<int32_t> pd(c, pin_dat, pin_off[E]), dd(c, dst_dat, dst_off[E]), da(c, assign, N);
    DevBuf<int32_t> dpins(c, (int64_t)E * K), dpin(c, (int64_t)E * K);
    c.zero(dpins.p, (int64_t)E * K);
    c.zero(dpin.p, (int64_t)E * K);
    if (E > 0) {
        pdl_launch(k_dense_pins, (unsigned)cdiv(E, 256), 256, 0, c.stream, E, po.p, pd.p, da.p, K, dpins.p);
        DHGP_LAUNCHED(c);
        pdl_launch(k_dense_pins, (unsigned)cdiv(E, 256), 256, 0, c.stream, E, dof.p, dd.p, da.p, K, dpin.p);
        DHGP_LAUNCHED(c);
    }
    dpins.get(pins);
    dpin.get(pins_in);
    SEAM_END
}

int dhgp_propose_moves(int32_t N, const int64_t *inc_off, const int32_t *inc_dat, int32_t E, const int64_t *pin_off,
                       const int32_t *pin_dat, const double *w, const int32_t *pins, int32_t K, const int32_t *assign,
                       const int64_t *part_sizes, const int32_t *node_size, int64_t max_size, int32_t device,
                       int32_t *target, double *gain) {
    SEAM_BEGIN
    DevBuf<int64_t> io(c, inc_off, (int64_t)N + 1), po(c, pin_off, (int64_t)E + 1), ps(c, part_sizes, K);
    DevBuf<int32_t> id(c, inc_dat, inc_off[N]), pd(c, pin_dat, pin_off[E]), dpins(c, pins, (int64_t)E * K);
    DevBuf<int32_t> da(c, assign, N), sz(c, node_size, N), dt(c, N);
    DevBuf<double> dw(c, w, E), dg(c, N);
    DevBuf<int64_t> work(c, N), woff(c, (int64_t)N + 1);
    if (N > 0) {
        pdl_launch(k_node_work, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, io.p, id.p, po.p, work.p);
        DHGP_LAUNCHED(c);
    }
    scan_excl<int64_t>(c, work.p, woff.p, N);
    int64_t X = 0;
    c.d2h(&X, woff.p + N, 1);
    c.sync();
    DevBuf<int32_t> cand(c, X), ep(c, X);
    DevBuf<double> pres(c, X);
    if (N > 0) {
        pdl_launch(k_propose_dense, (unsigned)cdiv(N, 128), 128, 0, c.stream, N, io.p, id.p, po.p, pd.p, dw.p, dpins.p, K, da.p,
                                                                     ps.p, sz.p, max_size, woff.p, cand.p, pres.p,
                                                                     ep.p, dt.p, dg.p);
        DHGP_LAUNCHED(c);
    }
    dt.get(target);
    dg.get(gain);
    SEAM_END
}

int dhgp_sequence_gains(int32_t N, const int64_t *inc_off, const int32_t *inc_dat, int32_t E, const int64_t *pin_off,
                        const int32_t *pin_dat, const double *w, const int32_t *pins, int32_t K, int32_t M,
                        const int32_t *node, const int32_t *from_part, const int32_t *to_part, const double *gain_iso,
                        const int64_t *pos, int32_t device, double *gain_seq) {
    SEAM_BEGIN
    DevBuf<int64_t> io(c, inc_off, (int64_t)N + 1), po(c, pin_off, (int64_t)E + 1), dpos(c, pos, N);
    DevBuf<int32_t> id(c, inc_dat, inc_off[N]), pd(c, pin_dat, pin_off[E]), dpins(c, pins, (int64_t)E * K);
    DevBuf<int32_t> dn(c, node, M), df(c, from_part, M), dt(c, to_part, M);
    DevBuf<double> dw(c, w, E), dgi(c, gain_iso, M), dgs(c, M);
    if (M > 0) {
        pdl_launch(k_seq_dense, (unsigned)cdiv(M, 128), 128, 0, c.stream, M, io.p, id.p, po.p, pd.p, dw.p, dpins.p, K, dn.p,
                                                                 df.p, dt.p, dgi.p, dpos.p, dgs.p);
        DHGP_LAUNCHED(c);
    }
    dgs.get(gain_seq);
    SEAM_END
}

int dhgp_build_events_and_select(int32_t N, const int64_t *in_off, const int32_t *in_dat, const int32_t *node_size,
                                 int32_t E, int32_t K, int32_t M, const int32_t *node, const int32_t *from_part,
                                 const int32_t *to_part, const double *gain_seq, const int32_t *pins_in,
                                 const int64_t *part_sizes, const int64_t *part_inbound, int64_t max_size,
                                 int64_t max_inbound, int32_t device, int64_t *k_out, double *total_gain_out,
                                 int64_t *active) {
    SEAM_BEGIN
    DevBuf<int64_t> io(c, in_off, (int64_t)N + 1), ps(c, part_sizes, K), pi(c, part_inbound, K);
    DevBuf<int32_t> id(c, in_dat, in_off[N]), ns(c, node_size, N), cnt(c, pins_in, (int64_t)E * K);
    DevBuf<int32_t> dn(c, node, M), df(c, from_part, M), dt(c, to_part, M);
    DevBuf<double> dg(c, gain_seq, M);
    DevBuf<int64_t> act(c, (int64_t)M + 1), res(c, 1);
    DevBuf<double> tot(c, 1);
    pdl_launch(k_seam_select, 1, 1, 0, c.stream, M, K, io.p, id.p, ns.p, dn.p, df.p, dt.p, dg.p, cnt.p, ps.p, pi.p, max_size,
                                         max_inbound, act.p, res.p, tot.p);
    DHGP_LAUNCHED(c);
    act.get(active);
    res.get(k_out);
    tot.get(total_gain_out);
    SEAM_END
}

}  // extern "C"

// ===========================================================================
// The reference-order f64 path (ordered.cuh): device launchers over the seam
// kernels above plus the candidate walk.
// ===========================================================================
#include "ordered.cuh"

namespace dhgp {
namespace ordk {
// warp per node: repeated argmax over the node's neighbour slots in (hist
// desc, id desc) order — the order np.lexsort((-ids, -hist, seg)) gives
// (coarsen.py:118-120) — first one passing the size and inbound-union checks
// (_kernels.pyx:75-103); slots failing a check are marked taken
__global__ void k_ord_select(int32_t N, const int64_t *nb_off, const int32_t *nb_dat, const double *hist,
                             const int32_t *size, const int64_t *in_off, const int32_t *in_dat, int64_t omega,
                             int64_t delta, uint8_t *taken, int32_t *pair, double *score) {
    pdl_entry();
    const int lane = lane_id();
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t n = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id(); n < N; n += nw) {
        const int64_t lo = nb_off[n], hi = nb_off[n + 1];
        const int64_t szn = size[n];
        for (int64_t j = lo + lane; j < hi; j += 32) taken[j] = szn + size[nb_dat[j]] > omega;
        __syncwarp();
        int32_t best_m = -1;
        double best_h = 0.0;
        while (true) {
            double bh = 0.0;
            int32_t bm = -1;
            int64_t bj = -1;
            for (int64_t j = lo + lane; j < hi; j += 32) {
                if (taken[j]) continue;
                const double h = hist[j];
                const int32_t m = nb_dat[j];
                if (bj < 0 || h > bh || (h == bh && m > bm)) {
                    bh = h;
                    bm = m;
                    bj = j;
                }
            }
            for (int d = 16; d > 0; d >>= 1) {
                const double oh = __shfl_xor_sync(FULL_MASK, bh, d);
                const int32_t om = __shfl_xor_sync(FULL_MASK, bm, d);
                const int64_t oj = __shfl_xor_sync(FULL_MASK, bj, d);
                if (oj >= 0 && (bj < 0 || oh > bh || (oh == bh && om > bm))) {
                    bh = oh;
                    bm = om;
                    bj = oj;
                }
            }
            if (bj < 0) break;
            // |in(n) u in(m)| <= delta
            const int64_t nlo = in_off[n], nn = in_off[n + 1] - nlo, mlo = in_off[bm], nm = in_off[bm + 1] - mlo;
            int64_t extra = 0;
            for (int64_t k = lane; k < nm; k += 32) extra += bsearch_dev(in_dat, nlo, nlo + nn, in_dat[mlo + k]) < 0;
            for (int d = 16; d > 0; d >>= 1) extra += __shfl_xor_sync(FULL_MASK, extra, d);
            if (nn + extra <= delta) {
                best_m = bm;
                best_h = bh;
                break;
            }
            if (lane == 0) taken[bj] = 1;
            __syncwarp();
        }
        if (lane == 0) {
            pair[n] = best_m;
            score[n] = best_m >= 0 ? best_h : 0.0;
        }
        __syncwarp();
    }
}
__global__ void k_ord_pinbound(int64_t EK, int32_t K, const int32_t *pins_in, int64_t *pinb) {
    pdl_entry();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < EK; i += (int64_t)gridDim.x * blockDim.x)
        if (pins_in[i] > 0) atomicAdd((unsigned long long *)&pinb[i % K], 1ull);
}
__global__ void k_ord_psizes(int32_t N, const int32_t *assign, const int32_t *size, int64_t *psizes) {
    pdl_entry();
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n < N) atomicAdd((unsigned long long *)&psizes[assign[n]], (unsigned long long)(int64_t)size[n]);
}
__global__ void k_ord_flags(int32_t N, const int32_t *target, uint8_t *flags) {
    pdl_entry();
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n < N) flags[n] = target[n] >= 0;
}
// movers in ascending node order, keyed by descending gain (gains are > 0,
// so the complemented bit pattern orders them): a stable sort by the key
// gives (gain desc, node asc) (refine.py:108-110)
__global__ void k_ord_mover_keys(int32_t N, const uint8_t *flags, const int64_t *mpos, const double *gain,
                                 uint64_t *keys, uint32_t *vals) {
    pdl_entry();
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N || !flags[n]) return;
    keys[mpos[n]] = ~(uint64_t)__double_as_longlong(gain[n]);
    vals[mpos[n]] = (uint32_t)n;
}
__global__ void k_ord_moves(int64_t M, const uint32_t *vals, const int32_t *assign, const int32_t *target,
                            const double *gain, int32_t *node, int32_t *from, int32_t *to, double *giso,
                            int64_t *pos) {
    pdl_entry();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M) return;
    const int32_t n = (int32_t)vals[i];
    node[i] = n;
    from[i] = assign[n];
    to[i] = target[n];
    giso[i] = gain[n];
    pos[n] = i;
}
__global__ void k_ord_apply(int64_t k, const int32_t *node, const int32_t *to, int32_t *assign) {
    pdl_entry();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < k) assign[node[i]] = to[i];
}
__global__ void k_ord_project(int32_t N, const int32_t *gamma, const int32_t *coarse, int32_t *fine) {
    pdl_entry();
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < N) fine[v] = coarse[gamma[v]];
}
}  // namespace ordk
using namespace ordk;

void ord_neighbors(Ctx &c, const DLevel &L, int64_t **nb_off, int32_t **nb_dat, int64_t *nnz_out) {
    const int32_t N = L.N;
    int64_t *cnt = c.alloc<int64_t>(N), *xoff = c.alloc<int64_t>((int64_t)N + 1);
    int64_t X = 0;
    if (N > 0) {
        pdl_launch(k_nbr_count, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, L.inc_off, L.inc_dat, L.pin_off, cnt);
        DHGP_LAUNCHED(c);
    }
    scan_excl<int64_t>(c, cnt, xoff, N);
    c.d2h(&X, xoff + N, 1);
    c.sync();
    uint64_t *k = c.alloc<uint64_t>(X), *kt = c.alloc<uint64_t>(X);
    uint32_t *v = c.alloc<uint32_t>(X), *vt = c.alloc<uint32_t>(X);
    if (N > 0) {
        pdl_launch(k_nbr_expand, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, L.inc_off, L.inc_dat, L.pin_off,
                   L.pin_dat, xoff, k, v);
        DHGP_LAUNCHED(c);
    }
    radix_sort_pairs(c, k, v, kt, vt, X, nullptr, 32 + bitlen((uint64_t)(N > 0 ? N - 1 : 0)));
    uint8_t *keep = c.alloc<uint8_t>(X);
    int64_t *kpos = c.alloc<int64_t>(X + 1);
    c.zero(cnt, N);
    if (X > 0) {
        pdl_launch(k_nbr_keep, (unsigned)cdiv(X, 256), 256, 0, c.stream, X, k, keep, cnt);
        DHGP_LAUNCHED(c);
    }
    scan_excl<uint8_t>(c, keep, kpos, X);
    int64_t nnz = 0;
    c.d2h(&nnz, kpos + X, 1);
    c.sync();
    int32_t *out = c.alloc<int32_t>(std::max<int64_t>(nnz, 1));
    if (X > 0) {
        pdl_launch(k_nbr_write, (unsigned)cdiv(X, 256), 256, 0, c.stream, X, k, keep, kpos, out);
        DHGP_LAUNCHED(c);
    }
    scan_excl<int64_t>(c, cnt, xoff, N);
    for (void *p : {(void *)cnt, (void *)k, (void *)kt, (void *)v, (void *)vt, (void *)keep, (void *)kpos}) c.free(p);
    *nb_off = xoff;
    *nb_dat = out;
    *nnz_out = nnz;
}

void ord_fill_hist(Ctx &c, const DLevel &L, const double *w, const int64_t *nb_off, const int32_t *nb_dat,
                   double *hist) {
    int64_t nnz = 0;
    c.d2h(&nnz, nb_off + L.N, 1);
    c.sync();
    c.zero(hist, nnz);
    if (L.N > 0) {
        pdl_launch(k_fill_hist, (unsigned)std::min<int64_t>(cdiv(L.N, 8), (int64_t)c.num_sms * 16), 256, 0, c.stream,
                   L.N, L.inc_off, L.inc_dat, L.pin_off, L.pin_dat, w, nb_off, nb_dat, hist);
        DHGP_LAUNCHED(c);
    }
}

void ord_select(Ctx &c, const DLevel &L, const int64_t *nb_off, const int32_t *nb_dat, const double *hist,
                int64_t nnz, int64_t omega, int64_t delta, int32_t *pair, double *score) {
    if (L.N == 0) return;
    uint8_t *taken = c.alloc<uint8_t>(std::max<int64_t>(nnz, 1));
    pdl_launch(k_ord_select, (unsigned)std::min<int64_t>(cdiv(L.N, 8), (int64_t)c.num_sms * 16), 256, 0, c.stream,
               L.N, nb_off, nb_dat, hist, L.size, L.in_off, L.in_dat, omega, delta, taken, pair, score);
    DHGP_LAUNCHED(c);
    c.free(taken);
}

void ord_dense_pins(Ctx &c, const DLevel &L, const int32_t *assign, int32_t K, int32_t *pins, int32_t *pins_in) {
    c.zero(pins, (int64_t)L.E * K);
    c.zero(pins_in, (int64_t)L.E * K);
    if (L.E > 0) {
        pdl_launch(k_dense_pins, (unsigned)cdiv(L.E, 256), 256, 0, c.stream, L.E, L.pin_off, L.pin_dat, assign, K, pins);
        DHGP_LAUNCHED(c);
        pdl_launch(k_dense_pins, (unsigned)cdiv(L.E, 256), 256, 0, c.stream, L.E, L.dst_off, L.dst_dat, assign, K,
                   pins_in);
        DHGP_LAUNCHED(c);
    }
}

void ord_propose(Ctx &c, const DLevel &L, const double *w, const int32_t *pins, int32_t K, const int32_t *assign,
                 const int64_t *psizes, int64_t omega, int32_t *target, double *gain) {
    const int32_t N = L.N;
    if (N == 0) return;
    int64_t *work = c.alloc<int64_t>(N), *woff = c.alloc<int64_t>((int64_t)N + 1);
    pdl_launch(k_node_work, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, L.inc_off, L.inc_dat, L.pin_off, work);
    DHGP_LAUNCHED(c);
    scan_excl<int64_t>(c, work, woff, N);
    int64_t X = 0;
    c.d2h(&X, woff + N, 1);
    c.sync();
    int32_t *cand = c.alloc<int32_t>(std::max<int64_t>(X, 1)), *ep = c.alloc<int32_t>(std::max<int64_t>(X, 1));
    double *pres = c.alloc<double>(std::max<int64_t>(X, 1));
    pdl_launch(k_propose_dense, (unsigned)cdiv(N, 128), 128, 0, c.stream, N, L.inc_off, L.inc_dat, L.pin_off,
               L.pin_dat, w, pins, K, assign, psizes, L.size, omega, woff, cand, pres, ep, target, gain);
    DHGP_LAUNCHED(c);
    for (void *p : {(void *)work, (void *)woff, (void *)cand, (void *)ep, (void *)pres}) c.free(p);
}

void ord_seq_gains(Ctx &c, const DLevel &L, const double *w, const int32_t *pins, int32_t K, int32_t M,
                   const int32_t *node, const int32_t *from, const int32_t *to, const double *giso,
                   const int64_t *pos, double *gseq) {
    if (M <= 0) return;
    pdl_launch(k_seq_dense, (unsigned)cdiv(M, 128), 128, 0, c.stream, M, L.inc_off, L.inc_dat, L.pin_off, L.pin_dat,
               w, pins, K, node, from, to, giso, pos, gseq);
    DHGP_LAUNCHED(c);
}

void ord_pinbound(Ctx &c, int32_t E, int32_t K, const int32_t *pins_in, int64_t *pinb) {
    c.zero(pinb, K);
    const int64_t EK = (int64_t)E * K;
    if (EK > 0) {
        pdl_launch(k_ord_pinbound, (unsigned)std::min<int64_t>(cdiv(EK, 256), (int64_t)c.num_sms * 32), 256, 0,
                   c.stream, EK, K, pins_in, pinb);
        DHGP_LAUNCHED(c);
    }
}

void ord_select_prefix(Ctx &c, const DLevel &L, int32_t K, int32_t M, const int32_t *node, const int32_t *from,
                       const int32_t *to, const double *gseq, int32_t *pins_in, int64_t *psizes, int64_t *pinb,
                       int64_t omega, int64_t delta, int64_t *active, int64_t *k_out, double *total) {
    pdl_launch(k_seam_select, 1, 1, 0, c.stream, M, K, L.in_off, L.in_dat, L.size, node, from, to, gseq, pins_in,
               psizes, pinb, omega, delta, active, k_out, total);
    DHGP_LAUNCHED(c);
}

double ord_connectivity(Ctx &c, const DLevel &L, const double *w, const int32_t *assign) {
    int32_t *tmp = c.alloc<int32_t>(std::max<int64_t>(L.U, 1));
    double *contrib = c.alloc<double>(std::max<int64_t>(L.E, 1)), *res = c.alloc<double>(5);
    seg_sort(c, L.E, L.pin_off, L.pin_dat, assign, tmp);
    if (L.E > 0) {
        pdl_launch(k_edge_lambda, (unsigned)cdiv(L.E, 256), 256, 0, c.stream, L.E, L.pin_off, tmp, w, contrib);
        DHGP_LAUNCHED(c);
    }
    exact_sum(c, L.E, contrib, res, res + 1);
    double h = 0.0;
    c.d2h(&h, res, 1);
    c.sync();
    c.free(tmp);
    c.free(contrib);
    c.free(res);
    return h;
}

void ord_score(Ctx &c, const DLevel &L, const double *w, int64_t omega, int64_t delta, int32_t *pair,
               double *score) {
    int64_t *nbo = nullptr, nnz = 0;
    int32_t *nbd = nullptr;
    ord_neighbors(c, L, &nbo, &nbd, &nnz);
    double *hist = c.alloc<double>(std::max<int64_t>(nnz, 1));
    ord_fill_hist(c, L, w, nbo, nbd, hist);
    ord_select(c, L, nbo, nbd, hist, nnz, omega, delta, pair, score);
    c.free(hist);
    c.free(nbo);
    c.free(nbd);
}

void ord_project(Ctx &c, int32_t N, const int32_t *gamma, const int32_t *coarse, int32_t *fine) {
    if (N > 0) {
        pdl_launch(k_ord_project, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, gamma, coarse, fine);
        DHGP_LAUNCHED(c);
    }
}

void ord_refine_level(Ctx &c, const DLevel &L, const double *w, int32_t *assign, int32_t K, int64_t omega,
                      int64_t delta, int32_t max_rounds, int32_t level, std::vector<double> &conns,
                      const RoundObserver *obs) {
    const int32_t N = L.N, E = L.E;
    const int64_t EK = (int64_t)E * K;
    int32_t *pins = c.alloc<int32_t>(std::max<int64_t>(EK, 1)), *pins_in = c.alloc<int32_t>(std::max<int64_t>(EK, 1));
    int64_t *psizes = c.alloc<int64_t>(std::max(K, 1)), *pinb = c.alloc<int64_t>(std::max(K, 1));
    int32_t *target = c.alloc<int32_t>(std::max(N, 1)), *node = c.alloc<int32_t>(std::max(N, 1));
    int32_t *from = c.alloc<int32_t>(std::max(N, 1)), *to = c.alloc<int32_t>(std::max(N, 1));
    double *gain = c.alloc<double>(std::max(N, 1)), *giso = c.alloc<double>(std::max(N, 1));
    double *gseq = c.alloc<double>(std::max(N, 1)), *tot = c.alloc<double>(1);
    uint8_t *flags = c.alloc<uint8_t>(std::max(N, 1));
    int64_t *mpos = c.alloc<int64_t>((int64_t)N + 1), *pos = c.alloc<int64_t>(std::max(N, 1));
    int64_t *active = c.alloc<int64_t>((int64_t)N + 1), *kd = c.alloc<int64_t>(1);
    uint64_t *mk = c.alloc<uint64_t>(std::max(N, 1)), *mkt = c.alloc<uint64_t>(std::max(N, 1));
    uint32_t *mv = c.alloc<uint32_t>(std::max(N, 1)), *mvt = c.alloc<uint32_t>(std::max(N, 1));
    conns.push_back(ord_connectivity(c, L, w, assign));
    for (int32_t rnd = 0; rnd < max_rounds; rnd++) {
        ord_dense_pins(c, L, assign, K, pins, pins_in);
        c.zero(psizes, K);
        if (N > 0) {
            pdl_launch(k_ord_psizes, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, assign, L.size, psizes);
            DHGP_LAUNCHED(c);
        }
        ord_propose(c, L, w, pins, K, assign, psizes, omega, target, gain);
        int64_t M = 0;
        if (N > 0) {
            pdl_launch(k_ord_flags, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, target, flags);
            DHGP_LAUNCHED(c);
            scan_excl<uint8_t>(c, flags, mpos, N);
            c.d2h(&M, mpos + N, 1);
            c.sync();
        }
        if (M == 0) break;
        pdl_launch(k_ord_mover_keys, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, flags, mpos, gain, mk, mv);
        DHGP_LAUNCHED(c);
        radix_sort_pairs(c, mk, mv, mkt, mvt, M, nullptr, 64);
        fill_i64(c, pos, -1, N);
        pdl_launch(k_ord_moves, (unsigned)cdiv(M, 256), 256, 0, c.stream, M, mv, assign, target, gain, node, from, to,
                   giso, pos);
        DHGP_LAUNCHED(c);
        ord_seq_gains(c, L, w, pins, K, (int32_t)M, node, from, to, giso, pos, gseq);
        ord_pinbound(c, E, K, pins_in, pinb);
        ord_select_prefix(c, L, K, (int32_t)M, node, from, to, gseq, pins_in, psizes, pinb, omega, delta, active, kd,
                          tot);
        int64_t k = 0;
        double total = 0.0;
        c.d2h(&k, kd, 1);
        c.d2h(&total, tot, 1);
        c.sync();
        if (obs && *obs) {
            RoundRecord rec;
            rec.level = level;
            rec.round = rnd;
            rec.num_parts = K;
            rec.k = (int32_t)k;
            rec.total_gain = total;
            rec.assign.resize(N);
            rec.node.resize(M);
            rec.from.resize(M);
            rec.to.resize(M);
            rec.gain_iso.resize(M);
            rec.gain_seq.resize(M);
            rec.active.resize(M + 1);
            c.d2h(rec.assign.data(), assign, N);
            c.d2h(rec.node.data(), node, M);
            c.d2h(rec.from.data(), from, M);
            c.d2h(rec.to.data(), to, M);
            c.d2h(rec.gain_iso.data(), giso, M);
            c.d2h(rec.gain_seq.data(), gseq, M);
            c.d2h(rec.active.data(), active, M + 1);
            c.sync();
            (*obs)(rec);
        }
        if (k == 0) break;
        pdl_launch(k_ord_apply, (unsigned)cdiv(k, 256), 256, 0, c.stream, k, node, to, assign);
        DHGP_LAUNCHED(c);
        conns.push_back(ord_connectivity(c, L, w, assign));
    }
    for (void *p : {(void *)pins, (void *)pins_in, (void *)psizes, (void *)pinb, (void *)target, (void *)node,
                    (void *)from, (void *)to, (void *)gain, (void *)giso, (void *)gseq, (void *)tot, (void *)flags,
                    (void *)mpos, (void *)pos, (void *)active, (void *)kd, (void *)mk, (void *)mkt, (void *)mv,
                    (void *)mvt})
        c.free(p);
}

}  // namespace dhgp
