// parse.cu — the `.dhg` text format on the GPU (hgraph.parse_dhg,
// hgraph.py:409-467).
//
// The file's edge lines are byte work: the newline positions are found by a
// count / scan / write pass over the text, then one warp per line classifies
// its bytes, finds its tokens with ballots and parses them (each lane parses
// the tokens that start in its byte).  Lines whose tokens are all unsigned
// decimal integers are handled entirely on the device ("fast" lines); the
// rare others (signs, decimal points, exponents, underscores, non-ASCII, very
// long literals) are listed for the host, which parses exactly those lines
// with the reference's own rules and hands back their counts and ids.  Every
// failing line is flagged; the host reports the first one with the
// reference's message (it re-derives the message from that single line).
#include <algorithm>

#include "prims.cuh"

namespace dhgp {
namespace {

constexpr int NL_THREADS = 256;
constexpr int NL_BYTES = 32;  // bytes per thread
constexpr int NL_TILE = NL_THREADS * NL_BYTES;

__global__ void k_nl_count(const char *text, int64_t len, int64_t *counts) {
    pdl_entry();
    __shared__ int64_t sh[33];
    const int64_t base = (int64_t)blockIdx.x * NL_TILE + (int64_t)threadIdx.x * NL_BYTES;
    int64_t c = 0;
    for (int i = 0; i < NL_BYTES; i++) {
        const int64_t p = base + i;
        if (p < len && text[p] == '\n') c++;
    }
    const int64_t t = block_sum<int64_t>(c, sh);
    if (threadIdx.x == 0) counts[blockIdx.x] = t;
}

// line_start[0] = 0; line_start[k + 1] = (position of the k-th newline) + 1
__global__ void k_nl_write(const char *text, int64_t len, const int64_t *block_off, int64_t *line_start) {
    pdl_entry();
    __shared__ int64_t sh[33];
    const int64_t base = (int64_t)blockIdx.x * NL_TILE + (int64_t)threadIdx.x * NL_BYTES;
    int64_t c = 0;
    for (int i = 0; i < NL_BYTES; i++) {
        const int64_t p = base + i;
        if (p < len && text[p] == '\n') c++;
    }
    // block exclusive scan of the per-thread counts
    const int lane = lane_id(), w = warp_id();
    int64_t incl = warp_incl_scan(c);
    if (lane == 31) sh[w] = incl;
    __syncthreads();
    if (w == 0) {
        const int nw = NL_THREADS / 32;
        int64_t x = lane < nw ? sh[lane] : 0;
        int64_t xi = warp_incl_scan(x);
        if (lane < nw) sh[lane] = xi - x;
    }
    __syncthreads();
    int64_t k = block_off[blockIdx.x] + incl - c + sh[w];
    for (int i = 0; i < NL_BYTES; i++) {
        const int64_t p = base + i;
        if (p < len && text[p] == '\n') line_start[1 + k++] = p + 1;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) line_start[0] = 0;
}

__device__ __forceinline__ bool is_ws(unsigned char c) {
    // str.split() separators within the ASCII range
    return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1f);
}
__device__ __forceinline__ bool is_digit(unsigned char c) { return c >= '0' && c <= '9'; }

constexpr uint64_t kSat = 1ull << 60;
// unsigned decimal at p (digits up to the next separator), saturating
__device__ __forceinline__ uint64_t parse_uint(const char *text, int64_t p, int64_t end) {
    uint64_t v = 0;
    while (p < end && is_digit((unsigned char)text[p])) {
        v = v * 10 + (uint64_t)(text[p] - '0');
        if (v > kSat) v = kSat;
        p++;
    }
    return v;
}

// per-line status
constexpr uint8_t LN_OK = 0, LN_SLOW = 1, LN_ERR = 2;

// Warp per line: token count, the first three tokens, slow / error status.
__global__ void k_line_pass1(const char *text, const int64_t *line_start, int64_t E, double *w, int64_t *ks,
                             int64_t *kd, uint8_t *status, int64_t *slow_idx, unsigned long long *nslow) {
    pdl_entry();
    const int lane = lane_id();
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t e = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id(); e < E; e += nw) {
        const int64_t lo = line_start[e], hi = line_start[e + 1] - 1;  // excluding '\n'
        int64_t ntok = 0;
        bool slow = false;
        uint64_t v0 = 0, v1 = 0, v2 = 0;
        for (int64_t b = lo; b < hi; b += 32) {
            const int64_t p = b + lane;
            unsigned char ch = p < hi ? (unsigned char)text[p] : ' ';
            unsigned char prev = p - 1 >= lo ? (unsigned char)text[p - 1] : ' ';
            const bool ws = is_ws(ch);
            if (!ws && !is_digit(ch)) slow = true;
            const bool start = !ws && is_ws(prev);
            const uint32_t bal = __ballot_sync(FULL_MASK, start);
            if (start) {
                const int64_t t = ntok + __popc(bal & lt);
                if (t < 3) {
                    // saturating value of this token (the weight must stay exact in f64)
                    int64_t q = p;
                    while (q < hi && !is_ws((unsigned char)text[q])) q++;
                    const uint64_t v = parse_uint(text, p, q);
                    if (t == 0) v0 = v;
                    if (t == 1) v1 = v;
                    if (t == 2) v2 = v;
                }
            }
            ntok += __popc(bal);
        }
        slow = __any_sync(FULL_MASK, slow);
        // the owners of tokens 0-2 sit on different lanes: combine (max; others hold 0)
        for (int d = 16; d > 0; d >>= 1) {
            v0 = max(v0, (uint64_t)__shfl_xor_sync(FULL_MASK, v0, d));
            v1 = max(v1, (uint64_t)__shfl_xor_sync(FULL_MASK, v1, d));
            v2 = max(v2, (uint64_t)__shfl_xor_sync(FULL_MASK, v2, d));
        }
        if (lane == 0) {
            uint8_t st = LN_OK;
            int64_t a = 0, c = 0;
            if (!slow && ntok >= 3 && (v0 >= (1ull << 53) || v1 >= (1ull << 31) || v2 >= (1ull << 31))) slow = true;
            if (slow) {
                st = LN_SLOW;
                slow_idx[atomicAdd(nslow, 1ull)] = e;
            } else if (ntok < 3 || v1 + v2 < 1 || ntok != 3 + (int64_t)(v1 + v2)) {
                st = LN_ERR;
            } else {
                a = (int64_t)v1;
                c = (int64_t)v2;
                w[e] = (double)v0;  // exact: v0 < 2^53
            }
            status[e] = st;
            ks[e] = a;
            kd[e] = c;
        }
    }
}

// Warp per fast line: pin ids into their slots; out-of-range ids flag the line.
__global__ void k_line_pass2(const char *text, const int64_t *line_start, int64_t E, int64_t num_nodes,
                             const uint8_t *status, const int64_t *ks, const int64_t *src_off, const int64_t *dst_off,
                             int32_t *src_dat, int32_t *dst_dat, uint8_t *bad) {
    pdl_entry();
    const int lane = lane_id();
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t e = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id(); e < E; e += nw) {
        if (status[e] != LN_OK) continue;
        const int64_t lo = line_start[e], hi = line_start[e + 1] - 1;
        const int64_t k_src = ks[e];
        bool oor = false;
        int64_t ntok = 0;
        for (int64_t b = lo; b < hi; b += 32) {
            const int64_t p = b + lane;
            unsigned char ch = p < hi ? (unsigned char)text[p] : ' ';
            unsigned char prev = p - 1 >= lo ? (unsigned char)text[p - 1] : ' ';
            const bool start = !is_ws(ch) && is_ws(prev);
            const uint32_t bal = __ballot_sync(FULL_MASK, start);
            if (start) {
                const int64_t t = ntok + __popc(bal & lt);
                if (t >= 3) {
                    int64_t q = p;
                    while (q < hi && !is_ws((unsigned char)text[q])) q++;
                    const uint64_t v = parse_uint(text, p, q);
                    if (v >= (uint64_t)num_nodes) oor = true;
                    const int32_t id = v >= (uint64_t)num_nodes ? -1 : (int32_t)v;
                    const int64_t j = t - 3;
                    if (j < k_src)
                        src_dat[src_off[e] + j] = id;
                    else
                        dst_dat[dst_off[e] + (j - k_src)] = id;
                }
            }
            ntok += __popc(bal);
        }
        if (__any_sync(FULL_MASK, oor) && lane == 0) bad[e] = 1;
    }
}

// host-parsed lines: counts in, then their ids scattered into place
__global__ void k_slow_counts(int64_t nslow, const int64_t *slow_idx, const int64_t *sks, const int64_t *skd,
                              const double *sw, const uint8_t *serr, int64_t *ks, int64_t *kd, double *w,
                              uint8_t *bad) {
    pdl_entry();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nslow) return;
    const int64_t e = slow_idx[i];
    ks[e] = sks[i];
    kd[e] = skd[i];
    w[e] = sw[i];
    if (serr[i]) bad[e] = 1;
}
__global__ void k_slow_ids(int64_t nslow, const int64_t *slow_idx, const int64_t *ids_off, const int32_t *ids,
                           const int64_t *ks, const int64_t *src_off, const int64_t *dst_off, int32_t *src_dat,
                           int32_t *dst_dat) {
    pdl_entry();
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id(); i < nslow; i += nw) {
        const int64_t e = slow_idx[i];
        const int64_t a = ks[e];
        for (int64_t j = ids_off[i] + lane_id(); j < ids_off[i + 1]; j += 32) {
            const int64_t k = j - ids_off[i];
            if (k < a)
                src_dat[src_off[e] + k] = ids[j];
            else
                dst_dat[dst_off[e] + (k - a)] = ids[j];
        }
    }
}

__global__ void k_err_flags(int64_t E, const uint8_t *status, uint8_t *bad) {
    pdl_entry();
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < E && status[e] == LN_ERR) bad[e] = 1;
}
// a repeated id within one side: adjacent equal values of the sorted side
__global__ void k_dup_flags(int64_t E, const int64_t *off, const int32_t *sorted, uint8_t *bad) {
    pdl_entry();
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    for (int64_t p = off[e] + 1; p < off[e + 1]; p++)
        if (sorted[p] == sorted[p - 1]) {
            bad[e] = 1;
            return;
        }
}
__global__ void k_first_bad(int64_t E, const uint8_t *bad, unsigned long long *first) {
    pdl_entry();
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < E && bad[e]) atomicMin(first, (unsigned long long)e);
}

}  // namespace
}  // namespace dhgp

using namespace dhgp;

struct dhgp_parse {
    int device = 0;
    int64_t E = 0, len = 0, N = 0;
    char *text = nullptr;
    int64_t *line_start = nullptr, *ks = nullptr, *kd = nullptr, *slow_idx = nullptr;
    double *w = nullptr;
    uint8_t *status = nullptr, *bad = nullptr;
    unsigned long long *nslow = nullptr;
    int64_t *src_off = nullptr, *dst_off = nullptr;
    int32_t *src_dat = nullptr, *dst_dat = nullptr;
    int64_t nsrc = 0, ndst = 0, hslow = 0;
    void release(Ctx &c) {
        for (void *p : {(void *)text, (void *)line_start, (void *)ks, (void *)kd, (void *)slow_idx, (void *)w,
                        (void *)status, (void *)bad, (void *)nslow, (void *)src_off, (void *)dst_off, (void *)src_dat,
                        (void *)dst_dat})
            c.free(p);
    }
};

namespace dhgp {
void seams_setup(Ctx &c, int device);
}

#define PARSE_GUARD_BEGIN \
    try {
#define PARSE_GUARD_END                     \
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

extern "C" {

int dhgp_parse_dhg_begin(const char *text, int64_t len, int64_t num_edges, int64_t num_nodes, int32_t device,
                         dhgp_parse **out, int64_t *lines_found, int64_t *num_slow) {
    PARSE_GUARD_BEGIN
    if (!text || len < 0 || num_edges < 0 || num_nodes < 0 || num_nodes > INT32_MAX || !out)
        throw Error{DHGP_ERR_ARG, "bad parse arguments"};
    Ctx c;
    seams_setup(c, device);
    dhgp_parse *ps = new dhgp_parse();
    ps->device = device;
    ps->len = len;
    ps->N = num_nodes;
    *out = ps;
    ps->text = c.alloc<char>(len + 1);
    c.h2d(ps->text, text, len);
    const int64_t nb = std::max<int64_t>(1, cdiv(len, NL_TILE));
    int64_t *counts = c.alloc<int64_t>(nb), *boff = c.alloc<int64_t>(nb + 1);
    pdl_launch(k_nl_count, (unsigned)nb, NL_THREADS, 0, c.stream, ps->text, len, counts);
    DHGP_LAUNCHED(c);
    scan_excl<int64_t>(c, counts, boff, nb);
    int64_t nl = 0;
    c.d2h(&nl, boff + nb, 1);
    c.sync();
    *lines_found = nl + 1;  // str.split("\n") semantics
    *num_slow = 0;
    if (nl + 1 != num_edges) {  // the caller reports the count mismatch
        c.free(counts);
        c.free(boff);
        c.sync();
        return DHGP_OK;
    }
    const int64_t E = num_edges;
    ps->E = E;
    ps->line_start = c.alloc<int64_t>(E + 1);
    pdl_launch(k_nl_write, (unsigned)nb, NL_THREADS, 0, c.stream, ps->text, len, boff, ps->line_start);
    DHGP_LAUNCHED(c);
    // sentinel: the last line ends at len (as if followed by '\n')
    const int64_t endp = len + 1;
    c.h2d(ps->line_start + E, &endp, 1);
    ps->w = c.alloc<double>(E);
    ps->ks = c.alloc<int64_t>(E);
    ps->kd = c.alloc<int64_t>(E);
    ps->status = c.alloc<uint8_t>(E);
    ps->bad = c.alloc<uint8_t>(E);
    ps->slow_idx = c.alloc<int64_t>(E);
    ps->nslow = c.alloc<unsigned long long>(1);
    c.zero(ps->bad, E);
    c.zero(ps->nslow, 1);
    c.zero(ps->w, E);
    if (E > 0) {
        const int blocks = (int)std::min<int64_t>(cdiv(E, 8), (int64_t)c.num_sms * 16);
        pdl_launch(k_line_pass1, blocks, 256, 0, c.stream, ps->text, ps->line_start, E, ps->w, ps->ks, ps->kd, ps->status,
                                                   ps->slow_idx, ps->nslow);
        DHGP_LAUNCHED(c);
    }
    unsigned long long ns = 0;
    c.d2h(&ns, ps->nslow, 1);
    c.sync();
    ps->hslow = (int64_t)ns;
    *num_slow = (int64_t)ns;
    // slow lines in ascending order (the host parses them in file order)
    if (ns > 1) {
        std::vector<int64_t> h(ns);
        c.d2h(h.data(), ps->slow_idx, (int64_t)ns);
        c.sync();
        std::sort(h.begin(), h.end());
        c.h2d(ps->slow_idx, h.data(), (int64_t)ns);
    }
    c.free(counts);
    c.free(boff);
    c.sync();
    PARSE_GUARD_END
}

int dhgp_parse_dhg_slow_lines(dhgp_parse *ps, int64_t *idx, int64_t *byte_lo, int64_t *byte_hi) {
    PARSE_GUARD_BEGIN
    Ctx c;
    seams_setup(c, ps->device);
    const int64_t n = ps->hslow;
    if (n == 0) return DHGP_OK;
    c.d2h(idx, ps->slow_idx, n);
    c.sync();
    for (int64_t i = 0; i < n; i++) {
        int64_t b[2];
        c.d2h(b, ps->line_start + idx[i], 2);
        c.sync();
        byte_lo[i] = b[0];
        byte_hi[i] = b[1] - 1;
    }
    PARSE_GUARD_END
}

int dhgp_parse_dhg_finish(dhgp_parse *ps, const int64_t *slow_ks, const int64_t *slow_kd, const double *slow_w,
                          const uint8_t *slow_err, const int64_t *slow_ids_off, const int32_t *slow_ids,
                          int64_t *first_bad_line, int64_t *nsrc, int64_t *ndst) {
    PARSE_GUARD_BEGIN
    Ctx c;
    seams_setup(c, ps->device);
    const int64_t E = ps->E, ns = ps->hslow;
    if (ns > 0) {
        int64_t *dks = c.alloc<int64_t>(ns), *dkd = c.alloc<int64_t>(ns);
        double *dw = c.alloc<double>(ns);
        uint8_t *de = c.alloc<uint8_t>(ns);
        c.h2d(dks, slow_ks, ns);
        c.h2d(dkd, slow_kd, ns);
        c.h2d(dw, slow_w, ns);
        c.h2d(de, slow_err, ns);
        pdl_launch(k_slow_counts, (unsigned)cdiv(ns, 256), 256, 0, c.stream, ns, ps->slow_idx, dks, dkd, dw, de, ps->ks,
                                                                      ps->kd, ps->w, ps->bad);
        DHGP_LAUNCHED(c);
        c.free(dks);
        c.free(dkd);
        c.free(dw);
        c.free(de);
    }
    ps->src_off = c.alloc<int64_t>(E + 1);
    ps->dst_off = c.alloc<int64_t>(E + 1);
    scan_excl<int64_t>(c, ps->ks, ps->src_off, E);
    scan_excl<int64_t>(c, ps->kd, ps->dst_off, E);
    int64_t tot[2];
    c.d2h(&tot[0], ps->src_off + E, 1);
    c.d2h(&tot[1], ps->dst_off + E, 1);
    c.sync();
    ps->nsrc = tot[0];
    ps->ndst = tot[1];
    ps->src_dat = c.alloc<int32_t>(tot[0]);
    ps->dst_dat = c.alloc<int32_t>(tot[1]);
    if (E > 0) {
        const int blocks = (int)std::min<int64_t>(cdiv(E, 8), (int64_t)c.num_sms * 16);
        pdl_launch(k_line_pass2, blocks, 256, 0, c.stream, ps->text, ps->line_start, E, ps->N, ps->status, ps->ks,
                                                   ps->src_off, ps->dst_off, ps->src_dat, ps->dst_dat, ps->bad);
        DHGP_LAUNCHED(c);
        pdl_launch(k_err_flags, (unsigned)cdiv(E, 256), 256, 0, c.stream, E, ps->status, ps->bad);
        DHGP_LAUNCHED(c);
    }
    if (ns > 0) {
        const int64_t nids = slow_ids_off[ns];
        int64_t *doff = c.alloc<int64_t>(ns + 1);
        int32_t *dids = c.alloc<int32_t>(nids);
        c.h2d(doff, slow_ids_off, ns + 1);
        c.h2d(dids, slow_ids, nids);
        const int blocks = (int)std::min<int64_t>(cdiv(ns, 8), (int64_t)c.num_sms * 16);
        pdl_launch(k_slow_ids, blocks, 256, 0, c.stream, ns, ps->slow_idx, doff, dids, ps->ks, ps->src_off, ps->dst_off,
                                                 ps->src_dat, ps->dst_dat);
        DHGP_LAUNCHED(c);
        c.free(doff);
        c.free(dids);
    }
    // repeated pins within one side (hgraph.py:462-463)
    if (E > 0) {
        // per-side sort (any length) + adjacent check
        int32_t *tmp = c.alloc<int32_t>(std::max(tot[0], tot[1]));
        seg_sort(c, E, ps->src_off, ps->src_dat, nullptr, tmp);
        pdl_launch(k_dup_flags, (unsigned)cdiv(E, 256), 256, 0, c.stream, E, ps->src_off, tmp, ps->bad);
        DHGP_LAUNCHED(c);
        seg_sort(c, E, ps->dst_off, ps->dst_dat, nullptr, tmp);
        pdl_launch(k_dup_flags, (unsigned)cdiv(E, 256), 256, 0, c.stream, E, ps->dst_off, tmp, ps->bad);
        DHGP_LAUNCHED(c);
        c.free(tmp);
    }
    unsigned long long *first = c.alloc<unsigned long long>(1);
    const unsigned long long none = ~0ull;
    c.h2d(first, &none, 1);
    if (E > 0) {
        pdl_launch(k_first_bad, (unsigned)cdiv(E, 256), 256, 0, c.stream, E, ps->bad, first);
        DHGP_LAUNCHED(c);
    }
    unsigned long long fb = 0;
    c.d2h(&fb, first, 1);
    c.sync();
    c.free(first);
    *first_bad_line = fb == ~0ull ? -1 : (int64_t)fb;
    *nsrc = tot[0];
    *ndst = tot[1];
    PARSE_GUARD_END
}

int dhgp_parse_dhg_fetch(dhgp_parse *ps, double *w, int64_t *src_off, int32_t *src_dat, int64_t *dst_off,
                         int32_t *dst_dat) {
    PARSE_GUARD_BEGIN
    Ctx c;
    seams_setup(c, ps->device);
    c.d2h(w, ps->w, ps->E);
    c.d2h(src_off, ps->src_off, ps->E + 1);
    c.d2h(dst_off, ps->dst_off, ps->E + 1);
    c.d2h(src_dat, ps->src_dat, ps->nsrc);
    c.d2h(dst_dat, ps->dst_dat, ps->ndst);
    c.sync();
    PARSE_GUARD_END
}

int dhgp_parse_dhg_line_range(dhgp_parse *ps, int64_t line, int64_t *byte_lo, int64_t *byte_hi) {
    PARSE_GUARD_BEGIN
    if (!ps || line < 0 || line >= ps->E) throw Error{DHGP_ERR_ARG, "line out of range"};
    Ctx c;
    seams_setup(c, ps->device);
    int64_t b[2];
    c.d2h(b, ps->line_start + line, 2);
    c.sync();
    *byte_lo = b[0];
    *byte_hi = b[1] - 1;
    PARSE_GUARD_END
}

void dhgp_parse_free(dhgp_parse *ps) {
    if (!ps) return;
    try {
        Ctx c;
        seams_setup(c, ps->device);
        ps->release(c);
        c.sync();
    } catch (...) {
    }
    delete ps;
}

}  // extern "C"
