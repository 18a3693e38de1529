// coarsen.cu — candidate scoring/selection, matching and contraction.
//
// Scoring never materialises the neighbour sets or the histogram in HBM:
// a node's neighbours are exactly the pins of its incident h-edges minus
// itself (coarsen.py:78-85; the carried sets equal the rematerialised ones,
// test_coarsen.py:183-192), so each warp accumulates hist(n, .) for one node
// in a shared-memory hash table keyed by neighbour id, then scans it in
// (hist desc, id desc) order with the deferred size/inbound checks.
#include <cooperative_groups.h>

#include "coarsen.cuh"
#include "comm.cuh"
#include "prims.cuh"

namespace dhgp {

namespace {

// ---------------------------------------------------------------------------
// flattened iteration over the pins of a node's incident h-edges: the warp
// takes 32 incident h-edges at a time and spreads their pins evenly over the
// lanes (segmented prefix sum + per-slot owner search by shuffles).
// ---------------------------------------------------------------------------
// `work` (profiling only) accumulates the algorithmic bytes read: 28 B per
// incident h-edge (list entry, two offsets, weight) + 4 B per pin
constexpr int kPinsInFlight = 8;
template <int kPinsInFlight = kPinsInFlight, class F>
__device__ __forceinline__ void warp_for_pins(const int32_t *inc_dat, int64_t ilo, int64_t ihi, int64_t first,
                                              int64_t stride, const int64_t *pin_off, const int32_t *pin_dat,
                                              F &&f, unsigned long long *work = nullptr, int bsz = 32) {
    const int lane = lane_id();
    unsigned long long wb = 0;
    // software pipelining: the next batch's offsets and the entries of the
    // one after are loaded before this batch's pins
    auto entry = [&](int64_t b) { return (lane < bsz && b + lane < ihi) ? inc_dat[b + lane] : -1; };
    int32_t ne = entry(ilo + first);
    int64_t nplo = 0, nphi = 0;
    if (ne >= 0) {
        nplo = pin_off[ne];
        nphi = pin_off[ne + 1];
    }
    int32_t ne2 = entry(ilo + first + stride);
    for (int64_t base = ilo + first; base < ihi; base += stride) {
        const int32_t e = ne;
        const int64_t plo = nplo;
        const int len = (int)(nphi - nplo);
        ne = ne2;
        nplo = nphi = 0;
        if (ne >= 0) {
            nplo = pin_off[ne];
            nphi = pin_off[ne + 1];
        }
        ne2 = entry(base + 2 * stride);
        const int incl = warp_incl_scan(len);
        const int total = __shfl_sync(FULL_MASK, incl, 31);
        const int excl = incl - len;
        wb += 28ull * (unsigned long long)min((int64_t)bsz, ihi - base) + 4ull * (unsigned long long)total;
        // eight pins per lane in flight before any is used (the loads are the
        // latency; the hash inserts are cheap)
        for (int s0 = 0; s0 < total; s0 += 32 * kPinsInFlight) {
            int32_t oe[kPinsInFlight], m[kPinsInFlight];
#pragma unroll
            for (int u = 0; u < kPinsInFlight; u++) {
                const int s = s0 + u * 32 + lane;
                int owner = 0;
#pragma unroll
                for (int step = 16; step > 0; step >>= 1) {
                    int ex = __shfl_sync(FULL_MASK, excl, owner + step);
                    if (ex <= s) owner += step;
                }
                oe[u] = __shfl_sync(FULL_MASK, e, owner);
                const int64_t oplo = __shfl_sync(FULL_MASK, plo, owner);
                const int oex = __shfl_sync(FULL_MASK, excl, owner);
                m[u] = s < total ? pin_dat[oplo + (s - oex)] : -1;
            }
#pragma unroll
            for (int u = 0; u < kPinsInFlight; u++)
                if (s0 + u * 32 + lane < total) f(oe[u], m[u]);
        }
    }
    if (work && lane == 0 && wb) atomicAdd(work, wb);
}

struct ScoreArgs {
    int32_t N;
    const int64_t *inc_off;  // per-node list begin ...
    const int32_t *inc_dat;
    const int64_t *pin_off;
    const int32_t *pin_dat;
    const int64_t *wi;
    const int32_t *size;
    const int64_t *in_off;
    const int32_t *in_dat;
    const int64_t *inc_end = nullptr;  // ... and end (DLevel::inc_e / in_e)
    const int64_t *in_end = nullptr;
    int64_t omega, delta;
    int32_t *pair;
    double *score;
    int32_t *next;        // work counter
    int32_t *big_list;    // nodes escalated to the global dense tier
    int32_t *big_count;
    int32_t *heavy_list;  // nodes for the 1024-thread tier (hubs, or too many neighbours for a mid table)
    int32_t *heavy_count;
    Tiers t;
    int32_t lo, hi;  // this rank's node range (comm.cuh); [0, N) on one GPU
    // incremental scoring (score_select_inc): only the listed nodes ...
    const int32_t *list = nullptr;
    const int32_t *list_count = nullptr;
    // ... and, for merged clusters, their (neighbour, cluster, hist) pairs
    // that beat the neighbour's carried choice are emitted as tuples
    const int32_t *mb = nullptr;     // [N] partner of the cluster's min member (-1 = not merged)
    const int32_t *rep = nullptr;    // [N] min member (previous-level id)
    const int64_t *thr_s = nullptr;  // [N] carried score ...
    const int32_t *thr_p = nullptr;  // [N] ... and pair (previous-level id; -1 = none)
    int32_t *tup_v = nullptr, *tup_b = nullptr;
    int64_t *tup_h = nullptr;
    int32_t *tup_count = nullptr;
    int64_t tup_cap = 0;
    unsigned long long *work = nullptr;  // profiling: algorithmic bytes
    // diagnostics (DHGP_TRACE): candidate iterations and nodes, warp / block tier
    unsigned long long *probe = nullptr;
    // list mode with few listed nodes (<= this; 0 = off): the CTA pair tier
    // is preferred (idle SMs otherwise; a node's latency is the level's
    // critical path)
    int32_t heavy_small_list = 0;
    int32_t *mid_list = nullptr;   // nodes for the 256-thread tier
    int32_t *mid_count = nullptr;
    // incremental scoring: per node {size, mb, thr_p, thr_s} in one 16-byte
    // record, so a neighbour's checks in filter_emit cost one gather, not four
    const int4 *pk = nullptr;
};

// next node of a persistent scoring loop: [lo, hi) or the listed nodes in it
// (-1 = done, -2 = skip)
__device__ __forceinline__ int32_t score_node(const ScoreArgs &a, int idx) {
    if (a.list) {
        if (idx >= *a.list_count) return -1;
        const int32_t n = a.list[idx];
        return (n < a.lo || n >= a.hi) ? -2 : n;
    }
    const int64_t n = (int64_t)a.lo + idx;
    return n >= a.hi ? -1 : (int32_t)n;
}

// merged cluster `node`, neighbour m with hist h (size bound already met):
// a candidate for m when m did not merge and (h, node) outranks m's carried
// choice (score, pair) — hist desc, then id desc, where ids compare through
// the clusters' min members (coarse ids are order-isomorphic to them)
__device__ __forceinline__ void emit_tuple(const ScoreArgs &a, int32_t node, int32_t m, long long h) {
    if (!a.mb || a.mb[m] >= 0) return;
    const int32_t tp = a.thr_p[m];
    if (tp >= 0) {
        const long long ts = a.thr_s[m];
        if (!(h > ts || (h == ts && a.rep[node] >= tp))) return;
    }
    const int i = atomicAdd(a.tup_count, 1);
    if (i < a.tup_cap) {
        a.tup_v[i] = m;
        a.tup_b[i] = node;
        a.tup_h[i] = h;
    }
}

// Size filter (_kernels.pyx:92) and tuple emission over a hash table's
// slots [first, cap) with the given stride: the per-slot gathers (size, and
// for merged clusters the neighbour's partner and carried choice) are issued
// for U slots at once, so a thread waits for one round trip per U slots
// rather than one per slot.
template <int U, class Acc>
__device__ __forceinline__ void filter_emit(const ScoreArgs &a, int32_t node, int32_t *keys, const Acc *vals,
                                            int first, int stride, int cap) {
    const int64_t szn = a.size[node];
    const int32_t rn = a.mb ? a.rep[node] : 0;
    for (int s0 = first; s0 < cap; s0 += U * stride) {
        int32_t k[U], sz[U], mbv[U], tp[U];
        long long ts[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int s = s0 + u * stride;
            k[u] = s < cap ? keys[s] : -1;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const bool v = k[u] >= 0;
            if (a.pk) {
                const int4 q = v ? a.pk[k[u]] : make_int4(0, 0, -1, 0);
                sz[u] = q.x;
                mbv[u] = q.y;
                tp[u] = q.z;
                ts[u] = q.w;
            } else {
                sz[u] = v ? a.size[k[u]] : 0;
                mbv[u] = (v && a.mb) ? a.mb[k[u]] : 0;
                tp[u] = (v && a.mb) ? a.thr_p[k[u]] : -1;
                ts[u] = (v && a.mb) ? (long long)a.thr_s[k[u]] : 0;
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int s = s0 + u * stride;
            const bool valid = k[u] >= 0;
            const bool fail = valid && szn + sz[u] > a.omega;
            if (fail) keys[s] = -2;
            // emit_tuple with the gathers above; one atomic per warp
            bool emit = false;
            long long h = 0;
            if (valid && !fail && a.mb && mbv[u] < 0) {
                h = (long long)vals[s];
                emit = !(tp[u] >= 0 && !(h > ts[u] || (h == ts[u] && rn >= tp[u])));
            }
            const uint32_t bal = __ballot_sync(FULL_MASK, emit);
            if (bal) {
                const int lane = lane_id(), leader = __ffs(bal) - 1;
                int base = 0;
                if (lane == leader) base = atomicAdd(a.tup_count, __popc(bal));
                base = __shfl_sync(FULL_MASK, base, leader);
                const int i = base + __popc(bal & ((1u << lane) - 1u));
                if (emit && i < a.tup_cap) {
                    a.tup_v[i] = k[u];
                    a.tup_b[i] = node;
                    a.tup_h[i] = h;
                }
            }
        }
    }
}

constexpr int SS_WARPS = 8;
constexpr int SS_CAP = 1024;   // hash slots per warp (power of two)
// accumulator: 32-bit when the total weight < 2^32 (native shared atomics;
// 64-bit shared atomicAdd is a CAS spin loop on sm_100a), else 64-bit
template <class Acc>
constexpr int ss_smem() { return SS_WARPS * SS_CAP * (4 + (int)sizeof(Acc)); }

__device__ __forceinline__ uint32_t hslot(int32_t m) { return ((uint32_t)m * 2654435761u) >> (32 - 10); }

// |in(n) ∪ in(m)| <= delta, warp-cooperative (_kernels.pyx:94-98)
__device__ __forceinline__ bool warp_union_ok(const ScoreArgs &a, int32_t n, int32_t m) {
    const int64_t nlo = a.in_off[n], nn = a.in_end[n] - nlo;
    const int64_t mlo = a.in_off[m], nm = a.in_end[m] - mlo;
    if (nn + nm <= a.delta) return true;
    const bool ns = nn <= nm;
    const int32_t *sp = a.in_dat + (ns ? nlo : mlo);
    const int32_t *lp = a.in_dat + (ns ? mlo : nlo);
    const int64_t cs = ns ? nn : nm, cl = ns ? nm : nn;
    int64_t common = 0;
    for (int64_t i = lane_id(); i < cs; i += 32) common += bsearch_dev(lp, 0, cl, sp[i]) >= 0;
    common = warp_sum(common);
    return nn + nm - common <= a.delta;
}

template <class Acc>
__global__ void __launch_bounds__(SS_WARPS * 32, 3) k_score_warp(ScoreArgs a) {
    pdl_entry();
    extern __shared__ unsigned long long smem_u64[];
    Acc *svals = (Acc *)smem_u64;
    int32_t *skeys = (int32_t *)(svals + SS_WARPS * SS_CAP);
    __shared__ int32_t snk[SS_WARPS];
    __shared__ int32_t sover[SS_WARPS];
    const int w = warp_id(), lane = lane_id();
    int32_t *keys = skeys + w * SS_CAP;
    Acc *vals = svals + w * SS_CAP;
    while (true) {
        int idx = 0;
        if (lane == 0) idx = atomicAdd(a.next, 1);
        idx = __shfl_sync(FULL_MASK, idx, 0);
        const int32_t node = score_node(a, idx);
        if (node == -1) break;
        if (node < 0) continue;
        const int64_t ilo = a.inc_off[node], ihi = a.inc_end[node];
        // list mode (merged clusters, rescored nodes): every node above
        // ss_list_inc incident h-edges gets a CTA (a node's latency is the
        // level's critical path); full scoring: above ss_heavy_inc
        const int64_t hthr = a.list ? min(a.t.ss_heavy_inc, a.t.ss_list_inc) : (int64_t)a.t.ss_heavy_inc;
        if (ihi - ilo > hthr) {
            if (lane == 0) {
                if (ihi - ilo > a.t.sm_heavy_inc)
                    a.heavy_list[atomicAdd(a.heavy_count, 1)] = node;
                else
                    a.mid_list[atomicAdd(a.mid_count, 1)] = node;
            }
            continue;
        }
        for (int s = lane; s < SS_CAP; s += 32) {
            keys[s] = -1;
            vals[s] = 0;
        }
        if (lane == 0) {
            snk[w] = 0;
            sover[w] = 0;
        }
        __syncwarp();
        warp_for_pins(a.inc_dat, ilo, ihi, 0, 32, a.pin_off, a.pin_dat, [&](int32_t e, int32_t m) {
            if (m == node) return;
            const Acc we = (Acc)a.wi[e];
            uint32_t h = hslot(m);
            for (int probe = 0; probe < SS_CAP; probe++) {
                if (probe % kFlagPoll == kFlagPoll - 1 && flag_get(&sover[w])) return;
                const int slot = (h + probe) & (SS_CAP - 1);
                int k = keys[slot];
                if (k == -1) {
                    int prev = atomicCAS(&keys[slot], -1, m);
                    if (prev == -1) {
                        if (atomicAdd(&snk[w], 1) >= a.t.ss_limit) flag_set(&sover[w]);
                        k = m;
                    } else {
                        k = prev;
                    }
                }
                if (k == m) {
                    atomicAdd(&vals[slot], we);
                    return;
                }
            }
            flag_set(&sover[w]);
        }, a.work);
        __syncwarp();
        if (sover[w]) {
            if (lane == 0) a.mid_list[atomicAdd(a.mid_count, 1)] = node;
            __syncwarp();
            continue;
        }
        // size check once per candidate (_kernels.pyx:92)
        filter_emit<8>(a, node, keys, vals, lane, 32, SS_CAP);
        __syncwarp();
        int32_t best_m = -1;
        int64_t best_v = 0;
        int iters = 0;
        while (true) {
            iters++;
            int64_t bv = -1;
            int32_t bk = -1;
            int bs = -1;
            for (int s = lane; s < SS_CAP; s += 32) {
                int k = keys[s];
                if (k >= 0) {
                    int64_t v = (int64_t)vals[s];
                    if (v > bv || (v == bv && k > bk)) {
                        bv = v;
                        bk = k;
                        bs = s;
                    }
                }
            }
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                int64_t ov = __shfl_xor_sync(FULL_MASK, bv, d);
                int32_t ok = __shfl_xor_sync(FULL_MASK, bk, d);
                int os = __shfl_xor_sync(FULL_MASK, bs, d);
                if (ov > bv || (ov == bv && ok > bk)) {
                    bv = ov;
                    bk = ok;
                    bs = os;
                }
            }
            if (bk < 0) break;
            if (warp_union_ok(a, node, bk)) {
                best_m = bk;
                best_v = bv;
                break;
            }
            if (lane == 0) keys[bs] = -2;
            __syncwarp();
        }
        if (lane == 0) {
            a.pair[node] = best_m;
            a.score[node] = best_m >= 0 ? (double)best_v : 0.0;
            if (a.probe) {
                atomicAdd(&a.probe[0], (unsigned long long)iters);
                atomicAdd(&a.probe[2], 1ull);
            }
        }
        __syncwarp();
    }
}

// Mid tier: a 256-thread CTA per node with a 4096-slot shared hash table —
// the merged clusters and rescored nodes of the incremental levels (a few
// hundred to a few thousand per level, each a few thousand pins), several
// CTAs per SM so that all of a level's nodes run at once.  The 8 warps
// flatten the pins of their share of the incident h-edges; nodes with more
// distinct neighbours than sm_limit go on to the 1024-thread tier.
constexpr int SM_THREADS = 256;
constexpr int SM_CAP = 4096;
template <class Acc>
constexpr int sm_smem() { return SM_CAP * (4 + (int)sizeof(Acc)); }

template <class Acc>
__global__ void __launch_bounds__(SM_THREADS, 5) k_score_mid(ScoreArgs a) {
    pdl_entry();
    extern __shared__ unsigned long long smem_u64[];
    Acc *vals = (Acc *)smem_u64;
    int32_t *keys = (int32_t *)(vals + SM_CAP);
    __shared__ int32_t snk, s_next;
    __shared__ int32_t sover;
    __shared__ long long r_v[SM_THREADS / 32], r_c[SM_THREADS / 32];
    __shared__ int32_t r_k[SM_THREADS / 32], r_s[SM_THREADS / 32];
    __shared__ long long s_pins;
    constexpr int NW = SM_THREADS / 32;
    const int w = warp_id(), lane = lane_id();
    const int nmid = *a.mid_count;
    if (nmid <= (int)gridDim.x / 4) {
        // few nodes (SMs would idle): the 1024-thread tier (CTA pairs) takes them
        for (int t = blockIdx.x * SM_THREADS + threadIdx.x; t < nmid; t += gridDim.x * SM_THREADS)
            a.heavy_list[atomicAdd(a.heavy_count, 1)] = a.mid_list[t];
        return;
    }
    while (true) {
        if (threadIdx.x == 0) s_next = atomicAdd(a.next + 3, 1);
        __syncthreads();
        const int t = s_next;
        if (t >= nmid) break;
        const int32_t node = a.mid_list[t];
        const int64_t ilo = a.inc_off[node], ihi = a.inc_end[node];
        {  // table sized to the node (>= twice its pin slots), as in k_score_heavy
            long long pe = 0;
            for (int64_t i = ilo + threadIdx.x; i < ihi; i += SM_THREADS) {
                const int32_t e = a.inc_dat[i];
                pe += a.pin_off[e + 1] - a.pin_off[e];
            }
            pe = warp_sum(pe);
            if (lane == 0) r_c[w] = pe;
            __syncthreads();
            if (threadIdx.x == 0) {
                long long tot = 0;
                for (int j = 0; j < NW; j++) tot += r_c[j];
                s_pins = tot;
            }
            __syncthreads();
        }
        int lg = 12;
        while (lg > 8 && (1ll << (lg - 1)) >= 2 * s_pins) lg--;
        const int cap = 1 << lg;
        const int limit = min(a.t.sm_limit, cap - (cap >> 2));
        for (int s = threadIdx.x; s < cap; s += SM_THREADS) {
            keys[s] = -1;
            vals[s] = 0;
        }
        if (threadIdx.x == 0) {
            snk = 0;
            sover = 0;
        }
        __syncthreads();
        const int bsz = (int)max((int64_t)1, min((int64_t)32, (ihi - ilo + NW - 1) / NW));
        warp_for_pins<4>(a.inc_dat, ilo, ihi, (int64_t)w * bsz, (int64_t)NW * bsz, a.pin_off, a.pin_dat,
                         [&](int32_t e, int32_t m) {
                             if (m == node) return;
                             const Acc we = (Acc)a.wi[e];
                             uint32_t h = ((uint32_t)m * 2654435761u) >> (32 - lg);
                             for (int probe = 0; probe < cap; probe++) {
                                 if (probe % kFlagPoll == kFlagPoll - 1 && flag_get(&sover)) return;
                                 const int slot = (h + probe) & (cap - 1);
                                 int k = keys[slot];
                                 if (k == -1) {
                                     const int prev = atomicCAS(&keys[slot], -1, m);
                                     if (prev == -1) {
                                         if (atomicAdd(&snk, 1) + 1 > limit) flag_set(&sover);
                                         k = m;
                                     } else {
                                         k = prev;
                                     }
                                 }
                                 if (k == m) {
                                     atomicAdd(&vals[slot], we);
                                     return;
                                 }
                             }
                             flag_set(&sover);
                         },
                         a.work, bsz);
        __syncthreads();
        if (sover) {
            if (threadIdx.x == 0) a.heavy_list[atomicAdd(a.heavy_count, 1)] = node;
            __syncthreads();
            continue;
        }
        filter_emit<8>(a, node, keys, vals, threadIdx.x, SM_THREADS, cap);
        __syncthreads();
        int32_t best_m = -1;
        long long best_v = 0;
        while (true) {
            long long bv = -1;
            int32_t bk = -1, bs = -1;
            for (int s = threadIdx.x; s < cap; s += SM_THREADS) {
                const int k = keys[s];
                if (k >= 0) {
                    const long long v = (long long)vals[s];
                    if (v > bv || (v == bv && k > bk)) {
                        bv = v;
                        bk = k;
                        bs = s;
                    }
                }
            }
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                const long long ov = __shfl_xor_sync(FULL_MASK, bv, d);
                const int32_t ok = __shfl_xor_sync(FULL_MASK, bk, d), os = __shfl_xor_sync(FULL_MASK, bs, d);
                if (ov > bv || (ov == bv && ok > bk)) {
                    bv = ov;
                    bk = ok;
                    bs = os;
                }
            }
            if (lane == 0) {
                r_v[w] = bv;
                r_k[w] = bk;
                r_s[w] = bs;
            }
            __syncthreads();
            bv = r_v[0];
            bk = r_k[0];
            bs = r_s[0];
#pragma unroll
            for (int j = 1; j < NW; j++)
                if (r_v[j] > bv || (r_v[j] == bv && r_k[j] > bk)) {
                    bv = r_v[j];
                    bk = r_k[j];
                    bs = r_s[j];
                }
            __syncthreads();
            if (bk < 0) break;
            const int64_t nlo = a.in_off[node], nn = a.in_end[node] - nlo;
            const int64_t mlo = a.in_off[bk], nm = a.in_end[bk] - mlo;
            bool ok = true;
            if (nn + nm > a.delta) {
                const bool ns = nn <= nm;
                const int32_t *sp = a.in_dat + (ns ? nlo : mlo), *lp = a.in_dat + (ns ? mlo : nlo);
                const int64_t cs = ns ? nn : nm, cl = ns ? nm : nn;
                long long common = 0;
                for (int64_t i = threadIdx.x; i < cs; i += SM_THREADS) common += bsearch_dev(lp, 0, cl, sp[i]) >= 0;
                common = warp_sum(common);
                if (lane == 0) r_c[w] = common;
                __syncthreads();
                long long tot = 0;
#pragma unroll
                for (int j = 0; j < NW; j++) tot += r_c[j];
                __syncthreads();
                ok = nn + nm - tot <= a.delta;
            }
            if (ok) {
                best_m = bk;
                best_v = bv;
                break;
            }
            if (threadIdx.x == 0) keys[bs] = -2;
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            a.pair[node] = best_m;
            a.score[node] = best_m >= 0 ? (double)best_v : 0.0;
        }
        __syncthreads();
    }
}

// Block tier: one 1024-thread block per heavy node, 16K-slot shared hash
// table (warps flatten the pins of 32 incident h-edges at a time); nodes
// with more distinct neighbours than the table holds go to the dense tier.
constexpr int SH_THREADS = 1024;
constexpr int SH_CAP = 16384;
template <class Acc>
constexpr int sh_smem() { return SH_CAP * (4 + (int)sizeof(Acc)); }

// CL = 2: a thread-block cluster (CTA pair on two SMs) per node.  Each CTA
// hashes half of the node's h-edges into its own table; the second then
// merges its table — distinct neighbours, far fewer than pins — into the
// first's over distributed shared memory, and the first selects.
// Pairs when the list fits them (a node each: the level's hubs, C2's merged
// clusters), else single CTAs over the whole list (many hubs: every SM on its
// own node); `pairs` = the pair launch's cluster count, the other launch exits.
template <class Acc, int CL>
__global__ void __launch_bounds__(SH_THREADS) k_score_heavy(ScoreArgs a, int pairs) {
    pdl_entry();
    extern __shared__ unsigned long long smem_u64[];
    Acc *vals = (Acc *)smem_u64;
    int32_t *keys = (int32_t *)(vals + SH_CAP);
    __shared__ int32_t snk;
    __shared__ int32_t sover;
    __shared__ long long r_v[SH_THREADS / 32];
    __shared__ int32_t r_k[SH_THREADS / 32], r_s[SH_THREADS / 32];
    __shared__ long long r_c[SH_THREADS / 32];
    __shared__ long long s_pins;
    static_assert(SH_THREADS == 1024, "the winner reduction reads one entry per lane");
    static_assert(CL == 1 || CL == 2, "one CTA or a CTA pair per node");
    const int w = warp_id(), lane = lane_id(), nw = SH_THREADS / 32;
    const int nheavy = *a.heavy_count;
    if ((CL == 2) != (nheavy <= pairs)) return;
    int rank = 0;
    if constexpr (CL == 2) rank = (int)cooperative_groups::this_cluster().block_rank();
    for (int t = (int)blockIdx.x / CL; t < nheavy; t += gridDim.x / CL) {
        const int32_t node = a.heavy_list[t];
        const int64_t ilo = a.inc_off[node], ihi = a.inc_end[node];
        // table sized to the node: at least twice its pin slots (its distinct
        // neighbours are fewer), so the clear / filter / argmax scans cost
        // what the node needs rather than the full 16K slots
        {
            long long pe = 0;
            for (int64_t i = ilo + threadIdx.x; i < ihi; i += SH_THREADS) {
                const int32_t e = a.inc_dat[i];
                pe += a.pin_off[e + 1] - a.pin_off[e];
            }
            pe = warp_sum(pe);
            if (lane == 0) r_c[w] = pe;
            __syncthreads();
            if (threadIdx.x == 0) {
                long long tot = 0;
                for (int j = 0; j < nw; j++) tot += r_c[j];
                s_pins = tot;
            }
            __syncthreads();
        }
        int lg = 14;
        while (lg > 10 && (1ll << (lg - 1)) >= 2 * s_pins) lg--;
        const int cap = 1 << lg;
        const int limit = min(a.t.sh_limit, cap - (cap >> 2));
        for (int s = threadIdx.x; s < cap; s += SH_THREADS) {
            keys[s] = -1;
            vals[s] = 0;
        }
        if (threadIdx.x == 0) {
            snk = 0;
            sover = 0;
        }
        __syncthreads();
        int pend = 0;  // this thread's new keys not yet added to snk
        // h-edges per warp batch: a node's h-edges spread over all warps
        // (of both CTAs of a pair)
        const int bsz = (int)max((int64_t)1, min((int64_t)32, (ihi - ilo + CL * nw - 1) / (CL * nw)));
        warp_for_pins<4>(a.inc_dat, ilo, ihi, (int64_t)(rank * nw + w) * bsz, (int64_t)CL * nw * bsz, a.pin_off,
                         a.pin_dat,
                      [&](int32_t e, int32_t m) {
                          if (m == node) return;
                          const Acc we = (Acc)a.wi[e];
                          uint32_t h = ((uint32_t)m * 2654435761u) >> (32 - lg);
                          for (int probe = 0; probe < cap; probe++) {
                              if (probe % kFlagPoll == kFlagPoll - 1 && flag_get(&sover)) return;
                              const int slot = (h + probe) & (cap - 1);
                              int k = keys[slot];
                              if (k == -1) {
                                  int prev = atomicCAS(&keys[slot], -1, m);
                                  if (prev == -1) {
                                      // new keys counted in pairs (half the
                                      // shared atomics; the limit only picks
                                      // the tier, never the result)
                                      if (++pend == 2) {
                                          pend = 0;
                                          if (atomicAdd(&snk, 2) + 2 > limit) flag_set(&sover);
                                      }
                                      k = m;
                                  } else {
                                      k = prev;
                                  }
                              }
                              if (k == m) {
                                  atomicAdd(&vals[slot], we);
                                  return;
                              }
                          }
                          flag_set(&sover);
                      },
                      a.work, bsz);
        __syncthreads();
        if constexpr (CL == 2) {
            cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
            cl.sync();  // both partial tables complete
            if (rank == 1) {
                int32_t *keys0 = cl.map_shared_rank(keys, 0);
                Acc *vals0 = cl.map_shared_rank(vals, 0);
                int32_t *snk0 = cl.map_shared_rank(&snk, 0);
                int32_t *sover0 = cl.map_shared_rank(&sover, 0);
                if (sover) {
                    if (threadIdx.x == 0) atomicExch(sover0, 1);
                } else {
                    for (int s = threadIdx.x; s < cap; s += SH_THREADS) {
                        const int32_t m = keys[s];
                        if (m < 0 || atomicAdd(sover0, 0)) continue;
                        const Acc v = vals[s];
                        const uint32_t h = ((uint32_t)m * 2654435761u) >> (32 - lg);
                        bool done = false;
                        for (int probe = 0; probe < cap && !done; probe++) {
                            const int slot = (h + probe) & (cap - 1);
                            int k = ((volatile int32_t *)keys0)[slot];
                            if (k == -1) {
                                const int prev = atomicCAS(&keys0[slot], -1, m);
                                if (prev == -1) {
                                    if (atomicAdd(snk0, 1) + 1 > limit) atomicExch(sover0, 1);
                                    k = m;
                                } else {
                                    k = prev;
                                }
                            }
                            if (k == m) {
                                atomicAdd(&vals0[slot], v);
                                done = true;
                            }
                        }
                        if (!done) atomicExch(sover0, 1);
                    }
                }
            }
            cl.sync();  // the merge is complete
            if (rank == 1) continue;
        }
        if (sover) {
            if (threadIdx.x == 0) a.big_list[atomicAdd(a.big_count, 1)] = node;
            __syncthreads();
            continue;
        }
        filter_emit<4>(a, node, keys, vals, threadIdx.x, SH_THREADS, cap);
        __syncthreads();
        int32_t best_m = -1;
        long long best_v = 0;
        int iters = 0;
        while (true) {
            iters++;
            long long bv = -1;
            int32_t bk = -1, bs = -1;
            for (int s = threadIdx.x; s < cap; s += SH_THREADS) {
                int k = keys[s];
                if (k >= 0) {
                    long long v = (long long)vals[s];
                    if (v > bv || (v == bv && k > bk)) {
                        bv = v;
                        bk = k;
                        bs = s;
                    }
                }
            }
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                long long ov = __shfl_xor_sync(FULL_MASK, bv, d);
                int32_t ok = __shfl_xor_sync(FULL_MASK, bk, d);
                int32_t os = __shfl_xor_sync(FULL_MASK, bs, d);
                if (ov > bv || (ov == bv && ok > bk)) {
                    bv = ov;
                    bk = ok;
                    bs = os;
                }
            }
            if (lane == 0) {
                r_v[w] = bv;
                r_k[w] = bk;
                r_s[w] = bs;
            }
            __syncthreads();
            // every warp reduces the 32 per-warp winners by shuffles
            bv = r_v[lane];
            bk = r_k[lane];
            bs = r_s[lane];
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                long long ov = __shfl_xor_sync(FULL_MASK, bv, d);
                int32_t ok = __shfl_xor_sync(FULL_MASK, bk, d);
                int32_t os = __shfl_xor_sync(FULL_MASK, bs, d);
                if (ov > bv || (ov == bv && ok > bk)) {
                    bv = ov;
                    bk = ok;
                    bs = os;
                }
            }
            __syncthreads();
            if (bk < 0) break;
            const int64_t nlo = a.in_off[node], nn = a.in_end[node] - nlo;
            const int64_t mlo = a.in_off[bk], nm = a.in_end[bk] - mlo;
            bool ok = true;
            if (nn + nm > a.delta) {
                const bool ns = nn <= nm;
                const int32_t *sp = a.in_dat + (ns ? nlo : mlo);
                const int32_t *lp = a.in_dat + (ns ? mlo : nlo);
                const int64_t cs = ns ? nn : nm, cl = ns ? nm : nn;
                long long common = 0;
                for (int64_t i = threadIdx.x; i < cs; i += SH_THREADS) common += bsearch_dev(lp, 0, cl, sp[i]) >= 0;
                common = warp_sum(common);
                if (lane == 0) r_c[w] = common;
                __syncthreads();
                long long tot = 0;
                for (int j = 0; j < nw; j++) tot += r_c[j];
                __syncthreads();
                ok = nn + nm - tot <= a.delta;
            }
            if (ok) {
                best_m = bk;
                best_v = bv;
                break;
            }
            if (threadIdx.x == 0) keys[bs] = -2;
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            a.pair[node] = best_m;
            a.score[node] = best_m >= 0 ? (double)best_v : 0.0;
            if (a.probe) {
                atomicAdd(&a.probe[1], (unsigned long long)iters);
                atomicAdd(&a.probe[3], 1ull);
            }
        }
        __syncthreads();
    }
}

// Block tier for nodes with many distinct neighbours: a dense per-block
// histogram over all node ids in global memory (L2-resident), restored to
// "untouched" (-1) after each node.
constexpr int SB_THREADS = 512;
__global__ void __launch_bounds__(SB_THREADS) k_score_block(ScoreArgs a, long long *dense_all, int32_t *touched_all,
                                                             long long *cval_all, int32_t n_real) {
    pdl_entry();
    (void)n_real;
    __shared__ int32_t s_nt;
    __shared__ long long s_bv[SB_THREADS / 32];
    __shared__ int32_t s_bk[SB_THREADS / 32];
    __shared__ int32_t s_bi[SB_THREADS / 32];
    __shared__ long long s_common[SB_THREADS / 32];
    long long *dense = dense_all + (int64_t)blockIdx.x * a.N;
    int32_t *touched = touched_all + (int64_t)blockIdx.x * a.N;
    long long *cval = cval_all + (int64_t)blockIdx.x * a.N;
    const int w = warp_id(), lane = lane_id(), nw = SB_THREADS / 32;
    const int nbig = *a.big_count;
    for (int t = blockIdx.x; t < nbig; t += gridDim.x) {
        const int32_t node = a.big_list[t];
        if (threadIdx.x == 0) s_nt = 0;
        __syncthreads();
        const int64_t ilo = a.inc_off[node], ihi = a.inc_end[node];
        // h-edges per warp batch: a node's h-edges spread over all warps
        const int bsz = (int)max((int64_t)1, min((int64_t)32, (ihi - ilo + nw - 1) / nw));
        warp_for_pins<4>(a.inc_dat, ilo, ihi, (int64_t)w * bsz, (int64_t)nw * bsz, a.pin_off, a.pin_dat,
                      [&](int32_t e, int32_t m) {
                          if (m == node) return;
                          long long old = atomicCAS((unsigned long long *)&dense[m], ~0ull, 0ull);
                          if (old == -1ll) touched[atomicAdd(&s_nt, 1)] = m;
                          atomicAdd((unsigned long long *)&dense[m], (unsigned long long)a.wi[e]);
                      },
                      a.work, bsz);
        __syncthreads();
        const int nt = s_nt;
        const int64_t szn = a.size[node];
        for (int i = threadIdx.x; i < nt; i += SB_THREADS) {
            int32_t m = touched[i];
            cval[i] = dense[m];
            dense[m] = -1ll;
            if (szn + a.size[m] > a.omega) touched[i] = -2;
            else emit_tuple(a, node, m, cval[i]);
        }
        __syncthreads();
        int32_t best_m = -1;
        long long best_v = 0;
        while (true) {
            long long bv = -1;
            int32_t bk = -1, bi = -1;
            for (int i = threadIdx.x; i < nt; i += SB_THREADS) {
                int32_t k = touched[i];
                if (k >= 0) {
                    long long v = cval[i];
                    if (v > bv || (v == bv && k > bk)) {
                        bv = v;
                        bk = k;
                        bi = i;
                    }
                }
            }
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                long long ov = __shfl_xor_sync(FULL_MASK, bv, d);
                int32_t ok = __shfl_xor_sync(FULL_MASK, bk, d);
                int32_t oi = __shfl_xor_sync(FULL_MASK, bi, d);
                if (ov > bv || (ov == bv && ok > bk)) {
                    bv = ov;
                    bk = ok;
                    bi = oi;
                }
            }
            if (lane == 0) {
                s_bv[w] = bv;
                s_bk[w] = bk;
                s_bi[w] = bi;
            }
            __syncthreads();
            bv = s_bv[0];
            bk = s_bk[0];
            bi = s_bi[0];
            for (int j = 1; j < nw; j++) {
                if (s_bv[j] > bv || (s_bv[j] == bv && s_bk[j] > bk)) {
                    bv = s_bv[j];
                    bk = s_bk[j];
                    bi = s_bi[j];
                }
            }
            __syncthreads();
            if (bk < 0) break;
            // union check by the whole block
            const int64_t nlo = a.in_off[node], nn = a.in_end[node] - nlo;
            const int64_t mlo = a.in_off[bk], nm = a.in_end[bk] - mlo;
            bool ok;
            if (nn + nm <= a.delta) {
                ok = true;
            } else {
                const bool ns = nn <= nm;
                const int32_t *sp = a.in_dat + (ns ? nlo : mlo);
                const int32_t *lp = a.in_dat + (ns ? mlo : nlo);
                const int64_t cs = ns ? nn : nm, cl = ns ? nm : nn;
                long long common = 0;
                for (int64_t i = threadIdx.x; i < cs; i += SB_THREADS) common += bsearch_dev(lp, 0, cl, sp[i]) >= 0;
                common = warp_sum(common);
                if (lane == 0) s_common[w] = common;
                __syncthreads();
                long long tot = 0;
                for (int j = 0; j < nw; j++) tot += s_common[j];
                __syncthreads();
                ok = nn + nm - tot <= a.delta;
            }
            if (ok) {
                best_m = bk;
                best_v = bv;
                break;
            }
            if (threadIdx.x == 0) touched[bi] = -2;
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            a.pair[node] = best_m;
            a.score[node] = best_m >= 0 ? (double)best_v : 0.0;
        }
        __syncthreads();
    }
}


// ---- incremental scoring (score_select_inc) ------------------------------
// kind: 0 merged cluster (rescored), 1 carried pair still a singleton,
// 2 no carried pair, 3 carried pair merged (rescored unless a tuple wins)
__global__ void k_inc_base(int32_t N, const int32_t *ma, const int32_t *mb, const int32_t *gamma_prev,
                           const int32_t *prev_pair, const double *prev_score, uint8_t *kind, int64_t *thr_s,
                           int32_t *thr_p, unsigned long long *best, int32_t *list, int32_t *list_count,
                           const int32_t *size, int4 *pk) {
    pdl_entry();
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= N) return;
    best[c] = 0ull;
    const int32_t m = mb[c], sz = size[c];
    if (m >= 0) {
        kind[c] = 0;
        thr_p[c] = -1;
        thr_s[c] = 0;  // (gathered alongside thr_p by filter_emit, never used when thr_p < 0)
        pk[c] = make_int4(sz, m, -1, 0);
        list[atomicAdd(list_count, 1)] = (int32_t)c;
        return;
    }
    const int32_t f = ma[c], p = prev_pair[f];
    if (p < 0) {
        kind[c] = 2;
        thr_p[c] = -1;
        thr_s[c] = 0;
        pk[c] = make_int4(sz, m, -1, 0);
        return;
    }
    // carried scores are hist values < 2^31 (incremental mode: total weight < 2^31)
    thr_s[c] = (int64_t)prev_score[f];
    thr_p[c] = p;
    pk[c] = make_int4(sz, m, p, (int32_t)(int64_t)prev_score[f]);
    kind[c] = mb[gamma_prev[p]] >= 0 ? 3 : 1;
}
// tuples that pass the inbound-union bound compete by (hist, cluster id):
// thread per tuple when |in(v)| + |in(b)| <= delta (no search needed), the
// others are listed for a warp each
__device__ __forceinline__ unsigned long long tuple_key(long long h, int32_t b) {
    return ((unsigned long long)(h + 1) << 32) | (unsigned long long)(uint32_t)b;
}
__global__ void k_inc_tuples_quick(ScoreArgs a, unsigned long long *best, int32_t *hard, int32_t *hard_count) {
    pdl_entry();
    const int64_t nt = min((int64_t)*a.tup_count, a.tup_cap);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nt; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = a.tup_v[i], b = a.tup_b[i];
        if ((a.in_end[v] - a.in_off[v]) + (a.in_end[b] - a.in_off[b]) <= a.delta)
            atomicMax(&best[v], tuple_key(a.tup_h[i], b));
        else
            hard[atomicAdd(hard_count, 1)] = (int32_t)i;
    }
}
__global__ void k_inc_tuples(ScoreArgs a, unsigned long long *best, const int32_t *hard, const int32_t *hard_count) {
    pdl_entry();
    const int64_t nt = *hard_count;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id(); t < nt; t += nw) {
        const int32_t i = hard[t];
        const int32_t v = a.tup_v[i], b = a.tup_b[i];
        if (warp_union_ok(a, v, b) && lane_id() == 0) atomicMax(&best[v], tuple_key(a.tup_h[i], b));
    }
}
__global__ void k_inc_finalize(int32_t N, const uint8_t *kind, const int64_t *thr_s, const int32_t *thr_p,
                               const unsigned long long *best, const int32_t *gamma_prev, const int32_t *tup_count,
                               int64_t tup_cap, int32_t *pair, double *score, int32_t *list, int32_t *list_count) {
    pdl_entry();
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= N) return;
    const int k = kind[c];
    if (k == 0) return;
    if ((int64_t)*tup_count > tup_cap) {  // tuples were dropped: rescore
        list[atomicAdd(list_count, 1)] = (int32_t)c;
        return;
    }
    const unsigned long long b = best[c];
    if (b) {
        pair[c] = (int32_t)(uint32_t)(b & 0xffffffffull);
        score[c] = (double)((long long)(b >> 32) - 1);
    } else if (k == 1) {
        pair[c] = gamma_prev[thr_p[c]];
        score[c] = (double)thr_s[c];
    } else if (k == 2) {
        pair[c] = -1;
        score[c] = 0.0;
    } else {
        list[atomicAdd(list_count, 1)] = (int32_t)c;
    }
}

__global__ void k_fill_ll(long long *p, long long v, int64_t n) {
    pdl_entry();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

}  // namespace

void score_scratch_init(Ctx &c, ScoreScratch &s, int64_t n_cap) {
    s.cap = std::max<int64_t>(n_cap, 1);
    // as many dense rows (20 B per node id each) as 4 GiB allows, <= 2 per SM
    s.blocks = (int)std::max<int64_t>(1, std::min<int64_t>(2ll * c.num_sms, (4ll << 30) / (20 * s.cap)));
    s.dense = c.alloc<long long>((int64_t)s.blocks * s.cap);
    s.cval = c.alloc<long long>((int64_t)s.blocks * s.cap);
    s.touched = c.alloc<int32_t>((int64_t)s.blocks * s.cap);
    s.big = c.alloc<int32_t>(s.cap);
    s.heavy = c.alloc<int32_t>(s.cap);
    s.mid = c.alloc<int32_t>(s.cap);
    s.ctr = c.alloc<int32_t>(6);
    pdl_launch(k_fill_ll, (unsigned)cdiv((int64_t)s.blocks * s.cap, 256), 256, 0, c.stream, s.dense, -1ll,
                                                                                   (int64_t)s.blocks * s.cap);
    DHGP_LAUNCHED(c);
}

void score_scratch_release(Ctx &c, ScoreScratch &s) {
    c.free(s.dense);
    c.free(s.cval);
    c.free(s.touched);
    c.free(s.big);
    c.free(s.heavy);
    c.free(s.mid);
    c.free(s.ctr);
    s = ScoreScratch();
}

// the block tier as CTA pairs (thread-block clusters of 2), as many pairs as
// can be co-resident
template <class Acc>
static void launch_heavy_pairs(Ctx &c, const ScoreArgs &a) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // as pdl_launch (the kernel waits first)
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.blockDim = dim3(SH_THREADS);
    cfg.dynamicSmemBytes = sh_smem<Acc>();
    cfg.stream = c.stream;
    cfg.attrs = at;
    cfg.numAttrs = 1;  // the occupancy query takes the cluster shape only
    static int pairs = 0;
    if (!pairs) {
        cfg.gridDim = dim3(2 * (c.num_sms / 2));
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, (void *)k_score_heavy<Acc, 2>, &cfg) != cudaSuccess || n < 1)
            n = c.num_sms / 2;
        pairs = std::min(n, c.num_sms / 2);
    }
    cfg.gridDim = dim3(2 * pairs);
    cfg.numAttrs = 2;
    DHGP_CUDA(cudaLaunchKernelEx(&cfg, k_score_heavy<Acc, 2>, a, pairs));
    DHGP_LAUNCHED(c);
    // more nodes than pairs: single CTAs (exactly one of the two launches works)
    pdl_launch(k_score_heavy<Acc, 1>, c.num_sms, SH_THREADS, sh_smem<Acc>(), c.stream, a, pairs);
    DHGP_LAUNCHED(c);
}

static void score_attrs(Ctx &c) {
    static bool attr = false;
    if (attr) return;
    DHGP_CUDA(cudaFuncSetAttribute(k_score_warp<unsigned>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   ss_smem<unsigned>()));
    DHGP_CUDA(cudaFuncSetAttribute(k_score_warp<unsigned long long>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   ss_smem<unsigned long long>()));
    DHGP_CUDA(cudaFuncSetAttribute(k_score_mid<unsigned>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   sm_smem<unsigned>()));
    DHGP_CUDA(cudaFuncSetAttribute(k_score_mid<unsigned long long>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   sm_smem<unsigned long long>()));
    DHGP_CUDA(cudaFuncSetAttribute(k_score_heavy<unsigned, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   sh_smem<unsigned>()));
    DHGP_CUDA(cudaFuncSetAttribute(k_score_heavy<unsigned long long, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   sh_smem<unsigned long long>()));
    DHGP_CUDA(cudaFuncSetAttribute(k_score_heavy<unsigned, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   sh_smem<unsigned>()));
    DHGP_CUDA(cudaFuncSetAttribute(k_score_heavy<unsigned long long, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   sh_smem<unsigned long long>()));
    attr = true;
}

// the three scoring tiers over all of [a.lo, a.hi) or over a.list
static void score_tiers(Ctx &c, ScoreArgs a, const DWeights &W, ScoreScratch &s, int32_t n_real) {
    c.zero(s.ctr, 6);
    a.mid_list = s.mid;
    a.mid_count = s.ctr + 4;
    const int64_t nmine = a.list ? ((int64_t)1 << 40) : std::max<int64_t>(1, (int64_t)a.hi - a.lo);
    KScope kw(c, "sc_warp");
    if (W.wsum < (1ll << 32)) {
        static int g32 = resident_grid(c, k_score_warp<unsigned>, SS_WARPS * 32, ss_smem<unsigned>());
        int blocks = (int)std::min<int64_t>(cdiv(nmine, SS_WARPS), g32);
        pdl_launch(k_score_warp<unsigned>, blocks, SS_WARPS * 32, ss_smem<unsigned>(), c.stream, a);
    } else {
        static int g64 = resident_grid(c, k_score_warp<unsigned long long>, SS_WARPS * 32, ss_smem<unsigned long long>());
        int blocks = (int)std::min<int64_t>(cdiv(nmine, SS_WARPS), g64);
        pdl_launch(k_score_warp<unsigned long long>, blocks, SS_WARPS * 32, ss_smem<unsigned long long>(), c.stream, a);
    }
    DHGP_LAUNCHED(c);
    kw.close();
    // mid tier: persistent CTAs over the escalated list (exits when empty)
    KScope km(c, "sc_mid");
    if (W.wsum < (1ll << 32)) {
        static int m32 = resident_grid(c, k_score_mid<unsigned>, SM_THREADS, sm_smem<unsigned>());
        pdl_launch(k_score_mid<unsigned>, m32, SM_THREADS, sm_smem<unsigned>(), c.stream, a);
    } else {
        static int m64 = resident_grid(c, k_score_mid<unsigned long long>, SM_THREADS, sm_smem<unsigned long long>());
        pdl_launch(k_score_mid<unsigned long long>, m64, SM_THREADS, sm_smem<unsigned long long>(), c.stream, a);
    }
    DHGP_LAUNCHED(c);
    km.close();
    // heavy tier: reads the escalation count on device, exits when zero
    KScope kh(c, "sc_heavy");
    if (W.wsum < (1ll << 32))
        launch_heavy_pairs<unsigned>(c, a);
    else
        launch_heavy_pairs<unsigned long long>(c, a);
    kh.close();
    KScope kd(c, "sc_dense");
    // dense tier: reads the escalation count on device, exits when zero;
    // dense rows have stride s.cap and are restored to -1 after each node
    a.N = (int32_t)s.cap;
    pdl_launch(k_score_block, s.blocks, SB_THREADS, 0, c.stream, a, s.dense, s.touched, s.cval, n_real);
    DHGP_LAUNCHED(c);
}

void score_select(Ctx &c, const DLevel &L, const DWeights &W, int64_t omega, int64_t delta, int32_t *pair,
                  double *score, ScoreScratch &s) {
    if (L.N == 0) return;
    KScope ks(c, "score_select", 0.0, L.N);
    score_attrs(c);
    ScoreArgs a{L.N, L.inc_off, L.inc_dat, L.pin_off, L.pin_dat, W.wi, L.size, L.in_off, L.in_dat, L.inc_e(), L.in_e(),
                omega, delta, pair, score, s.ctr, s.big, s.ctr + 1, s.heavy, s.ctr + 2, tiers(), 0, L.N};
    const Shard sh = shard_of(c.comm, L.N);
    a.lo = (int32_t)sh.lo;
    a.hi = (int32_t)sh.hi;
    unsigned long long *work = nullptr;
    if (c.profiling) {
        work = c.alloc<unsigned long long>(1);
        c.zero(work, 1);
        a.work = work;
    }
    score_tiers(c, a, W, s, L.N);
    if (work) {  // measured algorithmic bytes (lists actually read) + outputs
        ks.stop();
        unsigned long long h = 0;
        c.d2h(&h, work, 1);
        c.sync();
        ks.set_bytes((double)h + 12.0 * (double)(sh.hi - sh.lo));
        c.free(work);
    }
    if (sh.on) {  // complete (pair, score) from the other ranks' node ranges
        allgather(c, c.comm, pair, sizeof(int32_t), sh.chunk);
        allgather(c, c.comm, score, sizeof(double), sh.chunk);
    }
}

bool score_inc_supported(const Ctx &c, const DWeights &W) {
    (void)c;
    return W.wsum < (1ll << 31) - 2;
}

void score_select_inc(Ctx &c, const DLevel &L, const DWeights &W, int64_t omega, int64_t delta, int32_t *pair,
                      double *score, ScoreScratch &s, const ScoreCarry &cy) {
    const int32_t N = L.N;
    if (N == 0) return;
    KScope ks(c, "score_select", 0.0, L.N);
    score_attrs(c);
    uint8_t *kind = c.alloc<uint8_t>(N);
    int64_t *thr_s = c.alloc<int64_t>(N);
    int32_t *thr_p = c.alloc<int32_t>(N);
    unsigned long long *best = c.alloc<unsigned long long>(N);
    int32_t *list = c.alloc<int32_t>(N), *list2 = c.alloc<int32_t>(N), *lc = c.alloc<int32_t>(4);
    const int64_t cap = 8 * (int64_t)N + (1 << 20);
    int32_t *tv = c.alloc<int32_t>(cap), *tb = c.alloc<int32_t>(cap), *hard = c.alloc<int32_t>(cap);
    int64_t *th = c.alloc<int64_t>(cap);
    int4 *pk = c.alloc<int4>(N);
    c.zero(lc, 4);
    pdl_launch(k_inc_base, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, cy.ma, cy.mb, cy.gamma_prev, cy.prev_pair,
                                                            cy.prev_score, kind, thr_s, thr_p, best, list, lc, L.size, pk);
    DHGP_LAUNCHED(c);
    // pass 1: the merged clusters, emitting their beating neighbour tuples
    ScoreArgs a{N, L.inc_off, L.inc_dat, L.pin_off, L.pin_dat, W.wi, L.size, L.in_off, L.in_dat, L.inc_e(), L.in_e(),
                omega, delta, pair, score, s.ctr, s.big, s.ctr + 1, s.heavy, s.ctr + 2, tiers(), 0, N};
    a.list = list;
    a.list_count = lc;
    a.mb = cy.mb;
    a.rep = cy.ma;
    a.thr_s = thr_s;
    a.thr_p = thr_p;
    a.tup_v = tv;
    a.tup_b = tb;
    a.tup_h = th;
    a.tup_count = lc + 2;
    a.tup_cap = cap;
    a.pk = pk;
    a.heavy_small_list = 2 * c.num_sms;
    // node-range sharding (comm.cuh): each rank rescores the merged clusters
    // and rescore-listed nodes of its range; the per-node best tuple keys are
    // max-reduced across ranks and (pair, score) allgathered at the end
    const Shard sh = shard_of(c.comm, N);
    a.lo = (int32_t)sh.lo;
    a.hi = (int32_t)sh.hi;
    unsigned long long *probe = nullptr;
    if (trace_enabled()) {
        probe = c.alloc<unsigned long long>(4);
        c.zero(probe, 4);
        a.probe = probe;
    }
    unsigned long long *work = nullptr;
    if (c.profiling) {
        work = c.alloc<unsigned long long>(1);
        c.zero(work, 1);
        a.work = work;
    }
    score_tiers(c, a, W, s, N);
    KScope kt(c, "sc_tuples");
    static int gq = resident_grid(c, k_inc_tuples_quick, 256, 0);
    pdl_launch(k_inc_tuples_quick, gq, 256, 0, c.stream, a, best, hard, lc + 3);
    DHGP_LAUNCHED(c);
    static int gt = resident_grid(c, k_inc_tuples, 256, 0);
    pdl_launch(k_inc_tuples, gt, 256, 0, c.stream, a, best, hard, lc + 3);
    DHGP_LAUNCHED(c);
    kt.close();
    if (sh.on) {  // tuples of every rank's clusters; a tuple overflow anywhere rescores everywhere
        allreduce_max_u64(c, c.comm, best, N);
        allreduce_sum_i32(c, c.comm, lc + 2, 1);
    }
    pdl_launch(k_inc_finalize, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, kind, thr_s, thr_p, best, cy.gamma_prev, lc + 2,
                                                                cap, pair, score, list2, lc + 1);
    DHGP_LAUNCHED(c);
    // pass 2: singletons whose carried pair merged and no cluster outranks it
    ScoreArgs b{N, L.inc_off, L.inc_dat, L.pin_off, L.pin_dat, W.wi, L.size, L.in_off, L.in_dat, L.inc_e(), L.in_e(),
                omega, delta, pair, score, s.ctr, s.big, s.ctr + 1, s.heavy, s.ctr + 2, tiers(), 0, N};
    b.list = list2;
    b.list_count = lc + 1;
    b.work = work;
    b.probe = probe;
    b.lo = (int32_t)sh.lo;
    b.hi = (int32_t)sh.hi;
    score_tiers(c, b, W, s, N);
    if (sh.on) {  // every node's (pair, score) from the rank owning it
        allgather(c, c.comm, pair, sizeof(int32_t), sh.chunk);
        allgather(c, c.comm, score, sizeof(double), sh.chunk);
    }
    if (work) {  // measured algorithmic bytes: lists read by both passes, the per-node
                 // carry (pair, score, gamma, members: 24 B) and the tuples (16 B each)
        ks.stop();
        unsigned long long h = 0;
        int32_t nt = 0;
        c.d2h(&h, work, 1);
        c.d2h(&nt, lc + 2, 1);
        c.sync();
        ks.set_bytes((double)h + 36.0 * N + 16.0 * std::min<int64_t>(nt, cap));
        c.free(work);
    }
    if (trace_enabled()) {
        int32_t h[3];
        unsigned long long pr[4];
        c.d2h(h, lc, 3);
        c.d2h(pr, probe, 4);
        c.sync();
        fprintf(stderr, "scoreinc N %d merged %d rescored %d tuples %d warp_nodes %llu warp_iters %llu heavy_nodes %llu heavy_iters %llu\n",
                N, h[0], h[1], h[2], pr[2], pr[0], pr[3], pr[1]);
        c.free(probe);
    }
    for (void *q : {(void *)kind, (void *)thr_s, (void *)thr_p, (void *)best, (void *)list, (void *)list2, (void *)lc,
                    (void *)tv, (void *)tb, (void *)th, (void *)hard, (void *)pk})
        c.free(q);
}

// ===========================================================================
// A7 matching: claims by packed atomics, locks by odd run length of won
// claims toward the root (pointer jumping when a run is long).
// ===========================================================================
namespace {
__device__ __forceinline__ unsigned long long score_bits(double s) {
    return (unsigned long long)__double_as_longlong(s + 0.0);
}
__device__ __forceinline__ bool is_cyc(const int32_t *pair, int32_t v) {
    int32_t p = pair[v];
    return p >= 0 && pair[p] == v;
}
__device__ __forceinline__ bool claimant(const int32_t *pair, int32_t v) {
    int32_t p = pair[v];
    return p >= 0 && !is_cyc(pair, v) && !is_cyc(pair, p);
}

__global__ void k_match_claim1(int32_t N, const int32_t *pair, const double *score, unsigned long long *best,
                               int64_t *status) {
    pdl_entry();
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= N) return;
    int32_t p = pair[v];
    if (p < 0 || is_cyc(pair, (int32_t)v)) return;
    int32_t q = pair[p];
    // Certificate that no cycle of length != 2 exists: along v -> p -> q the
    // (score, id) order must strictly improve (hist symmetry + first-valid
    // selection); a violation triggers the exact sequential check.
    if (q >= 0 && !is_cyc(pair, p) && !(score[p] > score[v] || (score[p] == score[v] && q > (int32_t)v)))
        status[1] = 1;
    if (!is_cyc(pair, p)) atomicMax(&best[p], score_bits(score[v]));
}

__global__ void k_match_claim2(int32_t N, const int32_t *pair, const double *score, const unsigned long long *best,
                               int32_t *claim) {
    pdl_entry();
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= N) return;
    if (!claimant(pair, (int32_t)v)) return;
    int32_t p = pair[v];
    if (score_bits(score[v]) == best[p]) atomicMax(&claim[p], (int32_t)v);
}

__device__ __forceinline__ bool won(const int32_t *pair, const int32_t *claim, int32_t v) {
    return claimant(pair, v) && claim[pair[v]] == v;
}

constexpr int kWalkLimit = 64;

__global__ void k_match_final(int32_t N, const int32_t *pair, const int32_t *claim, const int32_t *runlen,
                              int32_t *match, uint8_t *isrep, int64_t *status) {
    pdl_entry();
    __shared__ int64_t sh[33];
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t moved = 0;
    if (v < N) {
        int32_t r;
        if (runlen) {
            r = runlen[v];
        } else {
            r = 0;
            int32_t u = (int32_t)v;
            while (won(pair, claim, u)) {
                r++;
                u = pair[u];
                if (r > kWalkLimit) {
                    status[2] = 1;
                    break;
                }
            }
        }
        const bool lock = (r & 1) != 0;
        int32_t m;
        if (is_cyc(pair, (int32_t)v) || lock)
            m = pair[v];
        else
            m = claim[v] >= 0 ? claim[v] : (int32_t)v;
        match[v] = m;
        isrep[v] = m >= (int32_t)v;
        moved = m != (int32_t)v;
    }
    int64_t t = block_sum<int64_t>(moved, sh);
    if (threadIdx.x == 0 && t) atomicAdd((unsigned long long *)&status[0], (unsigned long long)t);
}

__global__ void k_pj_init(int32_t N, const int32_t *pair, const int32_t *claim, int32_t *r, int32_t *nxt) {
    pdl_entry();
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= N) return;
    bool wv = won(pair, claim, (int32_t)v);
    r[v] = wv ? 1 : 0;
    nxt[v] = wv ? pair[v] : -1;
}
__global__ void k_pj_step(int32_t N, const int32_t *r0, const int32_t *n0, int32_t *r1, int32_t *n1) {
    pdl_entry();
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= N) return;
    int32_t nx = n0[v];
    r1[v] = r0[v] + (nx >= 0 ? r0[nx] : 0);
    n1[v] = nx >= 0 ? n0[nx] : -1;
}

// exact sequential cycle check, the reference's DFS (_kernels.pyx:124-155)
__global__ void k_cycle_check(int32_t N, const int32_t *pair, int8_t *state, int32_t *path, int32_t *out_len) {
    pdl_entry();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    *out_len = 0;
    for (int32_t s = 0; s < N; s++) {
        if (state[s]) continue;
        int32_t plen = 0, u = s;
        while (state[u] == 0 && pair[u] >= 0) {
            state[u] = 1;
            path[plen++] = u;
            u = pair[u];
        }
        if (state[u] == 1) {
            int32_t i = 0;
            while (path[i] != u) i++;
            if (plen - i != 2) {
                *out_len = plen - i;
                return;
            }
        }
        state[u] = 2;
        for (int32_t k = 0; k < plen; k++) state[path[k]] = 2;
    }
}
}  // namespace

void launch_matching(Ctx &c, int32_t N, const int32_t *pair, const double *score, int32_t *match, uint8_t *isrep,
                     int32_t *claim, int64_t *d_status) {
    if (N == 0) return;
    KScope ks(c, "matching", 32.0 * N);
    unsigned long long *best = c.alloc<unsigned long long>(N);
    c.zero(best, N);
    fill_i32(c, claim, -1, N);
    const unsigned g = (unsigned)cdiv(N, 256);
    pdl_launch(k_match_claim1, g, 256, 0, c.stream, N, pair, score, best, d_status);
    DHGP_LAUNCHED(c);
    pdl_launch(k_match_claim2, g, 256, 0, c.stream, N, pair, score, best, claim);
    DHGP_LAUNCHED(c);
    pdl_launch(k_match_final, g, 256, 0, c.stream, N, pair, claim, nullptr, match, isrep, d_status);
    DHGP_LAUNCHED(c);
    c.free(best);
}

bool matching_fallbacks(Ctx &c, int32_t N, const int32_t *pair, const double *score, int32_t *match,
                        uint8_t *isrep, const int32_t *claim, LevelStatus &st) {
    (void)score;
    bool redo = false;
    if (st.bad_cert) {
        int8_t *state = c.alloc<int8_t>(N);
        int32_t *path = c.alloc<int32_t>(N);
        int32_t *clen = c.alloc<int32_t>(1);
        c.zero(state, N);
        pdl_launch(k_cycle_check, 1, 1, 0, c.stream, N, pair, state, path, clen);
        DHGP_LAUNCHED(c);
        int32_t hl = 0;
        c.d2h(&hl, clen, 1);
        c.sync();
        c.free(state);
        c.free(path);
        c.free(clen);
        if (hl) throw Error{DHGP_ERR_MATCHING, "pairing cycle of length " + std::to_string(hl) + " (expected 2)"};
    }
    if (st.long_run) {  // a long run of won claims: pointer jumping
        const unsigned g = (unsigned)cdiv(N, 256);
        int32_t *r0 = c.alloc<int32_t>(N), *n0 = c.alloc<int32_t>(N);
        int32_t *r1 = c.alloc<int32_t>(N), *n1 = c.alloc<int32_t>(N);
        int64_t *status = c.alloc<int64_t>(kStatusWords);
        c.zero(status, kStatusWords);
        pdl_launch(k_pj_init, g, 256, 0, c.stream, N, pair, claim, r0, n0);
        DHGP_LAUNCHED(c);
        for (int it = 0; it <= bitlen((uint64_t)N); it++) {
            pdl_launch(k_pj_step, g, 256, 0, c.stream, N, r0, n0, r1, n1);
            DHGP_LAUNCHED(c);
            std::swap(r0, r1);
            std::swap(n0, n1);
        }
        pdl_launch(k_match_final, g, 256, 0, c.stream, N, pair, claim, r0, match, isrep, status);
        DHGP_LAUNCHED(c);
        c.d2h(&st.moved, status, 1);
        c.sync();
        c.free(r0);
        c.free(n0);
        c.free(r1);
        c.free(n1);
        c.free(status);
        redo = true;
    }
    return redo;
}

int64_t resolve_matching(Ctx &c, int32_t N, const int32_t *pair, const double *score, int32_t *match,
                         uint8_t *isrep) {
    if (N == 0) return 0;
    int64_t *status = c.alloc<int64_t>(kStatusWords);
    int32_t *claim = c.alloc<int32_t>(N);
    c.zero(status, kStatusWords);
    launch_matching(c, N, pair, score, match, isrep, claim, status);
    LevelStatus st;
    c.d2h((int64_t *)&st, status, kStatusWords);
    c.sync();
    c.free(status);
    matching_fallbacks(c, N, pair, score, match, isrep, claim, st);
    c.free(claim);
    return st.moved / 2;
}

// ===========================================================================
// A9 contraction
// ===========================================================================
namespace {
__global__ void k_gamma(int32_t N, const int32_t *match, const int64_t *rank, const int32_t *size, int32_t *gamma,
                        int32_t *ma, int32_t *mb, int32_t *csize, int32_t *mlist, int32_t *mcount) {
    pdl_entry();
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= N) return;
    int32_t m = match[v];
    int32_t r = m < (int32_t)v ? m : (int32_t)v;
    gamma[v] = (int32_t)rank[r];
    if (r == (int32_t)v) {
        int64_t cn = rank[v];
        ma[cn] = (int32_t)v;
        mb[cn] = m != (int32_t)v ? m : -1;
        if (m != (int32_t)v) mlist[atomicAdd(mcount, 1)] = (int32_t)cn;  // merged clusters (any order)
        // sizes add up; the reference casts the int64 sum to int32 (hgraph.py:226)
        csize[cn] = (int32_t)((int64_t)size[v] + (m != (int32_t)v ? (int64_t)size[m] : 0));
    }
}
// gathers the coarse totals into the status words
__global__ void k_contract_status(int32_t N, int32_t E, const int64_t *rank, const int64_t *so, const int64_t *dof,
                                  const int64_t *po, const int64_t *io, const int64_t *co, int64_t *status,
                                  const unsigned long long *pool_ctr, int64_t fine_sin, int64_t fine_uinc) {
    pdl_entry();
    if (threadIdx.x || blockIdx.x) return;
    const int64_t nc = rank[N];
    status[3] = nc;
    status[4] = so[E];
    status[5] = dof[E];
    status[6] = po[E];
    if (pool_ctr) {  // pooled: totals = fine totals - what the unions removed; the pool's tops
        status[7] = fine_sin - (int64_t)pool_ctr[2];
        status[8] = fine_uinc - (int64_t)pool_ctr[3];
        status[9] = (int64_t)pool_ctr[0];
        status[10] = (int64_t)pool_ctr[1];
    } else {
        status[7] = io[nc];
        status[8] = co[nc];
    }
}

// Per-node families (in, inc) of the coarse level: the sorted union of the
// two members' lists (coarse node_in / node_inc via hgraph.py:221-236 after
// coarsen.py:163-171).  H-edge ids are level-independent and an unmerged
// node keeps its list, so the coarse arrays are the fine arrays with the
// merged clusters' lists replaced by unions: runs of consecutive singleton
// clusters are one contiguous copy, and only the merged clusters (a few
// dozen per level on the SNN shapes) do set arithmetic, a CTA each.
struct NodeFam {
    const int64_t *off;
    const int32_t *dat;
    int64_t *cnt;            // count pass (CSR mode)
    const int64_t *out_off;  // write pass: where the coarse list starts
    int32_t *out;
    const int64_t *end = nullptr;   // fine list ends (DLevel::in_e / inc_e)
    int64_t *obeg = nullptr;        // pooled mode, count pass: coarse begin / end ...
    int64_t *oend = nullptr;
    unsigned long long *top = nullptr;     // ... the pool's next free slot
    unsigned long long *shrink = nullptr;  // ... and the total removed by the unions (|a|+|b|-|a u b|)
};
struct NodeFams {
    NodeFam f[2];
};
constexpr int kNodeChunk = 64;     // coarse nodes per copy work item (<= block size)
constexpr int kUnionStage = 4096;  // shorter member list staged in shared memory up to this length

__device__ __forceinline__ int64_t blk_excl_flags(bool f, int64_t *sh_w, int64_t *total) {
    const int lane = lane_id(), w = warp_id(), nw = blockDim.x >> 5;
    const uint32_t bal = __ballot_sync(FULL_MASK, f);
    if (lane == 0) sh_w[w] = __popc(bal);
    __syncthreads();
    int64_t before = 0, tot = 0;
    for (int j = 0; j < nw; j++) {
        if (j < w) before += sh_w[j];
        tot += sh_w[j];
    }
    __syncthreads();
    *total = tot;
    return before + __popc(bal & ((1u << lane) - 1u));
}

// thread per coarse node: a singleton's count is its member's length; zero
// past nc (the offsets scan runs over the fine count)
// (pooled mode: a singleton keeps its member's list where it is)
__global__ void k_node_count(int64_t nc_cap, const int64_t *d_nc, const int32_t *ma, const int32_t *mb, NodeFams fs) {
    pdl_entry();
    const NodeFam &f = fs.f[blockIdx.y];
    const int64_t nc = *d_nc;
    for (int64_t cn = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; cn < nc_cap;
         cn += (int64_t)gridDim.x * blockDim.x) {
        if (f.obeg) {
            if (cn < nc && mb[cn] < 0) {
                const int32_t a = ma[cn];
                f.obeg[cn] = f.off[a];
                f.oend[cn] = f.end[a];
            }
        } else if (cn >= nc) {
            f.cnt[cn] = 0;
        } else if (mb[cn] < 0) {
            const int32_t a = ma[cn];
            f.cnt[cn] = f.end[a] - f.off[a];
        }
    }
}
// count pass of a merged cluster: the union's length u (CSR: its count;
// pooled: slots reserved at the pool's top)
__device__ __forceinline__ void union_counted(const NodeFam &f, int32_t cn, int64_t na, int64_t nb, int64_t u) {
    if (f.obeg) {
        const int64_t b = (int64_t)atomicAdd(f.top, (unsigned long long)u);
        f.obeg[cn] = b;
        f.oend[cn] = b + u;
        if (na + nb - u) atomicAdd(f.shrink, (unsigned long long)(na + nb - u));
    } else {
        f.cnt[cn] = u;
    }
}

// Merged clusters, a CTA each (any order): the union of the members' sorted
// h-edge lists, |A u B| in the count pass, the list in the write pass.
//  - bitmap: the two lists are set in a shared-memory bitmap over the h-edge
//    ids (when E/8 bytes fit and the lists are long enough to pay for the
//    scan); the union is the set bits in order (block scan of popcounts);
//  - staged: the shorter list S sits in shared memory with, per element, the
//    running count of S-only elements: x = L[i] lands at i + (S-only
//    elements below x), y = S[j] not in L at lb_L(y) + (S-only before j);
//  - otherwise both directions by binary search in global memory.
// The count pass also flags, in emark, the h-edges of the absorbed member:
// only their src / dst / pin lists can map to an unsorted or duplicated
// gamma image (gamma is strictly increasing on the minimum members).
// Small unions (the common case: merged clusters of a few members), a warp
// each: the shorter list S and the running count of its elements absent from
// the longer list L sit in this warp's shared memory; x = L[i] lands at
// i + (S-only elements below x), y = S[j] not in L at lb_L(y) + (S-only
// elements before j).  The count pass is |A| + |B| - |A n B| by searches of
// S in L.  Larger unions are left to k_node_union (one CTA each).
constexpr int kWarpUnionS = 512;   // shorter list length for the warp path
constexpr int kWarpUnionL = 512;   // longer list length for the warp path (longer: a CTA)
constexpr int UW_WARPS = 4;
__device__ __forceinline__ bool warp_union_path(int64_t na, int64_t nb) {
    return min(na, nb) <= kWarpUnionS && max(na, nb) <= kWarpUnionL;
}
template <bool WRITE>
__global__ void __launch_bounds__(UW_WARPS * 32) k_node_union_warp(const int32_t *ma, const int32_t *mb,
                                                                  const int32_t *mlist, const int32_t *mcount,
                                                                  NodeFams fs, uint8_t *emark) {
    pdl_entry();
    __shared__ int32_t s_val[UW_WARPS][kWarpUnionS], s_pre[UW_WARPS][kWarpUnionS + 1];
    const NodeFam &f = fs.f[blockIdx.y];
    const int lane = lane_id(), w = warp_id();
    int32_t *sv = s_val[w], *sp = s_pre[w];
    const int n = *mcount;
    for (int t = blockIdx.x * UW_WARPS + w; t < n; t += gridDim.x * UW_WARPS) {
        const int32_t cn = mlist[t], a = ma[cn], b = mb[cn];
        const int64_t alo = f.off[a], na = f.end[a] - alo, blo = f.off[b], nb = f.end[b] - blo;
        if (!warp_union_path(na, nb)) continue;
        if (!WRITE && emark && blockIdx.y == 1)
            for (int64_t i = lane; i < nb; i += 32) emark[f.dat[blo + i]] = 1;
        const bool a_short = na <= nb;
        const int32_t *S = f.dat + (a_short ? alo : blo), *L = f.dat + (a_short ? blo : alo);
        const int ns = (int)(a_short ? na : nb), nl = (int)(a_short ? nb : na);
        if (!WRITE) {
            int common = 0;
            for (int j = lane; j < ns; j += 32) common += bsearch_dev(L, 0, nl, S[j]) >= 0;
            common = warp_sum(common);
            if (lane == 0) union_counted(f, cn, na, nb, na + nb - common);
            continue;
        }
        int32_t *o = f.out + f.out_off[cn];
        int run = 0;
        for (int j0 = 0; j0 < ns; j0 += 32) {
            const int j = j0 + lane;
            int32_t y = 0;
            int64_t lb = 0;
            bool only = false;
            if (j < ns) {
                y = S[j];
                lb = lower_bound_dev<int32_t>(L, 0, nl, y);
                only = !(lb < nl && L[lb] == y);
                sv[j] = y;
            }
            const uint32_t bal = __ballot_sync(FULL_MASK, only);
            const int ex = run + __popc(bal & ((1u << lane) - 1u));
            if (j < ns) {
                sp[j] = ex;
                if (only) o[lb + ex] = y;
            }
            run += __popc(bal);
        }
        if (lane == 0) sp[ns] = run;
        __syncwarp();
        for (int i = lane; i < nl; i += 32) {
            const int32_t x = L[i];
            o[i + sp[lower_bound_dev<int32_t>(sv, 0, ns, x)]] = x;
        }
        __syncwarp();
    }
}

constexpr int UN_THREADS = 1024;
template <bool WRITE>
__global__ void __launch_bounds__(UN_THREADS) k_node_union(const int32_t *ma, const int32_t *mb, const int32_t *mlist,
                                                           const int32_t *mcount, NodeFams fs, uint8_t *emark,
                                                           int words) {
    pdl_entry();
    extern __shared__ uint32_t s_bm[];
    __shared__ int32_t s_val[kUnionStage], s_pre[kUnionStage + 1];
    __shared__ int64_t sh[32];
    const NodeFam &f = fs.f[blockIdx.y];
    const int n = *mcount;
    for (int t = blockIdx.x; t < n; t += gridDim.x) {
        const int32_t cn = mlist[t], a = ma[cn], b = mb[cn];
        const int64_t alo = f.off[a], na = f.end[a] - alo, blo = f.off[b], nb = f.end[b] - blo;
        if (warp_union_path(na, nb)) continue;  // k_node_union_warp
        if (!WRITE && emark && blockIdx.y == 1)
            for (int64_t i = threadIdx.x; i < nb; i += blockDim.x) emark[f.dat[blo + i]] = 1;
        const bool a_short = na <= nb;
        const int32_t *S = f.dat + (a_short ? alo : blo), *L = f.dat + (a_short ? blo : alo);
        const int64_t ns = a_short ? na : nb, nl = a_short ? nb : na;
        if (words > 0 && na + nb >= 2 * (int64_t)words) {  // the bitmap's clear + scan pays off
            for (int w = threadIdx.x; w < words; w += blockDim.x) s_bm[w] = 0u;
            __syncthreads();
            for (int64_t i = threadIdx.x; i < na; i += blockDim.x) {
                const int32_t x = f.dat[alo + i];
                atomicOr(&s_bm[x >> 5], 1u << (x & 31));
            }
            for (int64_t i = threadIdx.x; i < nb; i += blockDim.x) {
                const int32_t x = f.dat[blo + i];
                atomicOr(&s_bm[x >> 5], 1u << (x & 31));
            }
            __syncthreads();
            const int per = (words + blockDim.x - 1) / blockDim.x;
            const int w0 = min(words, (int)threadIdx.x * per), w1 = min(words, w0 + per);
            int64_t cnt = 0;
            for (int w = w0; w < w1; w++) cnt += __popc(s_bm[w]);
            int64_t tot;
            // exclusive block prefix of the per-thread counts
            const int lane = lane_id(), wp = warp_id(), nwp = blockDim.x >> 5;
            const int64_t incl = warp_incl_scan(cnt);
            if (lane == 31) sh[wp] = incl;
            __syncthreads();
            int64_t before = 0;
            tot = 0;
            for (int j = 0; j < nwp; j++) {
                if (j < wp) before += sh[j];
                tot += sh[j];
            }
            before += incl - cnt;
            if (WRITE) {
                int32_t *o = f.out + f.out_off[cn] + before;
                for (int w = w0; w < w1; w++) {
                    uint32_t bits = s_bm[w];
                    while (bits) {
                        const int bpos = __ffs(bits) - 1;
                        bits &= bits - 1;
                        *o++ = w * 32 + bpos;
                    }
                }
            } else if (threadIdx.x == 0) {
                union_counted(f, cn, na, nb, tot);
            }
            __syncthreads();
            continue;
        }
        if (!WRITE) {
            int64_t common = 0;
            for (int64_t i = threadIdx.x; i < ns; i += blockDim.x) common += bsearch_dev(L, 0, nl, S[i]) >= 0;
            const int64_t tot = block_sum<int64_t>(common, sh);
            if (threadIdx.x == 0) union_counted(f, cn, na, nb, na + nb - tot);
            __syncthreads();
            continue;
        }
        int32_t *o = f.out + f.out_off[cn];
        if (ns <= kUnionStage) {
            int64_t run = 0;
            for (int64_t base = 0; base < ns; base += blockDim.x) {
                const int64_t j = base + threadIdx.x;
                bool only = false;
                int32_t y = 0;
                int64_t lb = 0;
                if (j < ns) {
                    y = S[j];
                    lb = lower_bound_dev<int32_t>(L, 0, nl, y);
                    only = !(lb < nl && L[lb] == y);
                    s_val[j] = y;
                }
                int64_t tot;
                const int64_t ex = blk_excl_flags(only, sh, &tot);
                if (j < ns) {
                    s_pre[j] = (int32_t)(run + ex);
                    if (only) o[lb + run + ex] = y;
                }
                run += tot;
            }
            if (threadIdx.x == 0) s_pre[ns] = (int32_t)run;
            __syncthreads();
            const int B = blockDim.x;
            int64_t i = threadIdx.x;
            for (; i + B < nl; i += 2 * B) {
                const int32_t x0 = L[i], x1 = L[i + B];
                const int64_t p0 = lower_bound_dev<int32_t>(s_val, 0, ns, x0);
                const int64_t p1 = lower_bound_dev<int32_t>(s_val, 0, ns, x1);
                o[i + s_pre[p0]] = x0;
                o[i + B + s_pre[p1]] = x1;
            }
            for (; i < nl; i += B) {
                const int32_t x = L[i];
                o[i + s_pre[lower_bound_dev<int32_t>(s_val, 0, ns, x)]] = x;
            }
            __syncthreads();
            continue;
        }
        const int32_t *A = f.dat + alo, *Bl = f.dat + blo;
        int64_t run = 0;
        for (int64_t base = 0; base < na; base += blockDim.x) {
            const int64_t i = base + threadIdx.x;
            int64_t lb = 0;
            bool in_other = false;
            int32_t x = 0;
            if (i < na) {
                x = A[i];
                lb = lower_bound_dev<int32_t>(Bl, 0, nb, x);
                in_other = lb < nb && Bl[lb] == x;
            }
            int64_t tot;
            const int64_t ex = blk_excl_flags(in_other, sh, &tot);
            if (i < na) o[i + lb - (run + ex)] = x;
            run += tot;
        }
        run = 0;
        for (int64_t base = 0; base < nb; base += blockDim.x) {
            const int64_t j = base + threadIdx.x;
            int64_t lb = 0;
            bool in_other = false;
            int32_t y = 0;
            if (j < nb) {
                y = Bl[j];
                lb = lower_bound_dev<int32_t>(A, 0, na, y);
                in_other = lb < na && A[lb] == y;
            }
            int64_t tot;
            const int64_t ex = blk_excl_flags(in_other, sh, &tot);
            if (j < nb && !in_other) o[lb + j - (run + ex)] = y;
            run += tot;
        }
    }
}

// Singleton lists.  Work item = (chunk of kNodeChunk coarse nodes, slice):
// a chunk of consecutive singletons (no merged cluster and no absorbed member
// between them) is one contiguous range, split over `split` CTAs; otherwise
// its singleton lists are flattened over the CTAs of the chunk (a slot's list
// is found by a search over the chunk's prefix).  Merged clusters are skipped.
__global__ void __launch_bounds__(256) k_node_write(int64_t nc, int split, const int32_t *ma, const int32_t *mb,
                                                    NodeFams fs) {
    pdl_entry();
    const NodeFam &f = fs.f[blockIdx.y];
    __shared__ int64_t s_src[kNodeChunk], s_dst[kNodeChunk], s_end[kNodeChunk];
    const int64_t nch = (nc + kNodeChunk - 1) / kNodeChunk;
    const int64_t items = nch * split;
    const int64_t stride = (int64_t)split * blockDim.x;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const int64_t ch = it / split, sl = it - ch * split;
        const int64_t c0 = ch * kNodeChunk, c1 = min(nc, c0 + kNodeChunk);
        const int64_t cn = c0 + threadIdx.x;
        const int32_t a0 = ma[c0];
        bool clean = true;
        if (cn < c1) clean = mb[cn] < 0 && ma[cn] == a0 + (int32_t)(cn - c0);
        if (__syncthreads_and(clean)) {
            const int32_t a1 = ma[c1 - 1];
            const int64_t lo = f.off[a0], len = f.end[a1] - lo;
            const int32_t *src = f.dat + lo;
            int32_t *dst = f.out + f.out_off[c0];
            int64_t i = sl * blockDim.x + threadIdx.x;
            for (; i + 3 * stride < len; i += 4 * stride) {
                const int32_t x0 = src[i], x1 = src[i + stride], x2 = src[i + 2 * stride], x3 = src[i + 3 * stride];
                dst[i] = x0;
                dst[i + stride] = x1;
                dst[i + 2 * stride] = x2;
                dst[i + 3 * stride] = x3;
            }
            for (; i < len; i += stride) dst[i] = src[i];
            continue;
        }
        if (threadIdx.x < 32) {
            int64_t len[2] = {0, 0};
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int64_t q = c0 + threadIdx.x + 32 * h;
                if (q < c1 && mb[q] < 0) {
                    const int32_t a = ma[q];
                    s_src[threadIdx.x + 32 * h] = f.off[a];
                    s_dst[threadIdx.x + 32 * h] = f.out_off[q];
                    len[h] = f.end[a] - f.off[a];
                }
            }
            const int64_t i0 = warp_incl_scan(len[0]);
            const int64_t t0 = __shfl_sync(FULL_MASK, i0, 31);
            const int64_t i1 = warp_incl_scan(len[1]) + t0;
            s_end[threadIdx.x] = i0;
            s_end[threadIdx.x + 32] = i1;
        }
        __syncthreads();
        const int64_t total = s_end[kNodeChunk - 1];
        for (int64_t i = sl * blockDim.x + threadIdx.x; i < total; i += stride) {
            int q = 0;  // first list whose end is past i
#pragma unroll
            for (int step = kNodeChunk / 2; step > 0; step >>= 1)
                if (s_end[q + step - 1] <= i) q += step;
            const int64_t k = i - (q > 0 ? s_end[q - 1] : 0);
            f.out[s_dst[q] + k] = f.dat[s_src[q] + k];
        }
        __syncthreads();
    }
}

// Fused per-h-edge contraction (h-edges of <= 128 pin slots): a warp maps
// each of the src / dst / pin lists through gamma, sorts it in registers
// (skipped when already strictly ascending: gamma is monotone on lists
// without a displaced cluster member) and de-duplicates it by ballots
// (coarsen.py:163-166; hgraph.py:221).  The count pass writes the coarse
// lengths, the write pass the lists at the scanned offsets.
template <int K>
__device__ __forceinline__ int warp_gamma_list(const int32_t *dat, int64_t lo, int len, const int32_t *gamma,
                                               int32_t *out) {
    const int lane = lane_id();
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t v[K];
    bool sorted = true;
#pragma unroll
    for (int k = 0; k < K; k++) {
        const int i = k * 32 + lane;
        v[k] = i < len ? (uint32_t)gamma[dat[lo + i]] : 0xffffffffu;
    }
#pragma unroll
    for (int k = 0; k < K; k++) {
        const int i = k * 32 + lane;
        const uint32_t up = __shfl_up_sync(FULL_MASK, v[k], 1);
        const uint32_t wrap = __shfl_sync(FULL_MASK, v[k > 0 ? k - 1 : 0], 31);
        const uint32_t prev = lane == 0 ? wrap : up;
        if (i > 0 && i < len && !(prev < v[k])) sorted = false;
    }
    if (!__all_sync(FULL_MASK, sorted)) warp_bitonic_sort<K>(v);
    int total = 0;
#pragma unroll
    for (int k = 0; k < K; k++) {
        const int i = k * 32 + lane;
        const uint32_t up = __shfl_up_sync(FULL_MASK, v[k], 1);
        const uint32_t wrap = __shfl_sync(FULL_MASK, v[k > 0 ? k - 1 : 0], 31);
        const uint32_t prev = lane == 0 ? wrap : up;
        const bool head = i < len && (i == 0 || v[k] != prev);
        const uint32_t bal = __ballot_sync(FULL_MASK, head);
        if (out && head) out[total + __popc(bal & lt)] = (int32_t)v[k];
        total += __popc(bal);
    }
    return total;
}
__device__ __forceinline__ int warp_gamma_any(const int32_t *dat, int64_t lo, int len, const int32_t *gamma,
                                              int32_t *out) {
    if (len <= 32) return warp_gamma_list<1>(dat, lo, len, gamma, out);
    if (len <= 64) return warp_gamma_list<2>(dat, lo, len, gamma, out);
    return warp_gamma_list<4>(dat, lo, len, gamma, out);
}
struct EdgeFam {
    const int64_t *off;
    const int32_t *dat;
    int32_t *cnt;            // count pass
    const int64_t *out_off;  // write pass
    int32_t *out;
};
// the common short case (all three lists <= 32): the six loads of the three
// lists are issued together, then each list is finished from registers
__device__ __forceinline__ int warp_gamma_short(uint32_t g, int len, int32_t *out) {
    const int lane = lane_id();
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t v[1] = {lane < len ? g : 0xffffffffu};
    const uint32_t up = __shfl_up_sync(FULL_MASK, v[0], 1);
    const bool ok = lane == 0 || lane >= len || up < v[0];
    if (!__all_sync(FULL_MASK, ok)) warp_bitonic_sort<1>(v);
    const uint32_t prev = __shfl_up_sync(FULL_MASK, v[0], 1);
    const bool head = lane < len && (lane == 0 || v[0] != prev);
    const uint32_t bal = __ballot_sync(FULL_MASK, head);
    if (out && head) out[__popc(bal & lt)] = (int32_t)v[0];
    return __popc(bal);
}
// count pass, thread per h-edge: an h-edge without an absorbed member keeps
// every slot of its three lists (gamma is strictly increasing on the cluster
// minima and the lists are sorted), the others are listed for the warp kernel
__global__ void k_edge_count_bulk(int32_t E, EdgeFam f0, EdgeFam f1, EdgeFam f2, const uint8_t *emark,
                                  int32_t *elist, int32_t *ecount) {
    pdl_entry();
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool marked = e < E && emark[e];
    if (e < E && !marked) {
        f0.cnt[e] = (int32_t)(f0.off[e + 1] - f0.off[e]);
        f1.cnt[e] = (int32_t)(f1.off[e + 1] - f1.off[e]);
        f2.cnt[e] = (int32_t)(f2.off[e + 1] - f2.off[e]);
    }
    const uint32_t bal = __ballot_sync(FULL_MASK, marked);
    if (!bal || !elist) return;
    const int lane = lane_id(), leader = __ffs(bal) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(ecount, __popc(bal));
    base = __shfl_sync(FULL_MASK, base, leader);
    if (marked) elist[base + __popc(bal & ((1u << lane) - 1u))] = (int32_t)e;
}
// Warp per h-edge: the sorted unique gamma image of its three lists.  Count
// pass: over the listed (marked) h-edges only.  Write pass: every h-edge; an
// unmarked one is a plain element-wise map (its image is already strictly
// ascending), a marked one is sorted when needed and de-duplicated.
__global__ void __launch_bounds__(256) k_contract_edges(int32_t E, const int32_t *gamma, EdgeFam f0, EdgeFam f1,
                                                        EdgeFam f2, bool write, const uint8_t *emark,
                                                        const int32_t *elist = nullptr,
                                                        const int32_t *ecount = nullptr) {
    pdl_entry();
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int lane = lane_id();
    const int64_t ne = elist ? (int64_t)*ecount : (int64_t)E;
    for (int64_t idx = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id(); idx < ne; idx += nw) {
        const int64_t e = elist ? elist[idx] : idx;
        const int64_t l0 = f0.off[e], l1 = f1.off[e], l2 = f2.off[e];
        const int n0 = (int)(f0.off[e + 1] - l0), n1 = (int)(f1.off[e + 1] - l1), n2 = (int)(f2.off[e + 1] - l2);
        if (!write && emark && !emark[e]) {  // no absorbed member: the image keeps every slot
            if (lane == 0) {
                f0.cnt[e] = n0;
                f1.cnt[e] = n1;
                f2.cnt[e] = n2;
            }
            continue;
        }
        if (write && emark && !emark[e]) {  // plain map, the three lists' loads issued together
            int32_t *o0 = f0.out + f0.out_off[e], *o1 = f1.out + f1.out_off[e], *o2 = f2.out + f2.out_off[e];
            const int nmax = max(n0, max(n1, n2));
            for (int i = lane; i < nmax; i += 32) {
                const int32_t x0 = i < n0 ? f0.dat[l0 + i] : 0, x1 = i < n1 ? f1.dat[l1 + i] : 0,
                              x2 = i < n2 ? f2.dat[l2 + i] : 0;
                if (i < n0) o0[i] = gamma[x0];
                if (i < n1) o1[i] = gamma[x1];
                if (i < n2) o2[i] = gamma[x2];
            }
            continue;
        }
        if (n0 <= 32 && n1 <= 32 && n2 <= 32) {
            const int32_t x0 = lane < n0 ? f0.dat[l0 + lane] : 0, x1 = lane < n1 ? f1.dat[l1 + lane] : 0,
                          x2 = lane < n2 ? f2.dat[l2 + lane] : 0;
            const uint32_t g0 = lane < n0 ? (uint32_t)gamma[x0] : 0u, g1 = lane < n1 ? (uint32_t)gamma[x1] : 0u,
                           g2 = lane < n2 ? (uint32_t)gamma[x2] : 0u;
            const int c0 = warp_gamma_short(g0, n0, write ? f0.out + f0.out_off[e] : nullptr);
            const int c1 = warp_gamma_short(g1, n1, write ? f1.out + f1.out_off[e] : nullptr);
            const int c2 = warp_gamma_short(g2, n2, write ? f2.out + f2.out_off[e] : nullptr);
            if (!write && lane == 0) {
                f0.cnt[e] = c0;
                f1.cnt[e] = c1;
                f2.cnt[e] = c2;
            }
            continue;
        }
#pragma unroll
        for (int q = 0; q < 3; q++) {
            const EdgeFam &f = q == 0 ? f0 : (q == 1 ? f1 : f2);
            const int64_t lo = f.off[e];
            const int len = (int)(f.off[e + 1] - lo);
            const int n = warp_gamma_any(f.dat, lo, len, gamma, write ? f.out + f.out_off[e] : nullptr);
            if (!write && lane_id() == 0) f.cnt[e] = n;
        }
    }
}

}  // namespace

namespace {
__global__ void k_marked_list(int32_t E, const uint8_t *emark, const int64_t *epos, int32_t *elist, int32_t *ecount) {
    pdl_entry();
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < E && emark[e]) elist[epos[e]] = (int32_t)e;
    if (e == 0) *ecount = (int32_t)epos[E];
}
// Write pass of the unmarked lists: between two marked h-edges every list is
// the element-wise gamma image at a constant shift (fine offset - coarse
// offset), so each family's data array is mapped linearly — 16-byte loads,
// chunks of MG_CHUNK slots per CTA — skipping the marked h-edges' slots (the
// warp kernel writes those).  A CTA finds the marked h-edges inside its
// chunk with one search of the ascending marked list and keeps up to
// MG_LOCAL of them (start, end, shift after) in shared memory.
constexpr int MG_CHUNK = 8192, MG_LOCAL = 256;
__global__ void __launch_bounds__(256, 6) k_map_gaps(int32_t E, const int32_t *gamma, EdgeFam f0, EdgeFam f1, EdgeFam f2,
                                                  const int32_t *elist, const int32_t *ecount) {
    pdl_entry();
    __shared__ int64_t s_b[MG_LOCAL], s_e[MG_LOCAL], s_sh[MG_LOCAL];
    __shared__ int64_t s_base, s_w1;
    __shared__ int s_k0;
    const EdgeFam f = blockIdx.y == 0 ? f0 : (blockIdx.y == 1 ? f1 : f2);
    const int64_t P = f.off[E];
    const int nm = *ecount;
    for (int64_t c0 = (int64_t)blockIdx.x * MG_CHUNK; c0 < P; c0 += (int64_t)gridDim.x * MG_CHUNK) {
        const int64_t c1 = min(P, c0 + MG_CHUNK);
        if (threadIdx.x < 32) {  // first marked h-edge ending after c0: a 32-ary search by warp 0
            const int lane = threadIdx.x;
            int lo = 0, hi = nm;  // answer in [lo, hi]
            while (hi - lo > 0) {
                const int64_t span = hi - lo;
                const int probe = lo + (int)((span * (lane + 1)) / 33);  // 32 pivots inside [lo, hi)
                const bool le = probe < hi && f.off[elist[probe] + 1] <= c0;
                const uint32_t bal = __ballot_sync(FULL_MASK, le);
                // pivots are ascending; the last one that is <= c0 bounds lo, the first one > c0 bounds hi
                const int nle = __popc(bal);
                const int plo = nle > 0 ? __shfl_sync(FULL_MASK, probe, nle - 1) + 1 : lo;
                const int phi = nle < 32 ? __shfl_sync(FULL_MASK, probe, nle) : hi;
                if (plo == lo && phi == hi) {  // span too small for distinct pivots: finish linearly
                    int k = lo;
                    while (k < hi && f.off[elist[k] + 1] <= c0) k++;
                    lo = hi = k;
                } else {
                    lo = plo;
                    hi = phi;
                }
            }
            if (lane == 0) s_k0 = lo;
        }
        __syncthreads();
        int64_t w0 = c0;
        while (w0 < c1) {
            const int k0 = s_k0;
            if (threadIdx.x == 0) {
                const int32_t prev = k0 > 0 ? elist[k0 - 1] : -1;
                s_base = prev >= 0 ? f.off[prev + 1] - f.out_off[prev + 1] : 0;
            }
            // the marked h-edges starting before c1, up to MG_LOCAL of them
            for (int j = threadIdx.x; j < MG_LOCAL; j += blockDim.x) {
                const int k = k0 + j;
                if (k < nm) {
                    const int32_t e = elist[k];
                    const int64_t b = f.off[e];
                    if (b < c1) {
                        s_b[j] = b;
                        s_e[j] = f.off[e + 1];
                        s_sh[j] = f.off[e + 1] - f.out_off[e + 1];
                    } else {
                        s_b[j] = INT64_MAX;
                    }
                } else {
                    s_b[j] = INT64_MAX;
                }
            }
            static_assert(MG_LOCAL == 256, "one local entry per thread");
            const int n = __syncthreads_count(s_b[threadIdx.x] != INT64_MAX);  // loaded entries are a prefix
            if (threadIdx.x == 0) {
                // a full window ends at the last loaded marked h-edge's end
                s_w1 = (n == MG_LOCAL) ? min(c1, s_e[n - 1]) : c1;
                s_k0 = k0 + n;
            }
            __syncthreads();
            const int64_t w1 = s_w1, base = s_base;
            // 16 consecutive slots per thread and pass (four 16-byte loads in
            // flight before the gathers); the local entry is found once per
            // group and advanced within it
            constexpr int G = 8;
            for (int64_t g0 = (w0 & ~(int64_t)3) + G * (int64_t)threadIdx.x; g0 < w1; g0 += G * (int64_t)blockDim.x) {
                int32_t x[G];
#pragma unroll
                for (int q = 0; q < G / 4; q++) {
                    const int64_t i0 = g0 + 4 * q;
                    if (i0 >= w0 && i0 + 4 <= w1) {
                        const int4 v = *(const int4 *)(f.dat + i0);
                        x[4 * q] = v.x; x[4 * q + 1] = v.y; x[4 * q + 2] = v.z; x[4 * q + 3] = v.w;
                    } else {
#pragma unroll
                        for (int u = 0; u < 4; u++) x[4 * q + u] = (i0 + u >= w0 && i0 + u < w1) ? f.dat[i0 + u] : 0;
                    }
                }
                int lo = 0, hi = n;  // last local marked h-edge starting at or before g0
                while (lo < hi) {
                    const int m = (lo + hi) >> 1;
                    if (s_b[m] <= g0) lo = m + 1; else hi = m;
                }
                int jr = lo - 1;
                int32_t y[G];
#pragma unroll
                for (int u = 0; u < G; u++) {
                    const int64_t i = g0 + u;
                    y[u] = (i >= w0 && i < w1) ? gamma[x[u]] : 0;
                }
#pragma unroll
                for (int u = 0; u < G; u++) {
                    const int64_t i = g0 + u;
                    if (i < w0 || i >= w1) continue;
                    while (jr + 1 < n && s_b[jr + 1] <= i) jr++;
                    if (jr >= 0 && i < s_e[jr]) continue;  // a marked list's slot
                    f.out[i - (jr >= 0 ? s_sh[jr] : base)] = y[u];
                }
            }
            __syncthreads();
            w0 = w1;
        }
        __syncthreads();
    }
}
}  // namespace

// words of the union kernel's shared bitmap over the h-edge ids (0 = no
// bitmap: more than ~1.3M h-edges)
static int union_words(Ctx &c, int32_t E) {
    static bool attr = false;
    constexpr int kMaxWords = 40960;  // 160 KB
    if (!attr) {
        DHGP_CUDA(cudaFuncSetAttribute(k_node_union<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kMaxWords));
        DHGP_CUDA(cudaFuncSetAttribute(k_node_union<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kMaxWords));
        attr = true;
    }
    const int64_t w = cdiv((int64_t)E, 32);
    return w <= kMaxWords ? (int)w : 0;
}

void contract_count(Ctx &c, DLevel &fine, const int32_t *match, const uint8_t *isrep, DLevel &coarse,
                    ContractScratch &s, int64_t *d_status, NodePool *pool) {
    // algorithmic bytes: each fine h-edge list entry and its gamma image read
    // once (8 B), per-h-edge offsets read and counts / coarse offsets written
    // (60 B), per-node rank / gamma / members (24 B)
    KScope ks(c, "contract", (double)(8.0 * (fine.Ps + fine.Pd + fine.U) + 60.0 * fine.E + 24.0 * fine.N));
    const int32_t N = fine.N, E = fine.E;
    s.rank = c.alloc<int64_t>((int64_t)N + 1);
    scan_excl<uint8_t>(c, isrep, s.rank, N);
    const int64_t *d_nc = s.rank + N;
    fine.gamma = c.alloc<int32_t>(N);
    s.ma = c.alloc<int32_t>(N);
    s.mb = c.alloc<int32_t>(N);
    coarse.E = E;
    coarse.size = c.alloc<int32_t>(N);  // capacity: the fine node count
    s.mlist = c.alloc<int32_t>(N / 2 + 1);
    s.mcount = c.alloc<int32_t>(1);
    s.emark = c.alloc<uint8_t>(E);
    zero_many(c, {{s.mcount, 4}, {s.emark, E}});
    pdl_launch(k_gamma, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, match, s.rank, fine.size, fine.gamma, s.ma, s.mb,
                                                         coarse.size, s.mlist, s.mcount);
    DHGP_LAUNCHED(c);
    // per-node families first: the merged clusters flag the h-edges whose
    // lists need the sort / de-duplication
    KScope kcn(c, "cc_nodes");
    int64_t *ncnt = pool ? nullptr : c.alloc<int64_t>(2 * (int64_t)N);
    coarse.in_off = c.alloc<int64_t>((int64_t)N + 1);
    coarse.inc_off = c.alloc<int64_t>((int64_t)N + 1);
    unsigned long long *pool_ctr = nullptr;  // pooled: [0..1] pool tops (in, inc), [2..3] union shrink
    if (pool) {
        coarse.in_end = c.alloc<int64_t>(N);
        coarse.inc_end = c.alloc<int64_t>(N);
        coarse.pooled = true;
        coarse.in_dat = pool->dat[0];
        coarse.inc_dat = pool->dat[1];
        s.pool_ctr = pool_ctr = c.alloc<unsigned long long>(4);
        c.d2d((int64_t *)pool_ctr, pool->top, 2);
        c.zero(pool_ctr + 2, 2);
    }
    {
        NodeFams fs{{NodeFam{fine.in_off, fine.in_dat, ncnt, nullptr, nullptr},
                     NodeFam{fine.inc_off, fine.inc_dat, ncnt ? ncnt + N : nullptr, nullptr, nullptr}}};
        fs.f[0].end = fine.in_e();
        fs.f[1].end = fine.inc_e();
        if (pool) {
            fs.f[0].obeg = coarse.in_off;
            fs.f[0].oend = coarse.in_end;
            fs.f[1].obeg = coarse.inc_off;
            fs.f[1].oend = coarse.inc_end;
            fs.f[0].top = pool_ctr;
            fs.f[1].top = pool_ctr + 1;
            fs.f[0].shrink = pool_ctr + 2;
            fs.f[1].shrink = pool_ctr + 3;
        }
        const unsigned ga = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(N, 256), (int64_t)c.num_sms * 8));
        pdl_launch(k_node_count, dim3(ga, 2), 256, 0, c.stream, N, d_nc, s.ma, s.mb, fs);
        DHGP_LAUNCHED(c);
        const int words = union_words(c, E);
        pdl_launch(k_node_union_warp<false>, dim3(4 * c.num_sms, 2), UW_WARPS * 32, 0, c.stream, s.ma, s.mb, s.mlist,
                   s.mcount, fs, s.emark);
        DHGP_LAUNCHED(c);
        pdl_launch(k_node_union<false>, dim3(c.num_sms, 2), UN_THREADS, 4 * words, c.stream, s.ma, s.mb, s.mlist, s.mcount, fs,
                                                                                     s.emark, words);
        DHGP_LAUNCHED(c);
    }
    if (!pool) {
        scan_excl3<int64_t>(c, ncnt, coarse.in_off, ncnt + N, coarse.inc_off, nullptr, nullptr, N);
        c.free(ncnt);
    }
    kcn.close();
    // per-h-edge families: sorted unique gamma image (coarsen.py:163-166)
    KScope kcs(c, "cc_edges");
    coarse.maxp = fine.maxp;
    // lists of <= 128 slots: counts in bulk + a warp per marked h-edge, then
    // the linear gap map (contract_write); longer lists: segmented sorts
    s.fused = fine.maxp <= 128;
    if (s.fused) {
        int32_t *cnt = c.alloc<int32_t>(3 * (int64_t)E);
        if (E > 0) {
            const EdgeFam f0{fine.src_off, fine.src_dat, cnt}, f1{fine.dst_off, fine.dst_dat, cnt + E},
                f2{fine.pin_off, fine.pin_dat, cnt + 2 * (int64_t)E};
            // unmarked h-edges in bulk (thread per h-edge), the marked ones
            // (ascending, kept for the write pass) a warp each
            // (the write pass's gap map needs the list ascending: a scan of the
            // marks when there are many h-edges; else the bulk kernel's list)
            s.elist = c.alloc<int32_t>(E);
            s.ecount = c.alloc<int32_t>(1);
            const bool sorted_list = (int64_t)E >= 32 * 48 * (int64_t)c.num_sms;
            c.zero(s.ecount, 1);
            pdl_launch(k_edge_count_bulk, (unsigned)cdiv(E, 256), 256, 0, c.stream, E, f0, f1, f2, s.emark,
                       sorted_list ? (int32_t *)nullptr : s.elist, s.ecount);
            DHGP_LAUNCHED(c);
            if (sorted_list) {
                s.epos = c.alloc<int64_t>((int64_t)E + 1);
                scan_excl<uint8_t>(c, s.emark, s.epos, E);
                pdl_launch(k_marked_list, (unsigned)cdiv(E, 256), 256, 0, c.stream, E, s.emark, s.epos, s.elist,
                           s.ecount);
                DHGP_LAUNCHED(c);
            }
            static int g = resident_grid(c, k_contract_edges, 256, 0);
            const unsigned gr = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(E, 8), g));
            pdl_launch(k_contract_edges, gr, 256, 0, c.stream, E, fine.gamma, f0, f1, f2, false, s.emark,
                       (const int32_t *)s.elist, (const int32_t *)s.ecount);
            DHGP_LAUNCHED(c);
        }
        coarse.src_off = c.alloc<int64_t>((int64_t)E + 1);
        coarse.dst_off = c.alloc<int64_t>((int64_t)E + 1);
        coarse.pin_off = c.alloc<int64_t>((int64_t)E + 1);
        scan_excl3<int32_t>(c, cnt, coarse.src_off, cnt + E, coarse.dst_off, cnt + 2 * (int64_t)E, coarse.pin_off,
                            E);
        c.free(cnt);
    } else {
    s.tmp_src = c.alloc<int32_t>(fine.Ps);
    s.tmp_dst = c.alloc<int32_t>(fine.Pd);
    s.tmp_pin = c.alloc<int32_t>(fine.U);
    int64_t *cnt = c.alloc<int64_t>(E);
    seg_sort(c, E, fine.src_off, fine.src_dat, fine.gamma, s.tmp_src);
    seg_unique_count(c, E, fine.src_off, s.tmp_src, cnt);
    coarse.src_off = c.alloc<int64_t>((int64_t)E + 1);
    scan_excl<int64_t>(c, cnt, coarse.src_off, E);
    seg_sort(c, E, fine.dst_off, fine.dst_dat, fine.gamma, s.tmp_dst);
    seg_unique_count(c, E, fine.dst_off, s.tmp_dst, cnt);
    coarse.dst_off = c.alloc<int64_t>((int64_t)E + 1);
    scan_excl<int64_t>(c, cnt, coarse.dst_off, E);
    seg_sort(c, E, fine.pin_off, fine.pin_dat, fine.gamma, s.tmp_pin);
    seg_unique_count(c, E, fine.pin_off, s.tmp_pin, cnt);
    coarse.pin_off = c.alloc<int64_t>((int64_t)E + 1);
    scan_excl<int64_t>(c, cnt, coarse.pin_off, E);
    c.free(cnt);
    }
    kcs.close();
    pdl_launch(k_contract_status, 1, 32, 0, c.stream, N, E, s.rank, coarse.src_off, coarse.dst_off, coarse.pin_off,
               coarse.in_off, coarse.inc_off, d_status, (const unsigned long long *)pool_ctr, fine.Sin, fine.U);
    DHGP_LAUNCHED(c);
}

// the merged clusters' node lists (and, CSR mode, the singletons' copies)
static void node_merge_launch(Ctx &c, DLevel &fine, DLevel &coarse, ContractScratch &s, const LevelStatus &st,
                              NodePool *pool, cudaStream_t stream) {
    NodeFams fs{{NodeFam{fine.in_off, fine.in_dat, nullptr, coarse.in_off, coarse.in_dat},
                 NodeFam{fine.inc_off, fine.inc_dat, nullptr, coarse.inc_off, coarse.inc_dat}}};
    fs.f[0].end = fine.in_e();
    fs.f[1].end = fine.inc_e();
    if (!pool) {  // CSR: the singletons' lists are copied (pooled: they stay where they are)
        // slices per chunk: about 4K list entries per CTA
        const int64_t per_chunk = cdiv(std::max(fine.Sin, fine.U) * kNodeChunk, std::max<int64_t>(1, fine.N));
        const int split = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(per_chunk, 4096), 64));
        const int64_t items = cdiv(st.nc, kNodeChunk) * split;
        const unsigned g = (unsigned)std::min<int64_t>(items, (int64_t)c.num_sms * 16);
        pdl_launch(k_node_write, dim3(g, 2), 256, 0, stream, st.nc, split, s.ma, s.mb, fs);
        DHGP_LAUNCHED(c);
    }
    const int words = union_words(c, fine.E);
    pdl_launch(k_node_union_warp<true>, dim3(4 * c.num_sms, 2), UW_WARPS * 32, 0, stream, s.ma, s.mb, s.mlist,
               s.mcount, fs, nullptr);
    DHGP_LAUNCHED(c);
    pdl_launch(k_node_union<true>, dim3(c.num_sms, 2), UN_THREADS, 4 * words, stream, s.ma, s.mb, s.mlist, s.mcount,
               fs, nullptr, words);
    DHGP_LAUNCHED(c);
}

void contract_write(Ctx &c, DLevel &fine, DLevel &coarse, ContractScratch &s, const LevelStatus &st,
                    NodePool *pool) {
    // algorithmic bytes: fine h-edge lists + gamma read (8 B per entry), coarse
    // lists written (4 B), fine node lists read and coarse ones written (4 B
    // each), offsets (16 B per h-edge, 16 B per coarse node)
    KScope ks(c, "contract_write",
              (double)(8.0 * (fine.Ps + fine.Pd + fine.U) + 4.0 * (st.ps + st.pd + st.u) +
                       4.0 * (fine.Sin + fine.U) + 4.0 * (st.sin + st.uinc) + 16.0 * fine.E + 16.0 * st.nc));
    const int32_t E = fine.E;
    coarse.N = (int32_t)st.nc;
    coarse.Ps = st.ps;
    coarse.Pd = st.pd;
    coarse.U = st.u;
    coarse.Sin = st.sin;
    {
        KScope k1(c, "cw_alloc");
        coarse.src_dat = c.alloc<int32_t>(st.ps);
        coarse.dst_dat = c.alloc<int32_t>(st.pd);
        coarse.pin_dat = c.alloc<int32_t>(st.u);
        if (!pool) {
            coarse.in_dat = c.alloc<int32_t>(st.sin);
            coarse.inc_dat = c.alloc<int32_t>(st.uinc);
        } else {  // the pool may have grown since the count pass
            coarse.in_dat = pool->dat[0];
            coarse.inc_dat = pool->dat[1];
            c.h2d(pool->top, st.pool_top, 2);
        }
    }
    // the node lists of the merged clusters (cw_merge) and the h-edge lists
    // (cw_unique) are independent: the merge runs on the side stream, forked
    // here and joined below, so its latency-bound union kernels overlap the
    // h-edge rewrite
    const bool fork = c.side && st.nc > 0;
    if (fork) {
        DHGP_CUDA(cudaEventRecord(c.ev_fork, c.stream));
        DHGP_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
        node_merge_launch(c, fine, coarse, s, st, pool, c.side);
        DHGP_CUDA(cudaEventRecord(c.ev_join, c.side));
    }
    {
        KScope k2(c, "cw_unique");
        if (s.fused) {
            if (E > 0) {
                const EdgeFam f0{fine.src_off, fine.src_dat, nullptr, coarse.src_off, coarse.src_dat},
                    f1{fine.dst_off, fine.dst_dat, nullptr, coarse.dst_off, coarse.dst_dat},
                    f2{fine.pin_off, fine.pin_dat, nullptr, coarse.pin_off, coarse.pin_dat};
                static int g = resident_grid(c, k_contract_edges, 256, 0);
                const unsigned gr = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(E, 8), g));
                if ((int64_t)E < 32 * 48 * (int64_t)c.num_sms) {
                    // few h-edges (a few per resident warp): a warp per h-edge, the
                    // unmarked ones as plain maps
                    pdl_launch(k_contract_edges, gr, 256, 0, c.stream, E, fine.gamma, f0, f1, f2, true,
                               (const uint8_t *)s.emark, (const int32_t *)nullptr, (const int32_t *)nullptr);
                    DHGP_LAUNCHED(c);
                } else {
                    // marked lists: sorted / de-duplicated images, a warp each
                    pdl_launch(k_contract_edges, gr, 256, 0, c.stream, E, fine.gamma, f0, f1, f2, true,
                               (const uint8_t *)nullptr, (const int32_t *)s.elist, (const int32_t *)s.ecount);
                    DHGP_LAUNCHED(c);
                    // everything else: linear element-wise map at the per-gap shift
                    const int64_t pmax = std::max(std::max(fine.Ps, fine.Pd), fine.U);
                    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(pmax, MG_CHUNK),
                                                                                        (int64_t)c.num_sms * 8));
                    pdl_launch(k_map_gaps, dim3(gx, 3), 256, 0, c.stream, E, fine.gamma, f0, f1, f2,
                               (const int32_t *)s.elist, (const int32_t *)s.ecount);
                    DHGP_LAUNCHED(c);
                }
            }
        } else {
            seg_unique_write(c, E, fine.src_off, s.tmp_src, coarse.src_off, coarse.src_dat);
            seg_unique_write(c, E, fine.dst_off, s.tmp_dst, coarse.dst_off, coarse.dst_dat);
            seg_unique_write(c, E, fine.pin_off, s.tmp_pin, coarse.pin_off, coarse.pin_dat);
        }
    }
    if (fork) {
        DHGP_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
    } else if (st.nc > 0) {
        KScope k2(c, "cw_merge");
        node_merge_launch(c, fine, coarse, s, st, pool, c.stream);
    }
    int32_t *ma = s.ma, *mb = s.mb;
    s.ma = s.mb = nullptr;
    contract_release(c, s);
    s.ma = ma;
    s.mb = mb;
}

namespace {
__global__ void k_members(int32_t N, const int32_t *gamma, int32_t *lo, int32_t *hi) {
    pdl_entry();
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= N) return;
    atomicMin(&lo[gamma[v]], (int32_t)v);
    atomicMax(&hi[gamma[v]], (int32_t)v);
}
__global__ void k_match_of(int32_t N, const int32_t *gamma, const int32_t *lo, const int32_t *hi, int32_t *match,
                           uint8_t *isrep) {
    pdl_entry();
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= N) return;
    const int32_t a = lo[gamma[v]], b = hi[gamma[v]];
    match[v] = (int32_t)v == a ? b : a;
    isrep[v] = (int32_t)v == a;
}
}  // namespace

void match_from_gamma(Ctx &c, int32_t N, int32_t nc, const int32_t *gamma, int32_t *match, uint8_t *isrep) {
    if (N == 0) return;
    int32_t *lo = c.alloc<int32_t>(nc), *hi = c.alloc<int32_t>(nc);
    fill_i32(c, lo, 0x7fffffff, nc);
    fill_i32(c, hi, -1, nc);
    pdl_launch(k_members, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, gamma, lo, hi);
    DHGP_LAUNCHED(c);
    pdl_launch(k_match_of, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, gamma, lo, hi, match, isrep);
    DHGP_LAUNCHED(c);
    c.free(lo);
    c.free(hi);
}

void level_to_stub(Ctx &c, DLevel &L) {
    int32_t *g = L.gamma;
    L.gamma = nullptr;
    DLevel keep;
    keep.N = L.N;
    keep.E = L.E;
    keep.Ps = L.Ps;
    keep.Pd = L.Pd;
    keep.U = L.U;
    keep.Sin = L.Sin;
    keep.maxp = L.maxp;
    L.release(c);
    L = keep;
    L.gamma = g;
    L.stub = true;
}

void contract_release_members(Ctx &c, ContractScratch &s) {
    c.free(s.ma);
    c.free(s.mb);
    s.ma = s.mb = nullptr;
}

void contract_release(Ctx &c, ContractScratch &s) {
    c.free(s.ma);
    c.free(s.mb);
    c.free(s.tmp_src);
    c.free(s.tmp_dst);
    c.free(s.tmp_pin);
    c.free(s.rank);
    c.free(s.mlist);
    c.free(s.mcount);
    c.free(s.emark);
    c.free(s.elist);
    c.free(s.ecount);
    c.free(s.epos);
    c.free(s.pool_ctr);
    s = ContractScratch();
}

void node_pool_init(Ctx &c, NodePool &pool, DLevel &L0, double factor) {
    const int64_t n[2] = {L0.Sin, L0.U};
    int32_t *src[2] = {L0.in_dat, L0.inc_dat};
    pool.top = c.alloc<int64_t>(2);
    for (int f = 0; f < 2; f++) {
        pool.cap[f] = (int64_t)(factor * (double)n[f]) + (1 << 20);
        pool.dat[f] = c.alloc<int32_t>(pool.cap[f]);
        c.d2d(pool.dat[f], src[f], n[f]);
        c.free(src[f]);
    }
    c.h2d(pool.top, n, 2);
    L0.in_dat = pool.dat[0];
    L0.inc_dat = pool.dat[1];
    L0.pooled = true;
}

void node_pool_fit(Ctx &c, NodePool &pool, const int64_t top[2], std::vector<DLevel> &levels, DLevel *extra) {
    for (int f = 0; f < 2; f++) {
        if (top[f] <= pool.cap[f]) continue;
        const int64_t cap = std::max<int64_t>(2 * pool.cap[f], top[f] + (top[f] >> 1));
        int32_t *d = c.alloc<int32_t>(cap);
        c.d2d(d, pool.dat[f], pool.cap[f]);
        int32_t *old = pool.dat[f];
        for (auto &L : levels)
            if (L.pooled) (f ? L.inc_dat : L.in_dat) = d;
        if (extra && extra->pooled) (f ? extra->inc_dat : extra->in_dat) = d;
        c.free(old);
        pool.dat[f] = d;
        pool.cap[f] = cap;
    }
}

}  // namespace dhgp
