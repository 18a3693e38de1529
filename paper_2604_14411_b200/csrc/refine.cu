// refine.cu — refinement rounds, exact-integer mode.
//
// The reference's dense (E x K) pins / pins_in matrices (_kernels.pyx:216-231)
// become per-h-edge run lists: for h-edge e, the distinct parts of its pins in
// ascending order with their pin count and destination-pin count, stored at
// e's own pin offsets (lambda(e) <= |pins(e)| entries).  Every value the
// algorithm reads from pins[e, p] / pins_in[e, p] is a binary search in that
// list (absent = 0), so the results are identical.
#include "comm.cuh"
#include "prims.cuh"
#include "refine.cuh"

namespace dhgp {

namespace {

struct Runs {
    const int64_t *off = nullptr;  // [E+1] run base per h-edge (>= |pins(e)| slots each)
    // [2U] per run slot k: pc[2k] = the part (ascending within an h-edge),
    // pc[2k+1] = the h-edge's pins in that part — interleaved so that one
    // sector serves both (the proposal tiers read them together)
    int32_t *pc = nullptr;
    int32_t *cin = nullptr;   // [U] destination pins of the h-edge in that part
    int32_t *len = nullptr;   // [E] lambda(e)
};

// Rounds are launched speculatively for up to kSpecCap movers before the
// host knows M (one host sync per round instead of two); kernels of such a
// launch are no-ops when M turns out larger, and the host redoes the tail.
constexpr int64_t kSpecCap = kSmallSort;

__device__ __forceinline__ int32_t run_find(const Runs &r, int64_t lo, int32_t len, int32_t p) {
    int64_t a = lo, b = lo + len;  // lower bound of p among the parts pc[2a], ...
    while (a < b) {
        const int64_t mid = (a + b) >> 1;
        if (r.pc[2 * mid] < p)
            a = mid + 1;
        else
            b = mid;
    }
    const int64_t k = a;
    return (k < lo + len && r.pc[2 * (k)] == p) ? (int32_t)(k - lo) : -1;
}

// per h-edge: run lists from the per-edge sorted parts, connectivity
// contribution w(e)(lambda-1) (_kernels.pyx:184-213) and distinct-inbound
// counts (hgraph.py:324-339)
__global__ void k_edge_runs(int32_t E, const int64_t *pin_off, const int32_t *sorted_parts, const int64_t *dst_off,
                            const int32_t *dst_dat, const int32_t *assign, const int64_t *wi, Runs r,
                            unsigned long long *conn, int64_t *pinbound) {
    pdl_entry();
    __shared__ int64_t sh[33];
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t contrib = 0;
    if (e < E) {
        const int64_t plo = pin_off[e], hi = pin_off[e + 1], lo = r.off[e];
        int32_t lam = 0;
        for (int64_t j = plo; j < hi;) {
            int32_t p = sorted_parts[j];
            int64_t j2 = j + 1;
            while (j2 < hi && sorted_parts[j2] == p) j2++;
            r.pc[2 * (lo + lam)] = p;
            r.pc[2 * (lo + lam) + 1] = (int32_t)(j2 - j);
            r.cin[lo + lam] = 0;
            lam++;
            j = j2;
        }
        r.len[e] = lam;
        for (int64_t q = dst_off[e]; q < dst_off[e + 1]; q++) {
            int32_t k = run_find(r, lo, lam, assign[dst_dat[q]]);
            r.cin[lo + k]++;
        }
        if (pinbound)
            for (int32_t k = 0; k < lam; k++)
                if (r.cin[lo + k] > 0) atomicAdd((unsigned long long *)&pinbound[r.pc[2 * (lo + k)]], 1ull);
        if (lam > 0) contrib = wi[e] * (int64_t)(lam - 1);
    }
    int64_t t = block_sum<int64_t>(contrib, sh);
    if (threadIdx.x == 0 && t) atomicAdd(conn, (unsigned long long)t);
}

// warp-per-h-edge variant for wide h-edges (average pins >= 12)
__global__ void k_edge_runs_warp(int32_t E, const int64_t *pin_off, const int32_t *sorted_parts,
                                 const int64_t *dst_off, const int32_t *dst_dat, const int32_t *assign,
                                 const int64_t *wi, Runs r, unsigned long long *conn, int64_t *pinbound) {
    pdl_entry();
    const int lane = lane_id();
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    int64_t contrib = 0;
    for (int64_t e = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id(); e < E; e += nw) {
        const int64_t plo = pin_off[e], len = pin_off[e + 1] - plo, lo = r.off[e];
        int32_t lam = 0;
        for (int64_t b = 0; b < len; b += 32) {  // heads of the sorted runs
            const int64_t i = b + lane;
            int32_t p = 0;
            bool head = false;
            if (i < len) {
                p = sorted_parts[plo + i];
                head = i == 0 || sorted_parts[plo + i - 1] != p;
            }
            const uint32_t bal = __ballot_sync(FULL_MASK, head);
            if (head) {
                const int32_t j = lam + __popc(bal & lt);
                r.pc[2 * (lo + j)] = p;
                r.pc[2 * (lo + j) + 1] = (int32_t)i;  // run start for now
                r.cin[lo + j] = 0;
            }
            lam += __popc(bal);
        }
        __syncwarp();
        for (int32_t j = lane; j < lam; j += 32) {
            const int32_t st = r.pc[2 * (lo + j) + 1];
            const int32_t nx = j + 1 < lam ? r.pc[2 * (lo + j + 1) + 1] : (int32_t)len;
            __syncwarp(__activemask());
            r.pc[2 * (lo + j) + 1] = nx - st;
        }
        __syncwarp();
        // second pass turns starts into lengths; the loop above may race when
        // lam > 32, so recompute those from the sorted parts directly
        if (lam > 32) {
            for (int32_t j = lane; j < lam; j += 32) {
                const int32_t p = r.pc[2 * (lo + j)];
                int64_t a0 = lower_bound_dev<int32_t>(sorted_parts, plo, plo + len, p);
                int64_t a1 = lower_bound_dev<int32_t>(sorted_parts, plo, plo + len, p + 1);
                r.pc[2 * (lo + j) + 1] = (int32_t)(a1 - a0);
            }
            __syncwarp();
        }
        if (lane == 0) r.len[e] = lam;
        for (int64_t q = dst_off[e] + lane; q < dst_off[e + 1]; q += 32) {
            const int32_t k = run_find(r, lo, lam, assign[dst_dat[q]]);
            atomicAdd(&r.cin[lo + k], 1);
        }
        __syncwarp();
        if (pinbound)
            for (int32_t j = lane; j < lam; j += 32)
                if (r.cin[lo + j] > 0) atomicAdd((unsigned long long *)&pinbound[r.pc[2 * (lo + j)]], 1ull);
        if (lane == 0 && lam > 0) contrib += wi[e] * (int64_t)(lam - 1);
    }
    if (lane == 0 && contrib) atomicAdd(conn, (unsigned long long)contrib);
}

// Fused run lists for h-edges of <= 128 pins: a warp maps the pins to parts,
// sorts them in registers (bitonic) and derives the runs from ballots; no
// temporary array and one launch per round.
template <int K>
__device__ __forceinline__ int32_t warp_edge_runs(int64_t e, int64_t plo, int64_t lo, int len, const int32_t *pin_dat,
                                                  const int64_t *dst_off, const int32_t *dst_dat,
                                                  const int32_t *assign, Runs r, int64_t *pinbound) {
    const int lane = lane_id();
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t v[K];
#pragma unroll
    for (int k = 0; k < K; k++) {
        const int i = k * 32 + lane;
        v[k] = i < len ? (uint32_t)assign[pin_dat[plo + i]] : 0xffffffffu;
    }
    warp_bitonic_sort<K>(v);
    uint32_t bal[K];
    bool head[K];
#pragma unroll
    for (int k = 0; k < K; k++) {
        const int i = k * 32 + lane;
        const uint32_t up = __shfl_up_sync(FULL_MASK, v[k], 1);
        const uint32_t wrap = __shfl_sync(FULL_MASK, v[k > 0 ? k - 1 : 0], 31);
        const uint32_t prev = lane == 0 ? wrap : up;
        head[k] = i < len && (i == 0 || v[k] != prev);
        bal[k] = __ballot_sync(FULL_MASK, head[k]);
    }
    int32_t before = 0;
#pragma unroll
    for (int k = 0; k < K; k++) {
        if (head[k]) {
            const int i = k * 32 + lane;
            const uint32_t rest = bal[k] & ~((2u << lane) - 1u);
            int next = len;
            if (rest) {
                next = k * 32 + __ffs(rest) - 1;
            } else {
#pragma unroll
                for (int k2 = K - 1; k2 > k; k2--)
                    if (bal[k2]) next = k2 * 32 + __ffs(bal[k2]) - 1;
            }
            const int32_t j = before + __popc(bal[k] & lt);
            r.pc[2 * (lo + j)] = (int32_t)v[k];
            r.pc[2 * (lo + j) + 1] = next - i;
            r.cin[lo + j] = 0;
        }
        before += __popc(bal[k]);
    }
    const int32_t lam = before;
    __syncwarp();
    for (int64_t q = dst_off[e] + lane; q < dst_off[e + 1]; q += 32) {
        const int32_t k = run_find(r, lo, lam, assign[dst_dat[q]]);
        atomicAdd(&r.cin[lo + k], 1);
    }
    __syncwarp();
    if (pinbound)
        for (int32_t j = lane; j < lam; j += 32)
            if (r.cin[lo + j] > 0) atomicAdd((unsigned long long *)&pinbound[r.pc[2 * (lo + j)]], 1ull);
    return lam;
}

__global__ void k_edge_runs_fused(int32_t E, const int64_t *pin_off, const int32_t *pin_dat, const int64_t *dst_off,
                                  const int32_t *dst_dat, const int32_t *assign, const int64_t *wi, Runs r,
                                  unsigned long long *conn, int64_t *pinbound) {
    pdl_entry();
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    int64_t contrib = 0;
    for (int64_t e = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id(); e < E; e += nw) {
        const int64_t plo = pin_off[e], lo = r.off[e];
        const int len = (int)(pin_off[e + 1] - plo);
        int32_t lam;
        if (len <= 32)
            lam = warp_edge_runs<1>(e, plo, lo, len, pin_dat, dst_off, dst_dat, assign, r, pinbound);
        else if (len <= 64)
            lam = warp_edge_runs<2>(e, plo, lo, len, pin_dat, dst_off, dst_dat, assign, r, pinbound);
        else
            lam = warp_edge_runs<4>(e, plo, lo, len, pin_dat, dst_off, dst_dat, assign, r, pinbound);
        if (lane_id() == 0) {
            r.len[e] = lam;
            if (lam > 0) contrib += wi[e] * (int64_t)(lam - 1);
        }
    }
    if (lane_id() == 0 && contrib) atomicAdd(conn, (unsigned long long)contrib);
}

__global__ void k_part_sizes(int32_t N, const int32_t *assign, const int32_t *size, int64_t *psizes) {
    pdl_entry();
    int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n < N) atomicAdd((unsigned long long *)&psizes[assign[n]], (unsigned long long)(int64_t)size[n]);
}

// ---------------------------------------------------------------------------
// A14 propose: one best strictly-improving target per node
// (_kernels.pyx:262-310).  Warp per node, parts -> present weight in a
// shared-memory hash table; nodes touching too many parts go to a block tier
// with a dense per-block array over all parts.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool better_gain(int64_t g, int32_t p, int64_t bg, int32_t bp) {
    // max gain, ties to the smaller part id (_kernels.pyx:305)
    return bp < 0 || g > bg || (g == bg && p < bp);
}

struct ProposeArgs {
    int32_t N, K;
    const int64_t *inc_off;
    const int32_t *inc_dat;
    const int64_t *wi;
    Runs r;
    const int32_t *assign;
    const int64_t *psizes;
    const int32_t *size;
    int64_t omega;
    int32_t *target;
    int64_t *gain;
    int32_t *next;
    int32_t *big_list;  // warp tier -> medium tier
    int32_t *big_count;
    int32_t *dense_list;  // medium tier -> dense tier
    int32_t *dense_count;
    Tiers t;
    int32_t lo, hi;  // this rank's node range (comm.cuh); [0, N) on one GPU
    // incremental mode: only the listed (dirty) nodes, their flags cleared
    const int32_t *list = nullptr;
    const int32_t *list_count = nullptr;
    int32_t *ndirty = nullptr;
    // per node: the positive-gain parts the size bound filtered out (the
    // proposal may change when one of them shrinks): fsens = their count
    // (3 = more than two), fpart[2n .. 2n+1] = the first two
    uint8_t *fsens = nullptr;
    int32_t *fpart = nullptr;
    // hub tier: nodes with very many incident h-edges, split over CTAs
    int32_t *hub_list = nullptr;
    int32_t *hub_count = nullptr;
    int32_t hub_max = 0;
    const int32_t *hub_pref = nullptr;  // [hub_max + 1] chunk prefix (k_hub_prefix)
    unsigned long long *work = nullptr;  // profiling: algorithmic bytes
    const int64_t *inc_end = nullptr;  // per-node list ends (DLevel::inc_e)
};
// hubs per propose pass: as many as 256 MB of accumulator rows allow (more go
// to the block tiers); the chunk prefix over them is one small kernel
inline int hub_max_for(int32_t K) {
    return (int)std::max<int64_t>(256, std::min<int64_t>(1 << 15, (256ll << 20) / (8ll * std::max(1, K))));
}
constexpr int HUB_CHUNK = 256;  // incident h-edges per CTA work item

// the next node of a persistent warp/CTA loop: all of [lo, hi), or the
// listed nodes inside [lo, hi); -1 = done, -2 = skip (another rank's node)
__device__ __forceinline__ int32_t propose_node(const ProposeArgs &a, int idx) {
    if (a.list) {
        if (idx >= *a.list_count) return -1;
        const int32_t n = a.list[idx];
        return (n < a.lo || n >= a.hi) ? -2 : n;
    }
    const int64_t n = (int64_t)a.lo + idx;
    return n >= a.hi ? -1 : (int32_t)n;
}

__device__ __forceinline__ void warp_best_gain(long long &bg, int32_t &bp) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const long long og = __shfl_xor_sync(FULL_MASK, bg, d);
        const int32_t op = __shfl_xor_sync(FULL_MASK, bp, d);
        if (op >= 0 && better_gain(og, op, bg, bp)) {
            bg = og;
            bp = op;
        }
    }
}
// one candidate part p with gain g: eligible ones compete for the target,
// size-filtered positive ones are recorded (shared counter nf, first two in f)
__device__ __forceinline__ void consider_part(int32_t p, long long g, bool fits, long long &bg, int32_t &bp, int *nf,
                                              int32_t *f) {
    if (fits) {
        if (better_gain(g, p, bg, bp)) {
            bg = g;
            bp = p;
        }
    } else if (g > 0) {
        const int i = atomicAdd(nf, 1);
        if (i < 2) f[i] = p;
    }
}
__device__ __forceinline__ void write_proposal(const ProposeArgs &a, int32_t node, long long g, int32_t p, int nf,
                                               const int32_t *f) {
    const bool emit = p >= 0 && g > 0;
    a.target[node] = emit ? p : -1;
    a.gain[node] = emit ? g : 0;
    if (a.fsens) {
        a.fsens[node] = (uint8_t)min(nf, 3);
        a.fpart[2 * (int64_t)node] = nf > 0 ? f[0] : -1;
        a.fpart[2 * (int64_t)node + 1] = nf > 1 ? f[1] : -1;
    }
}

// Flattened iteration over the (h-edge, run) pairs of a node's incident
// h-edges: the warp takes 32 incident h-edges at a time (ilo + first, then
// + stride) and spreads their runs evenly over the lanes, so one wide h-edge
// does not serialise on one lane.  f(e, w(e), k) with k the run's index in
// the run arrays.  Returns this lane's share of sum w(e).
template <class F>
__device__ __forceinline__ int64_t warp_for_runs(const int32_t *inc_dat, int64_t ilo, int64_t ihi, int64_t first,
                                                 int64_t stride, int bsz, const int64_t *pin_off, const int32_t *len,
                                                 const int64_t *wi, unsigned long long *work, const int32_t *rpc,
                                                 F &&f) {
    // `work` (profiling only): algorithmic bytes read — 24 B per incident
    // h-edge (list entry, run base, run count, weight) + 8 B per run
    constexpr int U = 4;  // run slots per lane in flight
    const int lane = lane_id();
    int64_t total = 0;
    unsigned long long wb = 0;
    // the next batch's h-edge entries are loaded before this batch's run
    // slots (software pipelining of the incident-list -> offsets chain)
    auto entry = [&](int64_t b) { return (lane < bsz && b + lane < ihi) ? inc_dat[b + lane] : -1; };
    int32_t ne = entry(ilo + first);
    int64_t nplo = 0, nwe = 0;
    int nl = 0;
    if (ne >= 0) {
        nplo = pin_off[ne];
        nl = len[ne];
        nwe = wi[ne];
    }
    int32_t ne2 = entry(ilo + first + stride);
    for (int64_t base = ilo + first; base < ihi; base += stride) {
        const int32_t e = ne;
        const int64_t plo = nplo, we = nwe;
        const int l = nl;
        if (e >= 0) total += we;
        // stage the next batch: its offsets / lengths / weights, and the
        // entries of the one after
        ne = ne2;
        nplo = 0;
        nwe = 0;
        nl = 0;
        if (ne >= 0) {
            nplo = pin_off[ne];
            nl = len[ne];
            nwe = wi[ne];
        }
        ne2 = entry(base + 2 * stride);
        const int incl = warp_incl_scan(l);
        const int tot = __shfl_sync(FULL_MASK, incl, 31);
        const int excl = incl - l;
        wb += 24ull * (unsigned long long)min((int64_t)bsz, ihi - base) + 8ull * (unsigned long long)tot;
        for (int s0 = 0; s0 < tot; s0 += 32 * U) {
            int32_t oe[U], rp[U], rc[U];
            int64_t owe[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int sl = s0 + u * 32 + lane;
                int owner = 0;
#pragma unroll
                for (int step = 16; step > 0; step >>= 1) {
                    const int ex = __shfl_sync(FULL_MASK, excl, owner + step);
                    if (ex <= sl) owner += step;
                }
                oe[u] = __shfl_sync(FULL_MASK, e, owner);
                const int64_t oplo = __shfl_sync(FULL_MASK, plo, owner);
                owe[u] = __shfl_sync(FULL_MASK, we, owner);
                const int oex = __shfl_sync(FULL_MASK, excl, owner);
                const int64_t k = oplo + (sl - oex);
                const int2 v = sl < tot ? reinterpret_cast<const int2 *>(rpc)[k] : make_int2(-1, 0);
                rp[u] = v.x;
                rc[u] = v.y;
            }
#pragma unroll
            for (int u = 0; u < U; u++)
                if (s0 + u * 32 + lane < tot) f(oe[u], owe[u], rp[u], rc[u]);
        }
    }
    if (work && lane == 0 && wb) atomicAdd(work, wb);
    return total;
}

constexpr int PR_WARPS = 8;
constexpr int PR_CAP = 512;
// 32-bit accumulators when the total weight < 2^32 (native shared atomics)
template <class Acc>
constexpr int pr_smem() { return PR_WARPS * PR_CAP * (4 + (int)sizeof(Acc)); }

__device__ __forceinline__ uint32_t pslot(int32_t p) { return ((uint32_t)p * 2654435761u) >> (32 - 9); }


template <class Acc>
__global__ void __launch_bounds__(PR_WARPS * 32, 4) k_propose_warp(ProposeArgs a) {
    pdl_entry();
    extern __shared__ unsigned long long smem_u64[];
    Acc *svals = (Acc *)smem_u64;
    int32_t *skeys = (int32_t *)(svals + PR_WARPS * PR_CAP);
    __shared__ int32_t snk[PR_WARPS];
    __shared__ int32_t sover[PR_WARPS];
    __shared__ int s_nf[PR_WARPS];
    __shared__ int32_t s_f[PR_WARPS][2];
    const int w = warp_id(), lane = lane_id();
    int32_t *keys = skeys + w * PR_CAP;
    Acc *vals = svals + w * PR_CAP;
    while (true) {
        int idx = 0;
        if (lane == 0) idx = atomicAdd(a.next, 1);
        idx = __shfl_sync(FULL_MASK, idx, 0);
        const int32_t node = propose_node(a, idx);
        if (node == -1) break;
        if (a.ndirty && lane == 0 && a.list) a.ndirty[a.list[idx]] = 0;
        if (node < 0) continue;
        const int64_t ilo = a.inc_off[node], ihi = a.inc_end[node];
        if (ihi == ilo || a.K < 2) {
            if (lane == 0) write_proposal(a, node, 0, -1, 0, nullptr);
            continue;
        }
        if (a.hub_list && ihi - ilo > a.t.pr_hub_inc) {  // hub: many CTAs take it
            if (lane == 0) {
                const int slot = atomicAdd(a.hub_count, 1);
                if (slot < a.hub_max)
                    a.hub_list[slot] = node;
                else
                    a.big_list[atomicAdd(a.big_count, 1)] = node;
            }
            continue;
        }
        if (ihi - ilo > a.t.pr_heavy_inc) {  // many incident h-edges: a whole block takes it
            if (lane == 0) a.big_list[atomicAdd(a.big_count, 1)] = node;
            continue;
        }
        for (int s = lane; s < PR_CAP; s += 32) {
            keys[s] = -1;
            vals[s] = 0;
        }
        if (lane == 0) {
            snk[w] = 0;
            sover[w] = 0;
        }
        __syncwarp();
        const int32_t ps = a.assign[node];
        int64_t total = 0, saving = 0;
        total = warp_for_runs(a.inc_dat, ilo, ihi, 0, 32, 32, a.r.off, a.r.len, a.wi, a.work, a.r.pc, [&](int32_t, int64_t we, int32_t p, int32_t pc) {
            if (p == ps && pc == 1) saving += we;
            const uint32_t h = pslot(p);
            for (int probe = 0; probe < PR_CAP; probe++) {
                if (probe % kFlagPoll == kFlagPoll - 1 && flag_get(&sover[w])) return;
                const int slot = (h + probe) & (PR_CAP - 1);
                int kk = keys[slot];
                if (kk == -1) {
                    const int prev = atomicCAS(&keys[slot], -1, p);
                    if (prev == -1) {
                        if (atomicAdd(&snk[w], 1) >= a.t.pr_limit) flag_set(&sover[w]);
                        kk = p;
                    } else {
                        kk = prev;
                    }
                }
                if (kk == p) {
                    atomicAdd(&vals[slot], (Acc)we);
                    return;
                }
            }
            flag_set(&sover[w]);
        });
        total = warp_sum(total);
        saving = warp_sum(saving);
        __syncwarp();
        if (sover[w]) {
            if (lane == 0) a.big_list[atomicAdd(a.big_count, 1)] = node;
            __syncwarp();
            continue;
        }
        const int64_t sz = a.size[node];
        long long bg = 0;
        int32_t bp = -1;
        if (lane == 0) s_nf[w] = 0;
        __syncwarp();
        // the parts' sizes are gathered 4 slots at a time (one round trip each)
        for (int s0 = lane; s0 < PR_CAP; s0 += 4 * 32) {
            int32_t pp[4];
            long long vv[4], pz[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int s = s0 + u * 32;
                pp[u] = s < PR_CAP ? keys[s] : -1;
                if (pp[u] == ps) pp[u] = -1;
                vv[u] = pp[u] >= 0 ? (long long)vals[s] : 0;
            }
#pragma unroll
            for (int u = 0; u < 4; u++) pz[u] = pp[u] >= 0 ? a.psizes[pp[u]] : 0;
#pragma unroll
            for (int u = 0; u < 4; u++)
                if (pp[u] >= 0)
                    consider_part(pp[u], saving - (total - vv[u]), pz[u] + sz <= a.omega, bg, bp, &s_nf[w], s_f[w]);
        }
        warp_best_gain(bg, bp);
        __syncwarp();
        if (lane == 0) write_proposal(a, node, bg, bp, s_nf[w], s_f[w]);
        __syncwarp();
    }
}

// Medium tier: one 256-thread CTA per node with a 4096-slot shared hash
// table (nodes with many incident h-edges, or more distinct parts than a
// warp's table holds).  Nodes touching more than PM_LIMIT parts go on to the
// dense tier.
constexpr int PM_THREADS = 256;
constexpr int PM_CAP = 8192;
template <class Acc>
constexpr int pm_smem() { return PM_CAP * (4 + (int)sizeof(Acc)); }

__device__ __forceinline__ void block_best_gain(long long bg, int32_t bp, long long *r_g, int32_t *r_p, int nw,
                                                long long *out_g, int32_t *out_p) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        long long og = __shfl_xor_sync(FULL_MASK, bg, d);
        int32_t op = __shfl_xor_sync(FULL_MASK, bp, d);
        if (op >= 0 && better_gain(og, op, bg, bp)) {
            bg = og;
            bp = op;
        }
    }
    if (lane_id() == 0) {
        r_g[warp_id()] = bg;
        r_p[warp_id()] = bp;
    }
    __syncthreads();
    long long g = r_g[0];
    int32_t p = r_p[0];
    for (int j = 1; j < nw; j++)
        if (r_p[j] >= 0 && better_gain(r_g[j], r_p[j], g, p)) {
            g = r_g[j];
            p = r_p[j];
        }
    *out_g = g;
    *out_p = p;
}

template <class Acc>
__global__ void __launch_bounds__(PM_THREADS, 4) k_propose_mid(ProposeArgs a) {
    pdl_entry();
    extern __shared__ unsigned long long smem_u64[];
    Acc *vals = (Acc *)smem_u64;
    int32_t *keys = (int32_t *)(vals + PM_CAP);
    __shared__ int32_t snk;
    __shared__ int32_t sover;
    __shared__ long long r_a[PM_THREADS / 32], r_b[PM_THREADS / 32];
    __shared__ int32_t r_p[PM_THREADS / 32];
    __shared__ int s_nf;
    __shared__ int32_t s_f[2];
    __shared__ long long s_runs;
    const int w = warp_id(), lane = lane_id(), nw = PM_THREADS / 32;
    const int nmid = *a.big_count;
    for (int t = blockIdx.x; t < nmid; t += gridDim.x) {
        const int32_t node = a.big_list[t];
        const int64_t ilo = a.inc_off[node], ihi = a.inc_end[node];
        // table sized to the node: its distinct parts are at most min(K, sum of
        // its h-edges' run counts); zeroing and scanning 8192 slots per node
        // dominated when K is large and nodes touch few parts
        if (threadIdx.x == 0) s_runs = 0;
        __syncthreads();
        long long nr = 0;
        for (int64_t i = ilo + threadIdx.x; i < ihi; i += PM_THREADS) nr += a.r.len[a.inc_dat[i]];
        nr = warp_sum(nr);
        if (lane == 0) atomicAdd((unsigned long long *)&s_runs, (unsigned long long)nr);
        __syncthreads();
        // a node with more runs than the table's part limit: straight to the
        // dense shared-memory tier, which indexes parts directly (the tier
        // never changes the result, only the cost)
        if (s_runs > (long long)a.t.pm_limit && a.K > a.t.pm_limit) {
            if (threadIdx.x == 0) a.dense_list[atomicAdd(a.dense_count, 1)] = node;
            __syncthreads();
            continue;
        }
        int lg = 6;
        while ((1ll << lg) < 2 * min((long long)a.K, s_runs) && lg < 13) lg++;
        const int cap = 1 << lg;
        const int limit = min(a.t.pm_limit, cap - cap / 4);
        for (int s = threadIdx.x; s < cap; s += PM_THREADS) {
            keys[s] = -1;
            vals[s] = 0;
        }
        if (threadIdx.x == 0) {
            snk = 0;
            sover = 0;
        }
        __syncthreads();
        const int32_t ps = a.assign[node];
        long long total = 0, saving = 0;
        // h-edges per warp batch: a node's h-edges spread over all warps
        const int rb = (int)max((int64_t)1, min((int64_t)32, (ihi - ilo + nw - 1) / nw));
        total = warp_for_runs(a.inc_dat, ilo, ihi, (int64_t)w * rb, (int64_t)nw * rb, rb, a.r.off, a.r.len, a.wi, a.work,
                              a.r.pc,
                              [&](int32_t, int64_t we, int32_t p, int32_t pc) {
                                  if (p == ps && pc == 1) saving += we;
                                  const uint32_t h = ((uint32_t)p * 2654435761u) >> (32 - lg);
                                  for (int probe = 0; probe < cap; probe++) {
                                      if (probe % kFlagPoll == kFlagPoll - 1 && flag_get(&sover)) return;
                                      const int slot = (h + probe) & (cap - 1);
                                      int kk = keys[slot];
                                      if (kk == -1) {
                                          const int prev = atomicCAS(&keys[slot], -1, p);
                                          if (prev == -1) {
                                              if (atomicAdd(&snk, 1) >= limit) flag_set(&sover);
                                              kk = p;
                                          } else {
                                              kk = prev;
                                          }
                                      }
                                      if (kk == p) {
                                          atomicAdd(&vals[slot], (Acc)we);
                                          return;
                                      }
                                  }
                                  flag_set(&sover);
                              });
        total = warp_sum(total);
        saving = warp_sum(saving);
        if (lane == 0) {
            r_a[w] = total;
            r_b[w] = saving;
        }
        __syncthreads();
        if (sover) {
            if (threadIdx.x == 0) a.dense_list[atomicAdd(a.dense_count, 1)] = node;
            __syncthreads();
            continue;
        }
        total = 0;
        saving = 0;
        for (int j = 0; j < nw; j++) {
            total += r_a[j];
            saving += r_b[j];
        }
        __syncthreads();
        const int64_t sz = a.size[node];
        long long bg = 0;
        int32_t bp = -1;
        if (threadIdx.x == 0) s_nf = 0;
        __syncthreads();
        for (int s0 = threadIdx.x; s0 < cap; s0 += 4 * PM_THREADS) {  // sizes gathered 4 slots at a time
            int32_t pp[4];
            long long vv[4], pz[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int s = s0 + u * PM_THREADS;
                pp[u] = s < cap ? keys[s] : -1;
                if (pp[u] == ps) pp[u] = -1;
                vv[u] = pp[u] >= 0 ? (long long)vals[s] : 0;
            }
#pragma unroll
            for (int u = 0; u < 4; u++) pz[u] = pp[u] >= 0 ? a.psizes[pp[u]] : 0;
#pragma unroll
            for (int u = 0; u < 4; u++)
                if (pp[u] >= 0)
                    consider_part(pp[u], saving - (total - vv[u]), pz[u] + sz <= a.omega, bg, bp, &s_nf, s_f);
        }
        long long g;
        int32_t p;
        block_best_gain(bg, bp, r_a, r_p, nw, &g, &p);
        if (threadIdx.x == 0) write_proposal(a, node, g, p, s_nf, s_f);
        __syncthreads();
    }
}

// Dense tier for K <= PH_MAXK: one block per node, present[] as a dense
// shared array indexed by part id plus the list of touched parts (each
// node costs O(its distinct parts), not O(K)).
constexpr int PH_THREADS = 1024;
// largest K whose dense arrays (present + touched list + bitmap) fit the
// 227 KB of shared memory of one CTA
template <class Acc>
constexpr int ph_maxk() { return (int)((220 * 1024 - 64) * 8 / (8 * (sizeof(Acc) + 4) + 1)); }
template <class Acc>
constexpr size_t ph_smem(int K) { return (size_t)K * (sizeof(Acc) + 4) + 4 * (size_t)((K + 31) / 32) + 16; }
template <class Acc, int THREADS = PH_THREADS>
__global__ void __launch_bounds__(THREADS) k_propose_heavy(ProposeArgs a) {
    pdl_entry();
    extern __shared__ unsigned long long smem_u64[];
    Acc *pres = (Acc *)smem_u64;
    int32_t *tlist = (int32_t *)(pres + a.K);
    uint32_t *touched = (uint32_t *)(tlist + a.K);
    __shared__ int32_t s_nt;
    __shared__ long long r_a[THREADS / 32], r_b[THREADS / 32];
    __shared__ int32_t r_p[THREADS / 32];
    __shared__ int s_nf;
    __shared__ int32_t s_f[2];
    const int w = warp_id(), lane = lane_id(), nw = THREADS / 32;
    const int nbig = *a.dense_count;
    if ((int)blockIdx.x >= nbig) return;
    const int tw = (a.K + 31) >> 5;
    for (int p = threadIdx.x; p < a.K; p += THREADS) pres[p] = 0;
    for (int p = threadIdx.x; p < tw; p += THREADS) touched[p] = 0;
    for (int t = blockIdx.x; t < nbig; t += gridDim.x) {
        const int32_t node = a.dense_list[t];
        if (threadIdx.x == 0) s_nt = 0;
        __syncthreads();
        const int64_t ilo = a.inc_off[node], ihi = a.inc_end[node];
        const int32_t ps = a.assign[node];
        long long total = 0, saving = 0;
        // h-edges per warp batch: a node's h-edges spread over all warps
        const int rb = (int)max((int64_t)1, min((int64_t)32, (ihi - ilo + nw - 1) / nw));
        total = warp_for_runs(a.inc_dat, ilo, ihi, (int64_t)w * rb, (int64_t)nw * rb, rb, a.r.off, a.r.len, a.wi, a.work,
                              a.r.pc,
                              [&](int32_t, int64_t we, int32_t p, int32_t pc) {
                                  if (p == ps && pc == 1) saving += we;
                                  atomicAdd(&pres[p], (Acc)we);
                                  const uint32_t bit = 1u << (p & 31);
                                  if (!(atomicOr(&touched[p >> 5], bit) & bit)) tlist[atomicAdd(&s_nt, 1)] = p;
                              });
        total = warp_sum(total);
        saving = warp_sum(saving);
        if (lane == 0) {
            r_a[w] = total;
            r_b[w] = saving;
        }
        __syncthreads();
        total = 0;
        saving = 0;
        for (int j = 0; j < nw; j++) {
            total += r_a[j];
            saving += r_b[j];
        }
        const int nt = s_nt;
        __syncthreads();
        const int64_t sz = a.size[node];
        long long bg = 0;
        int32_t bp = -1;
        if (threadIdx.x == 0) s_nf = 0;
        __syncthreads();
        for (int i0 = threadIdx.x; i0 < nt; i0 += 4 * THREADS) {  // sizes gathered 4 parts at a time
            int32_t pp[4];
            long long vv[4], pz[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int i = i0 + u * THREADS;
                pp[u] = -1;
                vv[u] = 0;
                if (i < nt) {
                    const int32_t p = tlist[i];
                    vv[u] = (long long)pres[p];
                    pres[p] = 0;
                    touched[p >> 5] = 0;
                    pp[u] = p == ps ? -1 : p;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; u++) pz[u] = pp[u] >= 0 ? a.psizes[pp[u]] : 0;
#pragma unroll
            for (int u = 0; u < 4; u++)
                if (pp[u] >= 0)
                    consider_part(pp[u], saving - (total - vv[u]), pz[u] + sz <= a.omega, bg, bp, &s_nf, s_f);
        }
        long long g;
        int32_t p;
        block_best_gain(bg, bp, r_a, r_p, nw, &g, &p);
        if (threadIdx.x == 0) write_proposal(a, node, g, p, s_nf, s_f);
        __syncthreads();
    }
}


// chunk counts of the listed hubs, scanned by one CTA (the hub kernel's
// work items are (hub, chunk) pairs)
__global__ void __launch_bounds__(1024) k_hub_prefix(const int32_t *hub_list, const int32_t *hub_count, int hub_max,
                                                     const int64_t *inc_off, const int64_t *inc_end,
                                                     int32_t *pref) {
    pdl_entry();
    __shared__ int32_t s_wt[32];
    const int nh = min(*hub_count, hub_max);
    const int lane = lane_id(), w = warp_id();
    int32_t carry = 0;
    if (threadIdx.x == 0) pref[0] = 0;
    for (int b = 0; b < nh; b += 1024) {
        const int i = b + threadIdx.x;
        int32_t cnt = 0;
        if (i < nh) {
            const int32_t n = hub_list[i];
            cnt = (int32_t)cdiv_dev(inc_end[n] - inc_off[n], (int64_t)HUB_CHUNK);
        }
        const int32_t incl = warp_incl_scan(cnt);
        if (lane == 31) s_wt[w] = incl;
        __syncthreads();
        int32_t before = 0, tot = 0;
        for (int j = 0; j < 32; j++) {
            if (j < w) before += s_wt[j];
            tot += s_wt[j];
        }
        if (i < nh) pref[i + 1] = carry + before + incl;
        carry += tot;
        __syncthreads();
    }
}

// Hub tier (K <= small_k): a node with thousands of incident h-edges is cut
// into HUB_CHUNK-edge work items spread over the grid; each CTA accumulates
// present[] for its chunk in shared memory and adds it to the hub's global
// row; the CTA finishing a hub's last chunk selects the target.
template <class Acc>
__global__ void __launch_bounds__(256, 6) k_propose_hub(ProposeArgs a, long long *hacc, long long *htot,
                                                     int32_t *hdone) {
    pdl_entry();
    extern __shared__ unsigned long long smem_u64[];
    Acc *pres = (Acc *)smem_u64;
    __shared__ long long r_a[8], r_b[8];
    __shared__ int32_t r_p[8];
    __shared__ int s_last, s_nf;
    __shared__ int32_t s_f[2];
    const int nh = min(*a.hub_count, a.hub_max);
    if (nh == 0) return;
    const int w = warp_id(), lane = lane_id(), nw = 8;
    const int K = a.K;
    // work items = (hub, chunk), located in the chunk prefix of k_hub_prefix
    const int32_t *s_pref = a.hub_pref;
    const int64_t items = s_pref[nh];
    for (int64_t t = blockIdx.x; t < items; t += gridDim.x) {
        int lo = 0, hi = nh;  // the hub h with s_pref[h] <= t < s_pref[h + 1]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_pref[mid] <= t)
                lo = mid;
            else
                hi = mid;
        }
        const int h = lo;
        const int64_t chunk = t - s_pref[h];
        const int64_t nch = s_pref[h + 1] - s_pref[h];
        const int32_t node = a.hub_list[h];
        const int64_t ilo = a.inc_off[node] + chunk * HUB_CHUNK;
        const int64_t ihi = min(a.inc_end[node], ilo + (int64_t)HUB_CHUNK);
        for (int p = threadIdx.x; p < K; p += blockDim.x) pres[p] = 0;
        __syncthreads();
        const int32_t ps = a.assign[node];
        long long total = 0, saving = 0;
        // h-edges per warp batch: a node's h-edges spread over all warps
        const int rb = (int)max((int64_t)1, min((int64_t)32, (ihi - ilo + nw - 1) / nw));
        total = warp_for_runs(a.inc_dat, ilo, ihi, (int64_t)w * rb, (int64_t)nw * rb, rb, a.r.off, a.r.len, a.wi, a.work,
                              a.r.pc,
                              [&](int32_t, int64_t we, int32_t p, int32_t pc) {
                                  if (p == ps && pc == 1) saving += we;
                                  atomicAdd(&pres[p], (Acc)we);
                              });
        total = warp_sum(total);
        saving = warp_sum(saving);
        if (lane == 0) {
            r_a[w] = total;
            r_b[w] = saving;
        }
        __syncthreads();
        long long *row = hacc + (int64_t)h * K;
        for (int p = threadIdx.x; p < K; p += blockDim.x)
            if (pres[p]) atomicAdd((unsigned long long *)&row[p], (unsigned long long)pres[p]);
        if (threadIdx.x == 0) {
            long long t0 = 0, s0 = 0;
            for (int j = 0; j < nw; j++) {
                t0 += r_a[j];
                s0 += r_b[j];
            }
            atomicAdd((unsigned long long *)&htot[2 * h], (unsigned long long)t0);
            atomicAdd((unsigned long long *)&htot[2 * h + 1], (unsigned long long)s0);
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) s_last = atomicAdd(&hdone[h], 1) == (int)(nch - 1);
        __syncthreads();
        if (s_last) {
            __threadfence();
            const long long tot = __ldcg(&htot[2 * h]), sav = __ldcg(&htot[2 * h + 1]);
            const int64_t sz = a.size[node];
            long long bg = 0;
            int32_t bp = -1;
            if (threadIdx.x == 0) s_nf = 0;
            __syncthreads();
            for (int p = threadIdx.x; p < K; p += blockDim.x) {
                const long long v = __ldcg(&row[p]);
                if (v == 0) continue;  // absent, or only zero-weight h-edges (gain <= 0)
                row[p] = 0;
                if (p == ps) continue;
                consider_part(p, sav - (tot - v), a.psizes[p] + sz <= a.omega, bg, bp, &s_nf, s_f);
            }
            long long g;
            int32_t pp;
            block_best_gain(bg, bp, r_a, r_p, nw, &g, &pp);
            if (threadIdx.x == 0) {
                write_proposal(a, node, g, pp, s_nf, s_f);
                htot[2 * h] = 0;
                htot[2 * h + 1] = 0;
                hdone[h] = 0;
            }
        }
        __syncthreads();
    }
}

constexpr int PB_THREADS = 512;
__global__ void __launch_bounds__(PB_THREADS) k_propose_block(ProposeArgs a, long long *dense_all,
                                                               int32_t *touched_all) {
    pdl_entry();
    __shared__ int32_t s_nt;
    __shared__ long long s_red[PB_THREADS / 32][2];
    __shared__ int32_t s_p[PB_THREADS / 32];
    __shared__ int s_nf;
    __shared__ int32_t s_f[2];
    long long *dense = dense_all + (int64_t)blockIdx.x * a.K;
    int32_t *touched = touched_all + (int64_t)blockIdx.x * a.K;
    const int w = warp_id(), lane = lane_id(), nw = PB_THREADS / 32;
    const int nbig = *a.dense_count;
    for (int t = blockIdx.x; t < nbig; t += gridDim.x) {
        const int32_t node = a.dense_list[t];
        if (threadIdx.x == 0) s_nt = 0;
        __syncthreads();
        const int64_t ilo = a.inc_off[node], ihi = a.inc_end[node];
        const int32_t ps = a.assign[node];
        long long total = 0, saving = 0;
        // h-edges per warp batch: a node's h-edges spread over all warps
        const int rb = (int)max((int64_t)1, min((int64_t)32, (ihi - ilo + nw - 1) / nw));
        total = warp_for_runs(a.inc_dat, ilo, ihi, (int64_t)w * rb, (int64_t)nw * rb, rb, a.r.off, a.r.len, a.wi, a.work,
                              a.r.pc,
                              [&](int32_t, int64_t we, int32_t p, int32_t pc) {
                                  if (p == ps && pc == 1) saving += we;
                                  const long long old = atomicCAS((unsigned long long *)&dense[p], ~0ull, 0ull);
                                  if (old == -1ll) touched[atomicAdd(&s_nt, 1)] = p;
                                  atomicAdd((unsigned long long *)&dense[p], (unsigned long long)we);
                              });
        total = warp_sum(total);
        saving = warp_sum(saving);
        if (lane == 0) {
            s_red[w][0] = total;
            s_red[w][1] = saving;
        }
        __syncthreads();
        total = 0;
        saving = 0;
        for (int j = 0; j < nw; j++) {
            total += s_red[j][0];
            saving += s_red[j][1];
        }
        const int nt = s_nt;
        const int64_t sz = a.size[node];
        long long bg = 0;
        int32_t bp = -1;
        if (threadIdx.x == 0) s_nf = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < nt; i += PB_THREADS) {
            const int32_t p = touched[i];
            const long long pres = dense[p];
            dense[p] = -1ll;
            if (p == ps) continue;
            consider_part(p, saving - (total - pres), a.psizes[p] + sz <= a.omega, bg, bp, &s_nf, s_f);
        }
        warp_best_gain(bg, bp);
        __syncthreads();
        if (lane == 0) {
            s_red[w][0] = bg;
            s_p[w] = bp;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            long long g = s_red[0][0];
            int32_t p = s_p[0];
            for (int j = 1; j < nw; j++)
                if (s_p[j] >= 0 && better_gain(s_red[j][0], s_p[j], g, p)) {
                    g = s_red[j][0];
                    p = s_p[j];
                }
            write_proposal(a, node, g, p, s_nf, s_f);
        }
        __syncthreads();
    }
}

__global__ void k_fill_ll(long long *p, long long v, int64_t n) {
    pdl_entry();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

__global__ void k_mover_flags(int32_t N, const int32_t *target, uint8_t *flags, int32_t *reset) {
    pdl_entry();
    int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (reset && n == 0) *reset = 0;
    if (n < N) flags[n] = target[n] >= 0;
}

// sequence key: gain descending (stable sort keeps node ascending among ties,
// refine.py:108-110)
__global__ void k_mover_keys(int32_t N, const uint8_t *flags, const int64_t *pos, const int64_t *gain, int64_t gmax,
                             uint64_t *keys, uint32_t *vals) {
    pdl_entry();
    int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n < N && flags[n]) {
        keys[pos[n]] = (uint64_t)(gmax - gain[n]);
        vals[pos[n]] = (uint32_t)n;
    }
}

// ---------------------------------------------------------------------------
// A17 events.  Key = track | part | move index; track 0 = size, 1 = inbound.
// ---------------------------------------------------------------------------
struct EvArgs {
    int ibits, pbits;
    uint64_t *key;
    uint32_t *val;
    unsigned long long *count;
    // inbound track, pre-aggregated per move: _track_violations only reads
    // the delta sum of each (part, move) group, and move i's inbound
    // crossings all sit at its source (1 -> 0) or target (0 -> 1) part
    int32_t *in_from = nullptr, *in_to = nullptr;
};
__device__ __forceinline__ void inbound_leave(const EvArgs &ev, int32_t i) { atomicSub(&ev.in_from[i], 1); }
__device__ __forceinline__ void inbound_enter(const EvArgs &ev, int32_t i) { atomicAdd(&ev.in_to[i], 1); }

// inbound track (refine.py:210-237), per h-edge: the movers among its
// destination pins in sequence order; per part a running destination-pin
// count from pins_in[e, p]; crossings 0->1 / 1->0 emit distinct events.
// This is the walk for h-edges with many movers (the warp kernel
// k_round_edges takes the others).  The walk only couples movers through a
// shared part, so it runs per part: the block collects and sorts the movers,
// gathers the distinct parts they touch (shared hash), and a warp per part
// sweeps the movers 32 at a time — delta -1 when the mover leaves the part,
// +1 when it enters — with a warp scan for the running count: a leave that
// brings it to 0 and an enter that brings it to 1 are the crossings.
constexpr int kEvBlockMax = 2048;
constexpr int kEvParts = 2 * kEvBlockMax;  // hash slots (>= distinct parts: 2 per mover)
__global__ void __launch_bounds__(256) k_inbound_events_block(const int64_t *dst_off, const int32_t *dst_dat, Runs r,
                                       const int32_t *pos, const int32_t *from, const int32_t *to, EvArgs ev,
                                       const int32_t *big_list, const int32_t *big_count, int32_t *huge,
                                       int32_t *huge_count, int mv_max) {
    pdl_entry();
    __shared__ uint32_t smv[kEvBlockMax];
    __shared__ int32_t skey[kEvParts];
    __shared__ int32_t sparts[kEvParts];
    __shared__ int32_t snm, snp;
    const int lane = lane_id(), w = warp_id(), nw = blockDim.x >> 5;
    const int nbig = *big_count;
    for (int t = blockIdx.x; t < nbig; t += gridDim.x) {
        const int32_t e = big_list[t];
        if (threadIdx.x == 0) {
            snm = 0;
            snp = 0;
        }
        for (int s = threadIdx.x; s < kEvParts; s += blockDim.x) skey[s] = -1;
        __syncthreads();
        for (int64_t q = dst_off[e] + threadIdx.x; q < dst_off[e + 1]; q += blockDim.x) {
            int32_t j = pos[dst_dat[q]];
            if (j >= 0) {
                int s = atomicAdd(&snm, 1);
                if (s < kEvBlockMax) smv[s] = (uint32_t)j;
            }
        }
        __syncthreads();
        const int nm = snm;
        if (nm > mv_max) {  // global-memory path (k_edge_movers_huge)
            if (threadIdx.x == 0) huge[atomicAdd(huge_count, 1)] = e;
            __syncthreads();
            continue;
        }
        const int np = next_pow2(nm);
        for (int s = nm + threadIdx.x; s < np; s += blockDim.x) smv[s] = 0xffffffffu;
        block_bitonic_sort32(smv, np);
        // distinct parts among the movers' sources and targets
        for (int a = threadIdx.x; a < 2 * nm; a += blockDim.x) {
            const int32_t i = (int32_t)smv[a >> 1];
            const int32_t p = (a & 1) ? to[i] : from[i];
            uint32_t h = ((uint32_t)p * 2654435761u) & (kEvParts - 1);
            while (true) {
                const int32_t k = skey[h];
                if (k == p) break;
                if (k == -1) {
                    const int32_t prev = atomicCAS(&skey[h], -1, p);
                    if (prev == -1) {
                        sparts[atomicAdd(&snp, 1)] = p;
                        break;
                    }
                    if (prev == p) break;
                }
                h = (h + 1) & (kEvParts - 1);
            }
        }
        __syncthreads();
        const int npart = snp;
        const int64_t lo = r.off[e];
        const int32_t lam = r.len[e];
        for (int q = w; q < npart; q += nw) {
            const int32_t p = sparts[q];
            int32_t run = 0;
            if (lane == 0) {
                const int32_t f = run_find(r, lo, lam, p);
                run = f >= 0 ? r.cin[lo + f] : 0;
            }
            run = __shfl_sync(FULL_MASK, run, 0);
            for (int a0 = 0; a0 < nm; a0 += 32) {
                const int a = a0 + lane;
                int32_t i = 0, d = 0;
                if (a < nm) {
                    i = (int32_t)smv[a];
                    d = (to[i] == p) - (from[i] == p);
                }
                const int32_t incl = warp_incl_scan(d) + run;
                if (d < 0 && incl == 0) inbound_leave(ev, i);
                if (d > 0 && incl == 1) inbound_enter(ev, i);
                run = __shfl_sync(FULL_MASK, incl, 31);
            }
        }
        __syncthreads();
    }
}

// _track_violations (refine.py:145-175) as a segmented formulation over the
// events sorted by (track, part, i): group = equal key, segment = equal
// (track, part).  With ex = exclusive prefix sums of the deltas and the
// group / segment start indices from running-max scans, the value after a
// group is base + ex[end+1] - ex[seg0] and before it base + ex[g0] - ex[seg0];
// a group toggles its part's flag when the two sit on different sides of
// the limit.
__global__ void k_ev_prep(int64_t T, const uint64_t *key, const uint32_t *val, int ibits, int64_t *gs, int64_t *ss,
                          int64_t *dv) {
    pdl_entry();
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= T) return;
    const uint64_t kk = key[k];
    gs[k] = (k == 0 || key[k - 1] != kk) ? k : 0;
    ss[k] = (k == 0 || (key[k - 1] >> ibits) != (kk >> ibits)) ? k : 0;
    dv[k] = (int64_t)(int32_t)val[k];
}
__global__ void k_ev_toggle(int64_t T, const uint64_t *key, const int64_t *ex, const int64_t *gstart,
                            const int64_t *sstart, int ibits, int pbits, const int64_t *psizes,
                            const int64_t *pinbound, int64_t omega, int64_t delta, int64_t *dlt) {
    pdl_entry();
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= T) return;
    const uint64_t kk = key[k];
    if (k + 1 < T && key[k + 1] == kk) return;  // not the last event of its group
    const int track = (int)(kk >> (ibits + pbits));
    const int32_t p = (int32_t)((kk >> ibits) & ((1ull << pbits) - 1ull));
    const uint64_t i = kk & ((1ull << ibits) - 1ull);
    const int64_t base = track ? pinbound[p] : psizes[p];
    const int64_t limit = track ? delta : omega;
    const int64_t s0 = ex[sstart[k]];
    const bool after = base + ex[k + 1] - s0 > limit;
    const bool before = base + ex[gstart[k]] - s0 > limit;
    if (after != before) atomicAdd((unsigned long long *)&dlt[i + 1], (unsigned long long)(after ? 1ll : -1ll));
}

// smallest argmax of cum over prefixes with active == 0 (refine.py:244-247)
__global__ void k_best_prefix_partial(int64_t n, const int64_t *active_ex, const int64_t *cum, long long *bv,
                                      long long *bk) {
    pdl_entry();
    __shared__ long long sv[32], sk[32];
    long long v = LLONG_MIN, k = LLONG_MAX;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        // active[j] = inclusive cumsum of delta up to j = active_ex[j + 1]
        if (active_ex[j + 1] == 0) {
            long long c = cum[j];
            if (c > v || (c == v && j < k)) {
                v = c;
                k = j;
            }
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        long long ov = __shfl_xor_sync(FULL_MASK, v, d), ok = __shfl_xor_sync(FULL_MASK, k, d);
        if (ov > v || (ov == v && ok < k)) {
            v = ov;
            k = ok;
        }
    }
    if (lane_id() == 0) {
        sv[warp_id()] = v;
        sk[warp_id()] = k;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); w++)
            if (sv[w] > v || (sv[w] == v && sk[w] < k)) {
                v = sv[w];
                k = sk[w];
            }
        bv[blockIdx.x] = v;
        bk[blockIdx.x] = k;
    }
}
__global__ void k_best_prefix_final(int nb, const long long *bv, const long long *bk, long long *out) {
    pdl_entry();
    if (threadIdx.x != 0) return;
    long long v = LLONG_MIN, k = LLONG_MAX;
    for (int b = 0; b < nb; b++)
        if (bv[b] > v || (bv[b] == v && bk[b] < k)) {
            v = bv[b];
            k = bk[b];
        }
    out[0] = k;
    out[1] = v;
}

// ---------------------------------------------------------------------------
// A17 in one CTA for small rounds (T <= SEL_T events, M <= SEL_M moves): the
// event sort, the segmented toggle formulation, active[] and the best prefix
// in shared memory — the same arithmetic as the multi-kernel path below, in
// one launch and without reading T on the host.  res[2] = 1 when the round
// is too large (the host then runs the multi-kernel path).
// ---------------------------------------------------------------------------
constexpr int SEL_T = 4096, SEL_M = 4096, SEL_THREADS = 1024;
constexpr size_t sel_smem() {
    return (size_t)SEL_T * 8 + (size_t)SEL_T * 4 + (size_t)(SEL_T + 1) * 8 + 2 * (size_t)SEL_T * 4 +
           (size_t)(SEL_M + 2) * 4 + (size_t)(SEL_M + 1) * 8 + 64;
}

// block-wide exclusive scan of a per-thread value (SEL_THREADS threads)
__device__ __forceinline__ int64_t sel_excl(int64_t v, int64_t *sh, int64_t *total) {
    const int lane = lane_id(), w = warp_id(), nw = SEL_THREADS / 32;
    const int64_t incl = warp_incl_scan(v);
    if (lane == 31) sh[w] = incl;
    __syncthreads();
    if (w == 0) {
        const int64_t x = lane < nw ? sh[lane] : 0;
        const int64_t xi = warp_incl_scan(x);
        if (lane < nw) sh[lane] = xi - x;
        if (lane == nw - 1) sh[32] = xi;
    }
    __syncthreads();
    const int64_t r = incl - v + sh[w];
    *total = sh[32];
    __syncthreads();
    return r;
}
// out[0..n] = exclusive prefix sums of f(0..n-1) (each thread a contiguous chunk)
template <class F>
__device__ __forceinline__ void sel_scan_sum(int n, F f, int64_t *out, int64_t *sh) {
    const int per = (n + SEL_THREADS - 1) / SEL_THREADS;
    const int a = min(n, (int)threadIdx.x * per), b = min(n, a + per);
    int64_t loc = 0;
    for (int i = a; i < b; i++) loc += f(i);
    int64_t tot;
    int64_t run = sel_excl(loc, sh, &tot);
    for (int i = a; i < b; i++) {
        const int64_t v = f(i);
        out[i] = run;
        run += v;
    }
    if (threadIdx.x == 0) out[n] = tot;
    __syncthreads();
}
// in-place inclusive running maximum of a[0..n) (non-negative values)
__device__ __forceinline__ void sel_runmax(int n, int32_t *a, int64_t *sh) {
    const int per = (n + SEL_THREADS - 1) / SEL_THREADS;
    const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
    int32_t m = 0;
    for (int i = lo; i < hi; i++) m = max(m, a[i]);
    // exclusive running max over threads
    const int lane = lane_id(), w = warp_id();
    int32_t incl = m;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int32_t o = __shfl_up_sync(FULL_MASK, incl, d);
        if (lane >= d) incl = max(incl, o);
    }
    if (lane == 31) sh[w] = incl;
    __syncthreads();
    if (w == 0) {
        const int64_t x = lane < SEL_THREADS / 32 ? sh[lane] : 0;
        int64_t xi = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int64_t o = __shfl_up_sync(FULL_MASK, xi, d);
            if (lane >= d) xi = max(xi, o);
        }
        const int64_t prev = __shfl_up_sync(FULL_MASK, xi, 1);
        if (lane < SEL_THREADS / 32) sh[lane] = lane == 0 ? 0 : prev;
    }
    __syncthreads();
    int32_t excl = __shfl_up_sync(FULL_MASK, incl, 1);
    if (lane == 0) excl = 0;
    int32_t run = max(excl, (int32_t)sh[w]);
    for (int i = lo; i < hi; i++) {
        run = max(run, a[i]);
        a[i] = run;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(SEL_THREADS) k_select_small(const unsigned long long *ecount, const int64_t *dM,
                                                              const uint64_t *ekey, const uint32_t *evals,
                                                              const int64_t *gseq, const int64_t *psizes,
                                                              const int64_t *pinbound, int64_t omega, int64_t delta,
                                                              int ibits, int pbits, int64_t *act_ex_out,
                                                              long long *res, bool packed, unsigned long long *work) {
    pdl_entry();
    extern __shared__ unsigned long long smem_u64[];
    __shared__ int64_t sh[33];
    __shared__ long long s_bv[32], s_bk[32];
    const int64_t T = (int64_t)*ecount;
    const int64_t M = *dM;
    if (M == 0) return;  // a speculative launch for a round without movers (the host stops there)
    // algorithmic bytes (profiling): events (12 B), gains in and prefix flags out (16 B per move)
    if (work && threadIdx.x == 0 && T <= SEL_T && M <= SEL_M - 2) atomicAdd(work, 12ull * T + 16ull * M);
    if (T > SEL_T || M > SEL_M - 2) {
        if (threadIdx.x == 0) res[2] = 1;
        return;
    }
    uint64_t *sk = (uint64_t *)smem_u64;
    uint32_t *sv = (uint32_t *)(sk + SEL_T);
    int64_t *ex = (int64_t *)(sv + SEL_T);
    int32_t *gst = (int32_t *)(ex + SEL_T + 1);
    int32_t *sst = gst + SEL_T;
    int32_t *dlt = sst + SEL_T;
    int64_t *cum = (int64_t *)(((uintptr_t)(dlt + SEL_M + 2) + 7) & ~(uintptr_t)7);
    const int n = (int)T;
    // 1. sort the events by key (equal keys only need grouping)
    int np = 1;
    while (np < n) np <<= 1;
    if (packed) {  // key < 2^32: (key, delta) in one u64, register runs + co-rank merges
        for (int i = threadIdx.x; i < n; i += SEL_THREADS) sk[i] = (ekey[i] << 32) | (uint64_t)evals[i];
        __syncthreads();
        block_sort_u64_4096(sk, (uint64_t *)ex, n);  // ex is free until step 2
        for (int i = threadIdx.x; i < n; i += SEL_THREADS) {
            const uint64_t x = sk[i];
            sv[i] = (uint32_t)x;
            sk[i] = x >> 32;
        }
        np = 1;  // skip the bitonic network
    }
    for (int i = threadIdx.x; i < np && !packed; i += SEL_THREADS) {
        sk[i] = i < n ? ekey[i] : ~0ull;
        sv[i] = i < n ? evals[i] : 0u;
    }
    for (int size = 2; size <= np && !packed; size <<= 1) {
        for (int j = size >> 1; j > 0; j >>= 1) {
            __syncthreads();
            for (int t = threadIdx.x; t < (np >> 1); t += SEL_THREADS) {
                const int lo = 2 * j * (t / j) + (t % j), hi = lo + j;
                const bool asc = (lo & size) == 0;
                const uint64_t a = sk[lo], b = sk[hi];
                if ((a > b) == asc) {
                    sk[lo] = b;
                    sk[hi] = a;
                    const uint32_t va = sv[lo];
                    sv[lo] = sv[hi];
                    sv[hi] = va;
                }
            }
        }
    }
    __syncthreads();
    // 2. group / segment starts, deltas' exclusive sums
    for (int k = threadIdx.x; k < n; k += SEL_THREADS) {
        const uint64_t kk = sk[k];
        gst[k] = (k == 0 || sk[k - 1] != kk) ? k : 0;
        sst[k] = (k == 0 || (sk[k - 1] >> ibits) != (kk >> ibits)) ? k : 0;
    }
    for (int i = threadIdx.x; i < (int)M + 2; i += SEL_THREADS) dlt[i] = 0;
    __syncthreads();
    sel_scan_sum(n, [&](int k) { return (int64_t)(int32_t)sv[k]; }, ex, sh);
    sel_runmax(n, gst, sh);
    sel_runmax(n, sst, sh);
    // 3. toggles (refine.py:145-175)
    for (int k = threadIdx.x; k < n; k += SEL_THREADS) {
        const uint64_t kk = sk[k];
        if (k + 1 < n && sk[k + 1] == kk) continue;
        const int track = (int)(kk >> (ibits + pbits));
        const int32_t p = (int32_t)((kk >> ibits) & ((1ull << pbits) - 1ull));
        const int64_t i = (int64_t)(kk & ((1ull << ibits) - 1ull));
        const int64_t base = track ? pinbound[p] : psizes[p];
        const int64_t limit = track ? delta : omega;
        const int64_t s0 = ex[sst[k]];
        const bool after = base + ex[k + 1] - s0 > limit;
        const bool before = base + ex[gst[k]] - s0 > limit;
        if (after != before) atomicAdd(&dlt[i + 1], after ? 1 : -1);
    }
    __syncthreads();
    // 4. active[j] = act_ex[j + 1]; cum = exclusive sums of gain_seq
    int64_t *act = ex;  // reuse: the events are done
    sel_scan_sum((int)M + 1, [&](int j) { return (int64_t)dlt[j]; }, act, sh);
    for (int j = threadIdx.x; j < (int)M + 2; j += SEL_THREADS) act_ex_out[j] = act[j];
    sel_scan_sum((int)M, [&](int j) { return gseq[j]; }, cum, sh);
    // 5. smallest argmax of cum over prefixes with active == 0 (refine.py:244-247)
    long long v = LLONG_MIN, bk = LLONG_MAX;
    for (int j = threadIdx.x; j <= (int)M; j += SEL_THREADS)
        if (act[j + 1] == 0) {
            const long long c = cum[j];
            if (c > v || (c == v && j < bk)) {
                v = c;
                bk = j;
            }
        }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const long long ov = __shfl_xor_sync(FULL_MASK, v, d), ok = __shfl_xor_sync(FULL_MASK, bk, d);
        if (ov > v || (ov == v && ok < bk)) {
            v = ov;
            bk = ok;
        }
    }
    if (lane_id() == 0) {
        s_bv[warp_id()] = v;
        s_bk[warp_id()] = bk;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < SEL_THREADS / 32; w++)
            if (s_bv[w] > v || (s_bv[w] == v && s_bk[w] < bk)) {
                v = s_bv[w];
                bk = s_bk[w];
            }
        res[0] = bk;
        res[1] = v;
        res[2] = 0;
    }
}

__global__ void k_apply(int64_t k, const int32_t *node, const int32_t *to, int32_t *assign) {
    pdl_entry();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < k) assign[node[i]] = to[i];
}

}  // namespace

// builds the run lists for `assign`; connectivity accumulates into *conn
// (device), distinct-inbound counts into pinbound when requested
static void build_runs(Ctx &c, const DLevel &L, const DWeights &W, const int32_t *assign, Runs &r,
                       int32_t *tmp_parts, int64_t *pinbound, int32_t K, unsigned long long *conn,
                       int32_t max_edge_pins) {
    KScope ks(c, "edge_runs", (double)(20.0 * L.E + 20.0 * L.U + 8.0 * L.Pd));
    c.zero(conn, 1);
    if (pinbound) c.zero(pinbound, K);
    if (max_edge_pins <= 128) {
        if (L.E > 0) {
            static int g = resident_grid(c, k_edge_runs_fused, 256, 0);
            int blocks = (int)std::min<int64_t>(cdiv(L.E, 8), g);
            pdl_launch(k_edge_runs_fused, blocks, 256, 0, c.stream, L.E, L.pin_off, L.pin_dat, L.dst_off, L.dst_dat, assign,
                                                           W.wi, r, conn, pinbound);
            DHGP_LAUNCHED(c);
        }
        return;
    }
    seg_sort(c, L.E, L.pin_off, L.pin_dat, assign, tmp_parts);
    if (L.E > 0) {
        if (L.U >= 12 * (int64_t)L.E) {
            int blocks = (int)std::min<int64_t>(cdiv(L.E, 8), (int64_t)c.num_sms * 16);
            pdl_launch(k_edge_runs_warp, blocks, 256, 0, c.stream, L.E, L.pin_off, tmp_parts, L.dst_off, L.dst_dat, assign,
                                                          W.wi, r, conn, pinbound);
        } else {
            pdl_launch(k_edge_runs, (unsigned)cdiv(L.E, 256), 256, 0, c.stream, L.E, L.pin_off, tmp_parts, L.dst_off,
                                                                       L.dst_dat, assign, W.wi, r, conn, pinbound);
        }
        DHGP_LAUNCHED(c);
    }
}

namespace {
// moves: sequence arrays from the radix-sorted (key, node) pairs; M on device
__global__ void k_build_moves_dn(const int64_t *dM, const uint32_t *sorted_nodes, const int32_t *assign,
                                 const int32_t *target, const int64_t *gain, int32_t *node, int32_t *from, int32_t *to,
                                 int64_t *giso, int32_t *pos, bool spec) {
    pdl_entry();
    const int64_t M = *dM;
    if (spec && M > kSpecCap) return;  // speculative launch, M too large
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t n = (int32_t)sorted_nodes[i];
        node[i] = n;
        from[i] = assign[n];
        to[i] = target[n];
        giso[i] = gain[n];
        pos[n] = (int32_t)i;
    }
}
// A15: gains corrected for earlier moves, rules (a)-(d) (_kernels.pyx:326-363),
// computed per h-edge: the movers among an h-edge's pins, in sequence order,
// give every (move, h-edge) term from counts over the earlier movers on that
// h-edge — O(sum |e|) for the round instead of O(sum over moves of the pins
// of their h-edges).  Terms are integers, summed with atomics (exact).
__device__ __forceinline__ int64_t seq_net(int64_t we, int32_t base_ps, int32_t base_pd, int32_t leav_pd,
                                           int32_t ent_pd, int32_t leav_ps, int32_t ent_ps) {
    int64_t net = 0;
    if (base_pd > 0) {
        if (leav_pd - ent_pd == base_pd) net -= we;
    } else if (ent_pd > 0) {
        net += we;
    }
    if (base_ps == 1) {
        if (ent_ps > 0) net -= we;
    } else if (base_ps - 1 > 0 && leav_ps - ent_ps == base_ps - 1) {
        net += we;
    }
    return net;
}
// the same for h-edges with many movers: a block gathers and sorts them, each
// thread takes some movers and counts over the earlier ones
constexpr int kSgBlockMax = 2048;
__global__ void k_seq_gains_edge_block(const int64_t *pin_off, const int32_t *pin_dat, const int64_t *wi, Runs r,
                                       const int32_t *pos, const int32_t *from, const int32_t *to,
                                       unsigned long long *gacc, const int32_t *big_list, const int32_t *big_count,
                                       int32_t *huge, int32_t *huge_count, int mv_max) {
    pdl_entry();
    __shared__ uint32_t smv[kSgBlockMax];
    __shared__ int32_t sf[kSgBlockMax], st[kSgBlockMax];
    __shared__ int32_t snm;
    const int nbig = *big_count;
    for (int t = blockIdx.x; t < nbig; t += gridDim.x) {
        const int32_t e = big_list[t];
        if (threadIdx.x == 0) snm = 0;
        __syncthreads();
        const int64_t lo = pin_off[e], hi = pin_off[e + 1];
        for (int64_t pp = lo + threadIdx.x; pp < hi; pp += blockDim.x) {
            const int32_t j = pos[pin_dat[pp]];
            if (j >= 0) {
                const int q = atomicAdd(&snm, 1);
                if (q < kSgBlockMax) smv[q] = (uint32_t)j;
            }
        }
        __syncthreads();
        const int nm = snm;
        if (nm > mv_max) {  // global-memory path (k_edge_movers_huge)
            if (threadIdx.x == 0) huge[atomicAdd(huge_count, 1)] = e;
            __syncthreads();
            continue;
        }
        const int np = next_pow2(nm);
        for (int q = nm + threadIdx.x; q < np; q += blockDim.x) smv[q] = 0xffffffffu;
        block_bitonic_sort32(smv, np);
        for (int a = threadIdx.x; a < nm; a += blockDim.x) {
            sf[a] = from[smv[a]];
            st[a] = to[smv[a]];
        }
        __syncthreads();
        const int64_t we = wi[e];
        const int32_t lam = r.len[e];
        const int64_t ro = r.off[e];
        for (int a = threadIdx.x; a < nm; a += blockDim.x) {
            const int32_t ps = sf[a], pd = st[a];
            int32_t leav_pd = 0, ent_pd = 0, leav_ps = 0, ent_ps = 0;
            for (int b = 0; b < a; b++) {
                leav_pd += sf[b] == pd;
                ent_pd += st[b] == pd;
                leav_ps += sf[b] == ps;
                ent_ps += st[b] == ps;
            }
            int32_t k = run_find(r, ro, lam, ps);
            const int32_t base_ps = k >= 0 ? r.pc[2 * (ro + k) + 1] : 0;
            k = run_find(r, ro, lam, pd);
            const int32_t base_pd = k >= 0 ? r.pc[2 * (ro + k) + 1] : 0;
            const int64_t net = seq_net(we, base_ps, base_pd, leav_pd, ent_pd, leav_ps, ent_ps);
            if (net) atomicAdd(&gacc[smv[a]], (unsigned long long)net);
        }
        __syncthreads();
    }
}

// H-edges with more movers than the block kernels hold in shared memory: a
// CTA per h-edge with global scratch.  The movers' sequence positions are
// sorted; the (from, position) and (to, position) keys are sorted too, so
// "#earlier movers leaving / entering part x" for mover a is the distance
// between two lower bounds — O(m log m) per h-edge.  mode 0: sequence-gain
// terms over the pins (base = pin counts, rules (a)-(d)); mode 1: inbound
// crossings over the destination pins (base = destination-pin counts), the
// same running count as the per-part sweep of k_inbound_events_block.
__device__ __forceinline__ int64_t lb_u64(const unsigned long long *a, int64_t n, unsigned long long key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t m = (lo + hi) >> 1;
        if (a[m] < key) lo = m + 1; else hi = m;
    }
    return lo;
}
__device__ __forceinline__ int32_t earlier(const unsigned long long *keys, int64_t nm, int32_t part, int64_t a) {
    const unsigned long long k0 = (unsigned long long)(uint32_t)part << 32;
    return (int32_t)(lb_u64(keys, nm, k0 | (unsigned long long)a) - lb_u64(keys, nm, k0));
}
__global__ void __launch_bounds__(1024) k_edge_movers_huge(int mode, const int64_t *off, const int32_t *dat,
                                                           const int64_t *wi, Runs r, const int32_t *pos,
                                                           const int32_t *from, const int32_t *to,
                                                           unsigned long long *gacc, EvArgs ev, const int32_t *huge,
                                                           const int32_t *huge_count, uint8_t *gscr, int64_t gcap) {
    pdl_entry();
    __shared__ int32_t snm;
    const int nh = *huge_count;
    uint32_t *smv = (uint32_t *)(gscr + (int64_t)blockIdx.x * ((20 * gcap + 15) & ~(int64_t)7));
    unsigned long long *kf = (unsigned long long *)(smv + gcap + (gcap & 1));
    unsigned long long *kt = kf + gcap;
    for (int t = blockIdx.x; t < nh; t += gridDim.x) {
        const int32_t e = huge[t];
        if (threadIdx.x == 0) snm = 0;
        __syncthreads();
        for (int64_t q = off[e] + threadIdx.x; q < off[e + 1]; q += blockDim.x) {
            const int32_t j = pos[dat[q]];
            if (j >= 0) smv[atomicAdd(&snm, 1)] = (uint32_t)j;
        }
        __syncthreads();
        const int64_t nm = snm;
        block_sort_asc_any<uint32_t>(smv, nm);
        for (int64_t a = threadIdx.x; a < nm; a += blockDim.x) {
            const int32_t i = (int32_t)smv[a];
            kf[a] = ((unsigned long long)(uint32_t)from[i] << 32) | (unsigned long long)a;
            kt[a] = ((unsigned long long)(uint32_t)to[i] << 32) | (unsigned long long)a;
        }
        block_sort_asc_any<unsigned long long>(kf, nm);
        block_sort_asc_any<unsigned long long>(kt, nm);
        const int64_t ro = r.off[e];
        const int32_t lam = r.len[e];
        for (int64_t a = threadIdx.x; a < nm; a += blockDim.x) {
            const int32_t i = (int32_t)smv[a], ps = from[i], pd = to[i];
            const int32_t leav_ps = earlier(kf, nm, ps, a), ent_ps = earlier(kt, nm, ps, a);
            const int32_t leav_pd = earlier(kf, nm, pd, a), ent_pd = earlier(kt, nm, pd, a);
            const int32_t ks = run_find(r, ro, lam, ps), kd = run_find(r, ro, lam, pd);
            if (mode == 0) {
                const int32_t base_ps = ks >= 0 ? r.pc[2 * (ro + ks) + 1] : 0;
                const int32_t base_pd = kd >= 0 ? r.pc[2 * (ro + kd) + 1] : 0;
                const int64_t net = seq_net(wi[e], base_ps, base_pd, leav_pd, ent_pd, leav_ps, ent_ps);
                if (net) atomicAdd(&gacc[i], (unsigned long long)net);
            } else if (ps != pd) {
                const int32_t in_ps = ks >= 0 ? r.cin[ro + ks] : 0, in_pd = kd >= 0 ? r.cin[ro + kd] : 0;
                if (in_ps - leav_ps + ent_ps - 1 == 0) inbound_leave(ev, i);
                if (in_pd - leav_pd + ent_pd + 1 == 1) inbound_enter(ev, i);
            }
        }
        __syncthreads();
    }
}

// Warp per h-edge (all E, or the movers' h-edge list): the round's terms of
// one h-edge from its movers in sequence order — the sequence-gain terms of
// rules (a)-(d) over its pins (A15) and the inbound-track crossings over its
// destination pins (A17).  Lane a holds the a-th mover; the counts over the
// earlier movers are shuffles, so each term is independent:
//   dc[p] before mover a leaves = pins_in[e, p] - #{b < a: from_b = p} + #{b < a: to_b = p}
// and "--dc == 0" / "++dc == 1" of the sequential walk become tests on it.
// H-edges with more than `cap` movers go to the block kernels.
__device__ __forceinline__ int warp_collect_movers(const int32_t *dat, int64_t lo, int64_t hi, const int32_t *pos,
                                                   int32_t *smv) {
    const int lane = lane_id();
    const uint32_t lt = (1u << lane) - 1u;
    int nm = 0;
    for (int64_t b = lo; b < hi; b += 32) {
        const int64_t q = b + lane;
        const int32_t j = q < hi ? pos[dat[q]] : -1;
        const uint32_t bal = __ballot_sync(FULL_MASK, j >= 0);
        if (j >= 0) {
            const int slot = nm + __popc(bal & lt);
            if (slot < 64) smv[slot] = j;
        }
        nm += __popc(bal);
    }
    __syncwarp();
    return nm;
}
// the terms of one h-edge from its movers, lane a holding the a-th mover in
// sequence order (i = its move index; nm <= 32 movers)
__device__ __forceinline__ void edge_seq_terms(int32_t e, int nm, int32_t i, const int64_t *wi, const Runs &r,
                                               const int32_t *from, const int32_t *to, unsigned long long *gacc) {
    const int lane = lane_id();
    const int64_t ro = r.off[e];
    const int32_t lam = r.len[e];
    const int32_t ps = lane < nm ? from[i] : -1, pd = lane < nm ? to[i] : -1;
    int32_t leav_pd = 0, ent_pd = 0, leav_ps = 0, ent_ps = 0;
    for (int b = 0; b < nm; b++) {
        const int32_t fb = __shfl_sync(FULL_MASK, ps, b), tb = __shfl_sync(FULL_MASK, pd, b);
        if (b < lane) {
            leav_pd += fb == pd;
            ent_pd += tb == pd;
            leav_ps += fb == ps;
            ent_ps += tb == ps;
        }
    }
    if (lane < nm) {
        int32_t k = run_find(r, ro, lam, ps);
        const int32_t base_ps = k >= 0 ? r.pc[2 * (ro + k) + 1] : 0;
        k = run_find(r, ro, lam, pd);
        const int32_t base_pd = k >= 0 ? r.pc[2 * (ro + k) + 1] : 0;
        const int64_t net = seq_net(wi[e], base_ps, base_pd, leav_pd, ent_pd, leav_ps, ent_ps);
        if (net) atomicAdd(&gacc[i], (unsigned long long)net);
    }
}
__device__ __forceinline__ void edge_event_terms(int32_t e, int nm, int32_t i, const Runs &r, const int32_t *from,
                                                 const int32_t *to, EvArgs ev) {
    const int lane = lane_id();
    const int64_t ro = r.off[e];
    const int32_t lam = r.len[e];
    const int32_t pf = lane < nm ? from[i] : -1, pt = lane < nm ? to[i] : -1;
    int32_t df = 0, dt = 0;  // net arrivals minus departures of pf / pt before mover a
    for (int b = 0; b < nm; b++) {
        const int32_t fb = __shfl_sync(FULL_MASK, pf, b), tb = __shfl_sync(FULL_MASK, pt, b);
        if (b < lane) {
            df += (tb == pf) - (fb == pf);
            dt += (tb == pt) - (fb == pt);
        }
    }
    if (lane < nm) {
        int32_t k = run_find(r, ro, lam, pf);
        if ((k >= 0 ? r.cin[ro + k] : 0) + df - 1 == 0) inbound_leave(ev, i);
        k = run_find(r, ro, lam, pt);
        if ((k >= 0 ? r.cin[ro + k] : 0) + dt == 0) inbound_enter(ev, i);
    }
}

// the same for 33..64 movers: lane a holds movers a and 32 + a
__device__ __forceinline__ void edge_seq_terms2(int32_t e, int nm, const int32_t (&i)[2], const int64_t *wi,
                                                const Runs &r, const int32_t *from, const int32_t *to,
                                                unsigned long long *gacc) {
    const int lane = lane_id();
    const int64_t ro = r.off[e];
    const int32_t lam = r.len[e];
    int32_t ps[2], pd[2], leav_pd[2] = {0, 0}, ent_pd[2] = {0, 0}, leav_ps[2] = {0, 0}, ent_ps[2] = {0, 0};
#pragma unroll
    for (int k = 0; k < 2; k++) {
        const bool v = 32 * k + lane < nm;
        ps[k] = v ? from[i[k]] : -1;
        pd[k] = v ? to[i[k]] : -1;
    }
    for (int b = 0; b < nm; b++) {
        const int kb = b >> 5, lb = b & 31;
        const int32_t fb = __shfl_sync(FULL_MASK, kb ? ps[1] : ps[0], lb);
        const int32_t tb = __shfl_sync(FULL_MASK, kb ? pd[1] : pd[0], lb);
#pragma unroll
        for (int k = 0; k < 2; k++)
            if (b < 32 * k + lane) {
                leav_pd[k] += fb == pd[k];
                ent_pd[k] += tb == pd[k];
                leav_ps[k] += fb == ps[k];
                ent_ps[k] += tb == ps[k];
            }
    }
#pragma unroll
    for (int k = 0; k < 2; k++)
        if (32 * k + lane < nm) {
            int32_t q = run_find(r, ro, lam, ps[k]);
            const int32_t base_ps = q >= 0 ? r.pc[2 * (ro + q) + 1] : 0;
            q = run_find(r, ro, lam, pd[k]);
            const int32_t base_pd = q >= 0 ? r.pc[2 * (ro + q) + 1] : 0;
            const int64_t net = seq_net(wi[e], base_ps, base_pd, leav_pd[k], ent_pd[k], leav_ps[k], ent_ps[k]);
            if (net) atomicAdd(&gacc[i[k]], (unsigned long long)net);
        }
}
__device__ __forceinline__ void edge_event_terms2(int32_t e, int nm, const int32_t (&i)[2], const Runs &r,
                                                  const int32_t *from, const int32_t *to, EvArgs ev) {
    const int lane = lane_id();
    const int64_t ro = r.off[e];
    const int32_t lam = r.len[e];
    int32_t pf[2], pt[2], df[2] = {0, 0}, dt[2] = {0, 0};
#pragma unroll
    for (int k = 0; k < 2; k++) {
        const bool v = 32 * k + lane < nm;
        pf[k] = v ? from[i[k]] : -1;
        pt[k] = v ? to[i[k]] : -1;
    }
    for (int b = 0; b < nm; b++) {
        const int kb = b >> 5, lb = b & 31;
        const int32_t fb = __shfl_sync(FULL_MASK, kb ? pf[1] : pf[0], lb);
        const int32_t tb = __shfl_sync(FULL_MASK, kb ? pt[1] : pt[0], lb);
#pragma unroll
        for (int k = 0; k < 2; k++)
            if (b < 32 * k + lane) {
                df[k] += (tb == pf[k]) - (fb == pf[k]);
                dt[k] += (tb == pt[k]) - (fb == pt[k]);
            }
    }
#pragma unroll
    for (int k = 0; k < 2; k++)
        if (32 * k + lane < nm) {
            int32_t q = run_find(r, ro, lam, pf[k]);
            if ((q >= 0 ? r.cin[ro + q] : 0) + df[k] - 1 == 0) inbound_leave(ev, i[k]);
            q = run_find(r, ro, lam, pt[k]);
            if ((q >= 0 ? r.cin[ro + q] : 0) + dt[k] == 0) inbound_enter(ev, i[k]);
        }
}

// one h-edge's round terms, the warp together (movers gathered from its pin
// lists by position, sorted by sequence index; more than `cap` movers go to
// the block kernels' lists)
__device__ __forceinline__ void round_edge_warp(int32_t e, const int64_t *pin_off, const int32_t *pin_dat,
                                                const int64_t *dst_off, const int32_t *dst_dat, const int64_t *wi,
                                                const Runs &r, const int32_t *pos, const int32_t *from,
                                                const int32_t *to, unsigned long long *gacc, const EvArgs &ev,
                                                int32_t *sg_big, int32_t *sg_count, int32_t *ev_big,
                                                int32_t *ev_count, int cap, int32_t *smv) {
    const int lane = lane_id();
    // ---- sequence gains over all pins --------------------------------
    int nm = warp_collect_movers(pin_dat, pin_off[e], pin_off[e + 1], pos, smv);
    if (nm > cap) {
        if (lane == 0) sg_big[atomicAdd(sg_count, 1)] = e;
    } else if (nm > 32) {
        uint32_t v[2] = {(uint32_t)smv[lane], 32 + lane < nm ? (uint32_t)smv[32 + lane] : 0xffffffffu};
        warp_bitonic_sort<2>(v);
        const int32_t i2[2] = {(int32_t)v[0], (int32_t)v[1]};
        edge_seq_terms2(e, nm, i2, wi, r, from, to, gacc);
    } else if (nm > 0) {
        uint32_t v[1] = {lane < nm ? (uint32_t)smv[lane] : 0xffffffffu};
        warp_bitonic_sort<1>(v);
        edge_seq_terms(e, nm, (int32_t)v[0], wi, r, from, to, gacc);
    }
    __syncwarp();
    // ---- inbound-track crossings over the destination pins -----------
    nm = warp_collect_movers(dst_dat, dst_off[e], dst_off[e + 1], pos, smv);
    if (nm > cap) {
        if (lane == 0) ev_big[atomicAdd(ev_count, 1)] = e;
    } else if (nm > 32) {
        uint32_t v[2] = {(uint32_t)smv[lane], 32 + lane < nm ? (uint32_t)smv[32 + lane] : 0xffffffffu};
        warp_bitonic_sort<2>(v);
        const int32_t i2[2] = {(int32_t)v[0], (int32_t)v[1]};
        edge_event_terms2(e, nm, i2, r, from, to, ev);
    } else if (nm > 0) {
        uint32_t v[1] = {lane < nm ? (uint32_t)smv[lane] : 0xffffffffu};
        warp_bitonic_sort<1>(v);
        edge_event_terms(e, nm, (int32_t)v[0], r, from, to, ev);
    }
    __syncwarp();
}

__global__ void __launch_bounds__(256, 6) k_round_edges(int32_t E, const int32_t *elist, const int32_t *ecount,
                                                     const int64_t *pin_off, const int32_t *pin_dat,
                                                     const int64_t *dst_off, const int32_t *dst_dat,
                                                     const int64_t *wi, Runs r, const int32_t *pos,
                                                     const int32_t *from, const int32_t *to,
                                                     unsigned long long *gacc, EvArgs ev, int32_t *sg_big,
                                                     int32_t *sg_count, int32_t *ev_big, int32_t *ev_count,
                                                     int cap, const int64_t *spec_m, unsigned long long *work,
                                                     int64_t elo, int64_t ehi, const int32_t *alt_list,
                                                     const int32_t *alt_count, int64_t fe_min) {
    pdl_entry();
    if (spec_m && *spec_m > kSpecCap) return;  // speculative launch, M too large
    __shared__ int32_t s_mv[8][64];
    const int lane = lane_id();
    int32_t *smv = s_mv[warp_id()];
    // after k_round_edges_flat: when it took the round (at least fe_min
    // h-edges), only the h-edges it listed remain; else all of them
    if (alt_list && (elist ? (int64_t)*ecount : (int64_t)E) >= fe_min) {
        elist = alt_list;
        ecount = alt_count;
        work = nullptr;  // counted by the flat kernel
    }
    const int64_t ne = elist ? (int64_t)*ecount : (int64_t)E;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t idx = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id(); idx < ne; idx += nw) {
        const int32_t e = elist ? elist[idx] : (int32_t)idx;
        if (e < elo || e >= ehi) continue;  // another rank's h-edge (node-range sharding by h-edge id)
        // algorithmic bytes (profiling): pins and destination pins with their
        // positions (8 B each), offsets / runs / weight (48 B)
        if (work && lane == 0)
            atomicAdd(work, 8ull * (uint64_t)(pin_off[e + 1] - pin_off[e] + dst_off[e + 1] - dst_off[e]) + 48ull);
        round_edge_warp(e, pin_off, pin_dat, dst_off, dst_dat, wi, r, pos, from, to, gacc, ev, sg_big, sg_count, ev_big,
                        ev_count, cap, smv);
    }
}

// The same terms for many small h-edges at once.  Per-edge warps wait on a
// chain of dependent loads (list entry -> offsets -> pins -> positions ->
// moves -> runs) for a handful of pins each; here a warp takes 32 h-edges and
// flattens the pins of those with at most FE_SMALL pins over its lanes (up to
// FE_CAP pins per pass, eight in flight per lane), so one chain serves 32
// h-edges.  The movers found are appended in slot order, i.e. grouped by
// h-edge; a mover's counts over the earlier movers of its h-edge are taken by
// comparing sequence indices within the group (no sort), and a group's first
// mover has no terms (seq_net of zero counts is 0), so run lists are searched
// only where a term can be non-zero.  Larger h-edges are listed for the
// per-edge kernel (k_round_edges over that list).
constexpr int FE_WARPS = 8;
constexpr int FE_CAP = 256;
constexpr int FE_SMALL = 64;
struct FlatWarp {
    int32_t j[FE_CAP], f[FE_CAP], t[FE_CAP];
    uint8_t own[FE_CAP];
    int32_t cnt[32], seg[32], e[32], lam[32], dfr[32];
    int64_t ro[32];
    long long net[32];
};
constexpr int FE_GROUP = 16; // more movers on one h-edge: the per-edge warp kernel

// mode 0: the pins (sequence-gain terms); mode 1: the destination pins
// (inbound crossings).  Lanes with take=false contribute nothing.
template <int MODE>
__device__ __forceinline__ void flat_pass(FlatWarp &fw, bool take, int64_t lo, int len, const int32_t *dat,
                                          const int64_t *wi, const Runs &r, const int32_t *pos, const int32_t *from,
                                          const int32_t *to, unsigned long long *gacc, const EvArgs &ev,
                                          int32_t *big, int32_t *big_count, int cap, int32_t *lg_list,
                                          int32_t *lg_count) {
    const int lane = lane_id();
    const uint32_t lt = (1u << lane) - 1u;
    if (!take) len = 0;
    const int incl = warp_incl_scan(len);
    const int total = __shfl_sync(FULL_MASK, incl, 31);
    const int excl = incl - len;
    int nent = 0;
    constexpr int U = 8;
    for (int s0 = 0; s0 < total; s0 += 32 * U) {
        int32_t jj[U], ow[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int s = s0 + u * 32 + lane;
            int owner = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int ex = __shfl_sync(FULL_MASK, excl, owner + step);
                if (ex <= s) owner += step;
            }
            const int64_t olo = __shfl_sync(FULL_MASK, lo, owner);
            const int oex = __shfl_sync(FULL_MASK, excl, owner);
            ow[u] = owner;
            jj[u] = s < total ? dat[olo + (s - oex)] : -1;
        }
#pragma unroll
        for (int u = 0; u < U; u++) jj[u] = jj[u] >= 0 ? pos[jj[u]] : -1;
#pragma unroll
        for (int u = 0; u < U; u++) {
            const bool mv = jj[u] >= 0;
            const uint32_t bal = __ballot_sync(FULL_MASK, mv);
            if (mv) {
                const int k = nent + __popc(bal & lt);
                fw.j[k] = jj[u];
                fw.own[k] = (uint8_t)ow[u];
            }
            nent += __popc(bal);
        }
    }
    if (MODE == 0) fw.dfr[lane] = 0;
    if (nent == 0) return;  // uniform
    __syncwarp();
    {
        // the entries ascend by owner: each lane finds its group by search
        // (no same-address shared atomics)
        int a = 0, b = nent;
        while (a < b) {
            const int mid = (a + b) >> 1;
            if (fw.own[mid] < lane) a = mid + 1; else b = mid;
        }
        int z = a;
        b = nent;
        while (z < b) {
            const int mid = (z + b) >> 1;
            if (fw.own[mid] <= lane) z = mid + 1; else b = mid;
        }
        const int c = z - a;
        fw.cnt[lane] = c;
        fw.seg[lane] = a;
        // many movers on one h-edge (the O(c^2) counts would serialise on
        // one lane): the h-edge goes whole to the per-edge warp kernel,
        // decided on its pins (a superset of its destination pins)
        bool dfr = false;
        if (MODE == 0) {
            dfr = c > FE_GROUP;
            fw.dfr[lane] = dfr;
            const uint32_t bal = __ballot_sync(FULL_MASK, dfr);
            if (bal) {
                int b = 0;
                if (lane == 0) b = atomicAdd(lg_count, __popc(bal));
                b = __shfl_sync(FULL_MASK, b, 0);
                if (dfr) lg_list[b + __popc(bal & lt)] = fw.e[lane];
            }
        } else {
            dfr = fw.dfr[lane];
        }
        // a group beyond the warp tiers' capacity goes to the block kernels
        if (!dfr && c > cap) big[atomicAdd(big_count, 1)] = fw.e[lane];
    }
    for (int k = lane; k < nent; k += 32) {
        const int32_t jk = fw.j[k];
        fw.f[k] = from[jk];
        fw.t[k] = to[jk];
    }
    __syncwarp();
    // TU entries per lane at a time: their run-list searches advance in
    // lockstep, so a lane waits for one chain of loads per TU entries
    constexpr int TU = 2;
    for (int k0 = 0; k0 < nent; k0 += 32 * TU) {
        // per entry: sequence index, parts (from, to), its h-edge's warp slot
        // (-1 = no term) and the four counts over the earlier movers, packed
        // a byte each (at most FE_GROUP movers per group)
        int32_t jk[TU], pp[2 * TU], ow[TU];
        uint32_t dd[TU];
#pragma unroll
        for (int u = 0; u < TU; u++) {
            const int k = k0 + u * 32 + lane;
            ow[u] = -1;
            jk[u] = pp[2 * u] = pp[2 * u + 1] = 0;
            dd[u] = 0;
            if (k >= nent) continue;
            const int o = fw.own[k];
            const int c = fw.cnt[o];
            if (c > cap || fw.dfr[o]) continue;
            if (MODE == 0 && c == 1) continue;  // a lone mover: no sequence term
            const int b0 = fw.seg[o];
            jk[u] = fw.j[k];
            const int32_t pf = fw.f[k], pt = fw.t[k];
            uint32_t d = 0;
            for (int b = b0; b < b0 + c; b++) {
                if (fw.j[b] >= jk[u]) continue;
                const int32_t fb = fw.f[b], tb = fw.t[b];
                d += (fb == pt ? 1u : 0u)          // leav_pd (mode 0) / departures from pt (mode 1)
                     + (tb == pt ? 1u << 8 : 0u)   // ent_pd / arrivals at pt
                     + (fb == pf ? 1u << 16 : 0u)  // leav_ps / departures from pf
                     + (tb == pf ? 1u << 24 : 0u); // ent_ps / arrivals at pf
            }
            if (MODE == 0 && !d) continue;  // the first of its group: no term
            ow[u] = o;
            dd[u] = d;
            pp[2 * u] = pf;
            pp[2 * u + 1] = pt;
        }
        // lower bounds of pf / pt among the h-edge's run parts, in lockstep
        int32_t lo[2 * TU], hi[2 * TU];
#pragma unroll
        for (int q = 0; q < 2 * TU; q++) {
            lo[q] = 0;
            hi[q] = ow[q >> 1] >= 0 ? fw.lam[ow[q >> 1]] : 0;
        }
        while (true) {
            bool any = false;
            int32_t v[2 * TU];
#pragma unroll
            for (int q = 0; q < 2 * TU; q++)
                if (lo[q] < hi[q]) {
                    any = true;
                    v[q] = r.pc[2 * (fw.ro[ow[q >> 1]] + ((lo[q] + hi[q]) >> 1))];
                }
            if (!any) break;
#pragma unroll
            for (int q = 0; q < 2 * TU; q++)
                if (lo[q] < hi[q]) {
                    const int32_t mid = (lo[q] + hi[q]) >> 1;
                    if (v[q] < pp[q])
                        lo[q] = mid + 1;
                    else
                        hi[q] = mid;
                }
        }
        // the run's pin count (mode 0) / destination-pin count (mode 1); 0 if absent
        int32_t cv[2 * TU];
#pragma unroll
        for (int q = 0; q < 2 * TU; q++) {
            cv[q] = 0;
            const int o = ow[q >> 1];
            if (o >= 0 && lo[q] < fw.lam[o]) {
                const int64_t slot = fw.ro[o] + lo[q];
                const int2 pc = *(const int2 *)(r.pc + 2 * slot);
                if (pc.x == pp[q]) cv[q] = MODE == 0 ? pc.y : r.cin[slot];
            }
        }
        // the lanes' entries often belong to the same move (few movers, many
        // h-edges): one atomic per distinct move and warp instruction
#pragma unroll
        for (int u = 0; u < TU; u++) {
            const int32_t a0 = dd[u] & 255, a1 = (dd[u] >> 8) & 255, a2 = (dd[u] >> 16) & 255, a3 = dd[u] >> 24;
            const bool on = ow[u] >= 0;
            const uint32_t grp = __match_any_sync(FULL_MASK, on ? jk[u] : -1 - lane);
            const bool lead = on && lane == __ffs(grp) - 1;
            if (MODE == 0) {
                const int64_t net = on ? seq_net(wi[fw.e[ow[u]]], cv[2 * u], cv[2 * u + 1], a0, a1, a2, a3) : 0;
                fw.net[lane] = net;
                __syncwarp();
                if (lead) {
                    long long tot = 0;
                    for (uint32_t g = grp; g; g &= g - 1) tot += fw.net[__ffs(g) - 1];
                    if (tot) atomicAdd(&gacc[jk[u]], (unsigned long long)tot);
                }
                __syncwarp();
            } else {
                const uint32_t lv = __ballot_sync(FULL_MASK, on && cv[2 * u] + (a3 - a2) - 1 == 0) & grp;
                const uint32_t en = __ballot_sync(FULL_MASK, on && cv[2 * u + 1] + (a1 - a0) == 0) & grp;
                if (lead && lv) atomicSub(&ev.in_from[jk[u]], __popc(lv));
                if (lead && en) atomicAdd(&ev.in_to[jk[u]], __popc(en));
            }
        }
    }
    __syncwarp();
}

__global__ void __launch_bounds__(FE_WARPS * 32, 4) k_round_edges_flat(
    int32_t E, const int32_t *elist, const int32_t *ecount, const int64_t *pin_off, const int32_t *pin_dat,
    const int64_t *dst_off, const int32_t *dst_dat, const int64_t *wi, Runs r, const int32_t *pos,
    const int32_t *from, const int32_t *to, unsigned long long *gacc, EvArgs ev, int32_t *sg_big,
    int32_t *sg_count, int32_t *ev_big, int32_t *ev_count, int cap, const int64_t *spec_m,
    unsigned long long *work, int64_t elo, int64_t ehi, int32_t *lg_list, int32_t *lg_count, int64_t fe_min) {
    pdl_entry();
    if (spec_m && *spec_m > kSpecCap) return;  // speculative launch, M too large
    // few h-edges: a chunk's load chain would be the round's critical path,
    // the per-edge kernel (a warp each) takes them all
    if ((elist ? (int64_t)*ecount : (int64_t)E) < fe_min) return;
    __shared__ FlatWarp fe_w[FE_WARPS];
    FlatWarp &fw = fe_w[warp_id()];
    const int lane = lane_id();
    const int64_t ne = elist ? (int64_t)*ecount : (int64_t)E;
    const int64_t nw = (int64_t)gridDim.x * FE_WARPS;
    for (int64_t base = ((int64_t)blockIdx.x * FE_WARPS + warp_id()) * 32; base < ne; base += nw * 32) {
        const int64_t idx = base + lane;
        int32_t e = -1;
        if (idx < ne) {
            e = elist ? elist[idx] : (int32_t)idx;
            if (e < elo || e >= ehi) e = -1;  // another rank's h-edge
        }
        int64_t plo = 0, phi = 0, dlo = 0, dhi = 0, ro = 0;
        int32_t lam = 0;
        if (e >= 0) {
            plo = pin_off[e];
            phi = pin_off[e + 1];
            dlo = dst_off[e];
            dhi = dst_off[e + 1];
            ro = r.off[e];
            lam = r.len[e];
        }
        if (work) {  // algorithmic bytes (profiling), as k_round_edges
            unsigned long long b = e >= 0 ? 8ull * (uint64_t)(phi - plo + dhi - dlo) + 48ull : 0ull;
            b = warp_sum(b);
            if (lane == 0 && b) atomicAdd(work, b);
        }
        const bool small = e >= 0 && phi - plo <= FE_SMALL;
        fw.e[lane] = e;
        fw.ro[lane] = ro;
        fw.lam[lane] = lam;
        uint32_t rem = __ballot_sync(FULL_MASK, small);
        while (rem) {  // passes over the small h-edges, at most FE_CAP pins each
            const bool mine = (rem >> lane) & 1u;
            const int in = warp_incl_scan(mine ? (int)(phi - plo) : 0);
            const bool take = mine && in <= FE_CAP;
            rem &= ~__ballot_sync(FULL_MASK, take);
            flat_pass<0>(fw, take, plo, (int)(phi - plo), pin_dat, wi, r, pos, from, to, gacc, ev, sg_big, sg_count,
                         cap, lg_list, lg_count);
            flat_pass<1>(fw, take, dlo, (int)(dhi - dlo), dst_dat, wi, r, pos, from, to, gacc, ev, ev_big, ev_count,
                         cap, lg_list, lg_count);
        }
        // larger h-edges: listed for the per-edge warp kernel (a warp each)
        const bool lg = e >= 0 && !small;
        const uint32_t bal = __ballot_sync(FULL_MASK, lg);
        if (bal) {
            int b = 0;
            if (lane == 0) b = atomicAdd(lg_count, __popc(bal));
            b = __shfl_sync(FULL_MASK, b, 0);
            if (lg) lg_list[b + __popc(bal & ((1u << lane) - 1u))] = e;
        }
        __syncwarp();
    }
}

// movers compacted in any order (they are sorted right after): key = the
// sequence key (gain desc) with the node id in the low 32 bits, so equal
// gains order by node (refine.py:108-110) in any sort; pos[] reset on the way
__global__ void k_mover_compact(int32_t N, const int32_t *target, const int64_t *gain, int64_t gmax, uint64_t *keys,
                                uint32_t *vals, int32_t *pos, unsigned long long *count, int32_t *reset) {
    pdl_entry();
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (reset && n == 0) *reset = 0;
    const bool mv = n < N && target[n] >= 0;
    if (n < N) pos[n] = -1;
    const uint32_t bal = __ballot_sync(FULL_MASK, mv);
    if (!bal) return;
    const int lane = lane_id();
    unsigned long long base = 0;
    if (lane == __ffs(bal) - 1) base = atomicAdd(count, (unsigned long long)__popc(bal));
    base = __shfl_sync(FULL_MASK, base, __ffs(bal) - 1);
    if (mv) {
        const unsigned long long s = base + __popc(bal & ((1u << lane) - 1u));
        keys[s] = ((uint64_t)(gmax - gain[n]) << 32) | (uint64_t)(uint32_t)n;
        vals[s] = (uint32_t)n;
    }
}
// per move, after the h-edge kernels: the size track (refine.py:203-208),
// the aggregated inbound groups, and gain_seq = gain_iso + the h-edge terms
__device__ __forceinline__ void round_move(int64_t i, const int32_t *node, const int32_t *from, const int32_t *to,
                                           const int32_t *size, EvArgs ev, const int64_t *giso,
                                           const unsigned long long *gacc, int64_t *gseq) {
    gseq[i] = giso[i] + (int64_t)gacc[i];
    const int32_t s = size[node[i]], f = from[i], t = to[i];
    const int32_t a = ev.in_from[i], b = ev.in_to[i];
    unsigned long long k = atomicAdd(ev.count, (unsigned long long)(2 + (a != 0) + (b != 0)));
    auto put = [&](uint64_t track, int32_t p, int32_t d) {
        ev.key[k] = (track << (ev.pbits + ev.ibits)) | ((uint64_t)(uint32_t)p << ev.ibits) | (uint64_t)i;
        ev.val[k] = (uint32_t)d;
        k++;
    };
    put(0, f, -s);
    put(0, t, s);
    if (a) put(1, f, a);
    if (b) put(1, t, b);
}
// the round's results for the host in one record (one copy per round sync
// instead of five): selection (k, gain, large), movers, connectivity, the
// tiers' overflow counters
__global__ void k_round_summary(const long long *sres, const int32_t *ctr, const int32_t *sg, const int64_t *dM,
                                const unsigned long long *conn, long long *out) {
    pdl_entry();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    out[0] = sres[0];
    out[1] = sres[1];
    out[2] = sres[2];
    out[3] = dM ? (long long)*dM : 0;
    out[4] = conn ? (long long)*conn : 0;
    for (int i = 0; i < 4; i++) out[5 + i] = ctr[i];
    out[9] = sg[0];
    out[10] = sg[1];
}
__global__ void k_round_moves(const int64_t *dM, const int32_t *node, const int32_t *from, const int32_t *to,
                              const int32_t *size, EvArgs ev, const int64_t *giso, const unsigned long long *gacc,
                              int64_t *gseq, bool spec) {
    pdl_entry();
    const int64_t M = *dM;
    if (spec && M > kSpecCap) return;  // speculative launch, M too large
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x)
        round_move(i, node, from, to, size, ev, giso, gacc, gseq);
}


// ---------------------------------------------------------------------------
// Incremental refinement (RefineState, refine.cuh).
//
// Why a split during projection changes no other node's proposal: splitting
// cluster c (part P) into a, b raises pins[e, P] (and maybe pins_in[e, P]) by
// one on the h-edges holding both halves and changes nothing else.  A node
// n != a, b on such an h-edge with part P already counted both itself and c
// there (pins >= 2 before and after), so its saving term (pins == 1) is
// unchanged; for n outside P the set of parts on e and n's own count are
// unchanged, so present[] and saving are too.  Part sizes are sums over
// members and do not change.  Hence only a and b need new proposals, and the
// h-edges only need their counts refreshed.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void push_once(int32_t *flag, int32_t bits, int32_t x, int32_t *list, int32_t *count) {
    if (atomicOr(flag, bits) == 0) list[atomicAdd(count, 1)] = x;
}

// dirty h-edges: run lists recomputed for the current assignment.
// Split-only h-edges (bit 0) keep their parts and destination-part set, so
// only the counts change (no pinbound / connectivity terms).  H-edges dirtied
// by moves (bit 1) correct pinbound and connectivity by the difference and
// mark the pins whose proposal terms changed: a pin's proposal reads, per
// incident h-edge, the set of parts present (present[]) and whether its own
// part has exactly one pin there (saving).  So if the part set changed, every
// pin is dirty; otherwise only pins of a part whose "exactly one pin" state
// flipped (the movers themselves are marked by k_apply_inc).  pinbound
// deltas are aggregated per CTA in shared memory when K is small (the parts
// of a hub are hot addresses).
constexpr int RU_SMEM_K = 8192;
__global__ void k_runs_update(const int32_t *elist, const int32_t *ecount, int32_t *edirty, const int64_t *pin_off,
                              const int32_t *pin_dat, const int64_t *dst_off, const int32_t *dst_dat,
                              const int32_t *assign, const int64_t *wi, Runs r, unsigned long long *conn,
                              int64_t *pinbound, int32_t K, int32_t *ndirty, int32_t *nlist, int32_t *ncount,
                              int32_t *wide, int32_t *wide_count, unsigned long long *work) {
    pdl_entry();
    __shared__ int32_t sdelta[RU_SMEM_K];
    __shared__ int32_t s_oldp[8][128], s_oldc[8][128];
    const bool local = K <= RU_SMEM_K;
    if (local)
        for (int p = threadIdx.x; p < K; p += blockDim.x) sdelta[p] = 0;
    __syncthreads();
    const int lane = lane_id();
    const int64_t ne = *ecount;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    long long contrib = 0;
    for (int64_t idx = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id(); idx < ne; idx += nw) {
        const int32_t e = elist[idx];
        const int32_t flag = edirty[e];
        const bool moved = flag & 2;
        const int64_t plo = pin_off[e], lo = r.off[e];
        const int len = (int)(pin_off[e + 1] - plo);
        if (len > 128) {  // k_runs_update_wide takes it (a block per h-edge)
            if (lane_id() == 0) wide[atomicAdd(wide_count, 1)] = e;
            continue;
        }
        const int32_t old = r.len[e];
        // algorithmic bytes (profiling): the pin list and its parts (8 B per
        // pin), old and new runs (12 B each), offsets / flags / weight (32 B)
        if (work && lane == 0) atomicAdd(work, 8ull * len + 24ull * old + 32ull);
        int32_t *op = s_oldp[warp_id()], *oc = s_oldc[warp_id()];
        if (moved)
            for (int32_t j = lane; j < old; j += 32) {
                op[j] = r.pc[2 * (lo + j)];
                oc[j] = r.pc[2 * (lo + j) + 1];
                if (r.cin[lo + j] > 0) {
                    if (local)
                        atomicSub(&sdelta[r.pc[2 * (lo + j)]], 1);
                    else
                        atomicAdd((unsigned long long *)&pinbound[r.pc[2 * (lo + j)]], ~0ull);
                }
            }
        __syncwarp();
        int32_t lam;
        if (len <= 32)
            lam = warp_edge_runs<1>(e, plo, lo, len, pin_dat, dst_off, dst_dat, assign, r, nullptr);
        else if (len <= 64)
            lam = warp_edge_runs<2>(e, plo, lo, len, pin_dat, dst_off, dst_dat, assign, r, nullptr);
        else
            lam = warp_edge_runs<4>(e, plo, lo, len, pin_dat, dst_off, dst_dat, assign, r, nullptr);
        __syncwarp();
        if (moved) {
            for (int32_t j = lane; j < lam; j += 32)
                if (r.cin[lo + j] > 0) {
                    if (local)
                        atomicAdd(&sdelta[r.pc[2 * (lo + j)]], 1);
                    else
                        atomicAdd((unsigned long long *)&pinbound[r.pc[2 * (lo + j)]], 1ull);
                }
            bool same = lam == old;
            uint32_t flips[4] = {0u, 0u, 0u, 0u};
            if (same) {
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const int32_t j = q * 32 + lane;
                    bool f = false;
                    if (j < lam) {
                        same &= r.pc[2 * (lo + j)] == op[j];
                        f = (r.pc[2 * (lo + j) + 1] == 1) != (oc[j] == 1);
                    }
                    flips[q] = __ballot_sync(FULL_MASK, f);
                }
                same = __all_sync(FULL_MASK, same);
            }
            const bool any = flips[0] | flips[1] | flips[2] | flips[3];
            if (!same || any)
                for (int64_t j = plo + lane; j < plo + len; j += 32) {
                    const int32_t n = pin_dat[j];
                    bool mark = !same;
                    if (!mark) {
                        const int32_t k = run_find(r, lo, lam, assign[n]);
                        mark = (flips[k >> 5] >> (k & 31)) & 1u;
                    }
                    if (mark) push_once(&ndirty[n], 1, n, nlist, ncount);
                }
        }
        if (lane == 0) {
            r.len[e] = lam;
            edirty[e] = 0;
            if (moved) contrib += wi[e] * (long long)((lam > 0 ? lam - 1 : 0) - (old > 0 ? old - 1 : 0));
        }
    }
    if (lane == 0 && contrib) atomicAdd(conn, (unsigned long long)contrib);
    if (local) {
        __syncthreads();
        for (int p = threadIdx.x; p < K; p += blockDim.x)
            if (sdelta[p]) atomicAdd((unsigned long long *)&pinbound[p], (unsigned long long)(long long)sdelta[p]);
    }
}

// (item, incidence) pairs of a list of nodes, spread over the whole grid:
// item i takes `slices` CTAs, each striding over i's incident h-edges, so a
// hub's thousands of h-edges do not serialise on one warp
template <class NodeOf, class F>
__device__ __forceinline__ void grid_incidences(int64_t nitems, NodeOf node_of, const int64_t *inc_off,
                                                const int64_t *inc_end, const int32_t *inc_dat, F f) {
    if (nitems <= 0) return;
    const int64_t G = gridDim.x;
    const int64_t slices = G > nitems ? G / nitems : 1;  // CTAs per item
    for (int64_t t = blockIdx.x; t < nitems * slices; t += G) {
        const int64_t i = t / slices, sl = t - i * slices;
        const int32_t n = node_of(i);
        const int64_t hi = inc_end[n];
        for (int64_t j = inc_off[n] + sl * blockDim.x + threadIdx.x; j < hi; j += slices * blockDim.x)
            f(i, inc_dat[j]);
    }
}

// The same update for h-edges of more than 128 pin slots (power-law inputs):
// a CTA per h-edge sorts the pins' parts in shared memory (<= kMaxSegSort),
// derives the runs by a block scan of the heads, and applies the identical
// pinbound / connectivity differences and pin marking.
__global__ void __launch_bounds__(1024) k_runs_update_wide(const int32_t *wide, const int32_t *wide_count,
                                                           int32_t *edirty, const int64_t *pin_off,
                                                           const int32_t *pin_dat, const int64_t *dst_off,
                                                           const int32_t *dst_dat, const int32_t *assign,
                                                           const int64_t *wi, Runs r, unsigned long long *conn,
                                                           int64_t *pinbound, int32_t *ndirty, int32_t *nlist,
                                                           int32_t *ncount, uint8_t *gscr, int64_t gcap,
                                                           int smem_max) {
    pdl_entry();
    extern __shared__ unsigned long long smem_u64[];
    __shared__ int32_t s_wsum[32];
    __shared__ int s_same;
    const int t = threadIdx.x, lane = lane_id(), w = warp_id(), nwarp = blockDim.x >> 5;
    const int nwide = *wide_count;
    for (int q = blockIdx.x; q < nwide; q += gridDim.x) {
        const int32_t e = wide[q];
        const bool moved = edirty[e] & 2;
        const int64_t plo = pin_off[e], lo = r.off[e];
        const int len = (int)(pin_off[e + 1] - plo);
        const int32_t old = r.len[e];
        // working arrays: shared memory up to kMaxSegSort slots, else this
        // CTA's slice of the global scratch (h-edges of up to gcap pins)
        const bool huge = len > smem_max || old > smem_max;
        const int64_t cap = huge ? gcap : kMaxSegSort;
        uint8_t *wbuf = huge ? gscr + (int64_t)blockIdx.x * ((13 * gcap + 15) & ~(int64_t)15) : (uint8_t *)smem_u64;
        uint32_t *sv = (uint32_t *)wbuf;           // [cap] sorted parts
        int32_t *op = (int32_t *)(sv + cap);       // [cap] old parts
        int32_t *oc = op + cap;                    // [cap] old counts
        uint8_t *flip = (uint8_t *)(oc + cap);     // [cap] per new run
        for (int j = t; j < old; j += blockDim.x) {
            op[j] = r.pc[2 * (lo + j)];
            oc[j] = r.pc[2 * (lo + j) + 1];
            if (moved && r.cin[lo + j] > 0) atomicAdd((unsigned long long *)&pinbound[op[j]], ~0ull);
        }
        if (huge) {
            for (int j = t; j < len; j += blockDim.x) sv[j] = (uint32_t)assign[pin_dat[plo + j]];
            block_sort_asc_any<uint32_t>(sv, len);
        } else {
            const int np = next_pow2(len);
            for (int j = t; j < np; j += blockDim.x) sv[j] = j < len ? (uint32_t)assign[pin_dat[plo + j]] : 0xffffffffu;
            block_bitonic_sort32(sv, np);
        }
        // heads -> run slots by a block exclusive scan (one pass per 1024 slots)
        int base = 0;
        for (int c0 = 0; c0 < len; c0 += blockDim.x) {
            const int i = c0 + t;
            const bool head = i < len && (i == 0 || sv[i] != sv[i - 1]);
            const uint32_t bal = __ballot_sync(FULL_MASK, head);
            if (lane == 0) s_wsum[w] = __popc(bal);
            __syncthreads();
            int before = base, tot = 0;
            for (int j = 0; j < nwarp; j++) {
                if (j < w) before += s_wsum[j];
                tot += s_wsum[j];
            }
            if (head) {
                const int k = before + __popc(bal & ((1u << lane) - 1u));
                r.pc[2 * (lo + k)] = (int32_t)sv[i];
                r.cin[lo + k] = 0;
            }
            base += tot;
            __syncthreads();
        }
        const int lam = base;
        // run lengths from the sorted parts (binary searches; no in-place hazard)
        for (int k = t; k < lam; k += blockDim.x) {
            const uint32_t p = (uint32_t)r.pc[2 * (lo + k)];
            int a0 = 0, a1 = len;  // first index with sv >= p
            while (a0 < a1) {
                const int m = (a0 + a1) >> 1;
                if (sv[m] < p) a0 = m + 1; else a1 = m;
            }
            int b0 = a0, b1 = len;  // first index with sv > p
            while (b0 < b1) {
                const int m = (b0 + b1) >> 1;
                if (sv[m] <= p) b0 = m + 1; else b1 = m;
            }
            r.pc[2 * (lo + k) + 1] = b0 - a0;
        }
        __syncthreads();
        for (int64_t qd = dst_off[e] + t; qd < dst_off[e + 1]; qd += blockDim.x) {
            const int32_t k = run_find(r, lo, lam, assign[dst_dat[qd]]);
            atomicAdd(&r.cin[lo + k], 1);
        }
        __syncthreads();
        if (moved) {
            for (int k = t; k < lam; k += blockDim.x)
                if (r.cin[lo + k] > 0) atomicAdd((unsigned long long *)&pinbound[r.pc[2 * (lo + k)]], 1ull);
            if (t == 0) s_same = lam == old;
            __syncthreads();
            if (s_same)
                for (int k = t; k < lam; k += blockDim.x) {
                    if (r.pc[2 * (lo + k)] != op[k]) s_same = 0;
                    flip[k] = (r.pc[2 * (lo + k) + 1] == 1) != (oc[k] == 1);
                }
            __syncthreads();
            const bool same = s_same;
            for (int64_t j = plo + t; j < plo + len; j += blockDim.x) {
                const int32_t n = pin_dat[j];
                bool mark = !same;
                if (!mark) mark = flip[run_find(r, lo, lam, assign[n])];
                if (mark) push_once(&ndirty[n], 1, n, nlist, ncount);
            }
        }
        if (t == 0) {
            r.len[e] = lam;
            edirty[e] = 0;
            if (moved) {
                const long long d = wi[e] * (long long)((lam > 0 ? lam - 1 : 0) - (old > 0 ? old - 1 : 0));
                if (d) atomicAdd(conn, (unsigned long long)d);
            }
        }
        __syncthreads();
    }
}

// after moves: nodes whose proposal depends on a changed part size — the
// target no longer fits (a target that still fits stays the best eligible
// part), or a size-filtered positive-gain part shrank and may now fit
// (pflags bit 1 = shrank; fsens 3 = more filtered parts than recorded)
__global__ void k_mark_psize(int32_t N, const int32_t *target, const uint8_t *fsens, const int32_t *fpart,
                             const uint8_t *pflags, const int64_t *psizes, const int32_t *size, int64_t omega,
                             int32_t *ndirty, int32_t *nlist, int32_t *ncount) {
    pdl_entry();
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const int32_t t = target[n];
    bool d = t >= 0 && psizes[t] + size[n] > omega;
    const int f = fsens[n];
    if (f == 3)
        d = true;
    else if (f > 0)
        d |= (pflags[fpart[2 * n]] & 2) || (f == 2 && (pflags[fpart[2 * n + 1]] & 2));
    if (d) push_once(&ndirty[n], 1, (int32_t)n, nlist, ncount);
}

// the round's movers' h-edges (for the sequence gains and inbound events)
__global__ void k_mover_edges(const int64_t *dM, const int32_t *node, const int64_t *inc_off, const int64_t *inc_end,
                              const int32_t *inc_dat, int32_t *emflag, int32_t *mlist, int32_t *mcount, bool spec) {
    pdl_entry();
    if (spec && *dM > kSpecCap) return;  // speculative launch, M too large
    grid_incidences(*dM, [&](int64_t i) { return node[i]; }, inc_off, inc_end, inc_dat,
                    [&](int64_t, int32_t e) { push_once(&emflag[e], 1, e, mlist, mcount); });
}

// apply the first k moves (refine.py:250-254) and record what they dirty:
// part sizes, grown parts, the movers' h-edges; also clears the round's
// mover-edge flags
__global__ void k_apply_inc(int64_t k, const int32_t *node, const int32_t *from, const int32_t *to,
                            const int32_t *size, const int64_t *inc_off, const int64_t *inc_end,
                            const int32_t *inc_dat, int32_t *assign,
                            int64_t *psizes, uint8_t *pflags, int32_t *edirty, int32_t *elist, int32_t *ecount,
                            int32_t *emflag, const int32_t *mlist, const int32_t *mcount, int32_t *ndirty,
                            int32_t *nlist, int32_t *ncount) {
    pdl_entry();
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < k; i += nt) {
        const int32_t n = node[i];
        push_once(&ndirty[n], 1, n, nlist, ncount);
        const long long s = size[n];
        assign[n] = to[i];
        atomicAdd((unsigned long long *)&psizes[from[i]], (unsigned long long)(-s));
        atomicAdd((unsigned long long *)&psizes[to[i]], (unsigned long long)s);
        pflags[from[i]] = 2;
    }
    grid_incidences(k, [&](int64_t i) { return node[i]; }, inc_off, inc_end, inc_dat,
                    [&](int64_t, int32_t e) { push_once(&edirty[e], 2, e, elist, ecount); });
    const int64_t nm = *mcount;
    for (int64_t i = tid; i < nm; i += nt) emflag[mlist[i]] = 0;
}

__global__ void k_project(int32_t N, const int32_t *gamma, const int32_t *coarse, int32_t *fine) {
    pdl_entry();
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < N) fine[v] = coarse[gamma[v]];
}

__global__ void k_gamma_count(int32_t N, const int32_t *gamma, int32_t *ccount) {
    pdl_entry();
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n < N) atomicAdd(&ccount[gamma[n]], 1);
}

// projection of the carried state to the finer level; halves of split
// clusters are dirty (new nodes)
__global__ void k_project_state(int32_t N, const int32_t *gamma, const int32_t *ccount, const int32_t *assign_c,
                                const int32_t *target_c, const int64_t *gain_c, const uint8_t *fsens_c,
                                const int32_t *fpart_c, const int32_t *ndirty_c, int32_t *assign_f,
                                int32_t *target_f, int64_t *gain_f, uint8_t *fsens_f, int32_t *fpart_f,
                                int32_t *ndirty_f, int32_t *nlist, int32_t *ncount,
                                int32_t *splist, int32_t *spcount, int32_t *spfirst) {
    pdl_entry();
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const int32_t g = gamma[n];
    const bool split = ccount[g] == 2;
    assign_f[n] = assign_c[g];
    target_f[n] = target_c[g];
    gain_f[n] = gain_c[g];
    fsens_f[n] = fsens_c[g];
    fpart_f[2 * n] = fpart_c[2 * (int64_t)g];
    fpart_f[2 * n + 1] = fpart_c[2 * (int64_t)g + 1];
    const bool d = split || ndirty_c[g];
    ndirty_f[n] = d;
    if (d) nlist[atomicAdd(ncount, 1)] = (int32_t)n;
    if (split) {  // the second half of a cluster to arrive emits the pair
        const int32_t o = atomicExch(&spfirst[g], (int32_t)n);
        if (o >= 0) {
            const int i = atomicAdd(spcount, 1);
            splist[2 * i] = min(o, (int32_t)n);
            splist[2 * i + 1] = max(o, (int32_t)n);
        }
    }
}

// Run counts after a split: cluster c of part P splits into halves a, b.  An
// h-edge holding one half held c, so its counts stand; one holding both gains
// a pin of P (pins[e, P] + 1) and, when both halves are destinations, a
// destination pin (pins_in[e, P] + 1).  Parts, lambda and the distinct-inbound
// counts are unchanged.  A CTA per split: inc(a) n inc(b) and in(a) n in(b)
// by binary search of the shorter list in the longer.
__global__ void k_split_counts(const int32_t *splist, const int32_t *spcount, const int64_t *inc_off,
                               const int64_t *inc_end, const int32_t *inc_dat, const int64_t *in_off,
                               const int64_t *in_end, const int32_t *in_dat, const int32_t *assign, Runs r) {
    pdl_entry();
    const int n = *spcount;
    for (int t = blockIdx.x; t < n; t += gridDim.x) {
        const int32_t a = splist[2 * t], b = splist[2 * t + 1], P = assign[a];
#pragma unroll
        for (int fam = 0; fam < 2; fam++) {
            const int64_t *off = fam ? in_off : inc_off, *end = fam ? in_end : inc_end;
            const int32_t *dat = fam ? in_dat : inc_dat;
            const int64_t alo = off[a], na = end[a] - alo, blo = off[b], nb = end[b] - blo;
            const bool as = na <= nb;
            const int32_t *S = dat + (as ? alo : blo), *L = dat + (as ? blo : alo);
            const int64_t ns = as ? na : nb, nl = as ? nb : na;
            for (int64_t i = threadIdx.x; i < ns; i += blockDim.x) {
                const int32_t e = S[i];
                if (bsearch_dev(L, 0, nl, e) < 0) continue;
                const int64_t lo = r.off[e];
                const int32_t k = run_find(r, lo, r.len[e], P);
                atomicAdd(fam ? &r.cin[lo + k] : &r.pc[2 * (lo + k) + 1], 1);
            }
        }
    }
}

enum { CT_NLIST = 0, CT_ELIST = 1, CT_MLIST = 2, CT_SPLIST = 3, CT_WIDE = 4 };
}  // namespace

void refine_state_init(Ctx &c, RefineState &st, const DLevel &level0, int32_t K, bool incremental) {
    st = RefineState();
    st.inc = incremental;
    st.K = K;
    st.E = level0.E;
    st.ncap = std::max<int64_t>(1, shard_capacity(c.comm, level0.N));
    st.roff = level0.pin_off;
    st.rpc = c.alloc<int32_t>(2 * level0.U);
    st.rcin = c.alloc<int32_t>(level0.U);
    st.rlen = c.alloc<int32_t>(level0.E);
    st.psizes = c.alloc<int64_t>(K);
    st.pinbound = c.alloc<int64_t>(K);
    st.pflags = c.alloc<uint8_t>(K);
    st.conn = c.alloc<unsigned long long>(1);
    st.target = c.alloc<int32_t>(st.ncap);
    st.target2 = c.alloc<int32_t>(st.ncap);
    st.gain = c.alloc<int64_t>(st.ncap);
    st.gain2 = c.alloc<int64_t>(st.ncap);
    st.fsens = c.alloc<uint8_t>(st.ncap);
    st.fsens2 = c.alloc<uint8_t>(st.ncap);
    st.fpart = c.alloc<int32_t>(2 * st.ncap);
    st.fpart2 = c.alloc<int32_t>(2 * st.ncap);
    const int64_t n0 = std::max<int32_t>(1, level0.N), e0 = std::max<int32_t>(1, level0.E);
    st.ndirty = c.alloc<int32_t>(n0);
    st.ndirty2 = c.alloc<int32_t>(n0);
    st.nlist = c.alloc<int32_t>(n0);
    st.splist = c.alloc<int32_t>(n0);
    st.spfirst = c.alloc<int32_t>(n0);
    st.ccount = c.alloc<int32_t>(n0);
    st.edirty = c.alloc<int32_t>(e0);
    st.elist = c.alloc<int32_t>(e0);
    st.emflag = c.alloc<int32_t>(e0);
    st.mlist = c.alloc<int32_t>(e0);
    st.wide = c.alloc<int32_t>(e0);
    st.ctr = c.alloc<int32_t>(8);
    st.hub_max = hub_max_for(K);
    const int64_t hm = st.hub_max;
    st.hacc = c.alloc<long long>(hm * std::max(1, K));
    st.htot = c.alloc<long long>(2 * hm);
    st.hdone = c.alloc<int32_t>(hm);
    st.hlist = c.alloc<int32_t>(hm);
    st.hpref = c.alloc<int32_t>(hm + 1);
    c.zero(st.hacc, hm * std::max(1, K));
    c.zero(st.htot, 2 * hm);
    c.zero(st.hdone, hm);
    c.zero(st.pflags, K);
    c.zero(st.fsens, st.ncap);
    c.zero(st.ndirty, n0);
    c.zero(st.edirty, e0);
    c.zero(st.emflag, e0);
    c.zero(st.ctr, 8);
    c.zero(st.rlen, level0.E);
}

void refine_state_release(Ctx &c, RefineState &st) {
    for (void *p : {(void *)st.rpc, (void *)st.rcin, (void *)st.rlen, (void *)st.psizes,
                    (void *)st.pinbound, (void *)st.pflags, (void *)st.conn, (void *)st.target, (void *)st.target2,
                    (void *)st.gain, (void *)st.gain2, (void *)st.fsens, (void *)st.fsens2, (void *)st.fpart, (void *)st.fpart2, (void *)st.ndirty,
                    (void *)st.ndirty2, (void *)st.nlist, (void *)st.splist, (void *)st.spfirst, (void *)st.ccount, (void *)st.edirty,
                    (void *)st.elist, (void *)st.emflag, (void *)st.mlist, (void *)st.wide, (void *)st.ctr, (void *)st.hacc,
                    (void *)st.htot, (void *)st.hdone, (void *)st.hlist, (void *)st.hpref})
        c.free(p);
    st = RefineState();
}

void refine_project(Ctx &c, RefineState &st, const DLevel &fine, int32_t coarse_n, int32_t *&assign,
                    int32_t *&assign2) {
    const int32_t N = fine.N;
    // algorithmic bytes: gamma, the assignment and the carried proposal state per node
    KScope ks(c, "project", 40.0 * (double)N);
    if (N > 0) {
        if (st.inc) {
            c.zero(st.ccount, std::max<int32_t>(1, coarse_n));
            pdl_launch(k_gamma_count, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, fine.gamma, st.ccount);
            DHGP_LAUNCHED(c);
            c.zero(st.ctr + CT_NLIST, 1);
            c.zero(st.ctr + CT_SPLIST, 1);
            c.fill_bytes(st.spfirst, 0xff, std::max<int32_t>(1, coarse_n));
            pdl_launch(k_project_state, (unsigned)cdiv(N, 256), 256, 0, c.stream, 
                N, fine.gamma, st.ccount, assign, st.target, st.gain, st.fsens, st.fpart, st.ndirty, assign2,
                st.target2, st.gain2, st.fsens2, st.fpart2, st.ndirty2, st.nlist, st.ctr + CT_NLIST, st.splist,
                st.ctr + CT_SPLIST, st.spfirst);
            DHGP_LAUNCHED(c);
            Runs r;
            r.off = st.roff;
            r.pc = st.rpc;
            r.cin = st.rcin;
            r.len = st.rlen;
            pdl_launch(k_split_counts, 2 * c.num_sms, 256, 0, c.stream, st.splist, st.ctr + CT_SPLIST, fine.inc_off,
                       fine.inc_e(), fine.inc_dat, fine.in_off, fine.in_e(), fine.in_dat, assign2, r);
            DHGP_LAUNCHED(c);
            std::swap(st.target, st.target2);
            std::swap(st.gain, st.gain2);
            std::swap(st.fsens, st.fsens2);
            std::swap(st.fpart, st.fpart2);
            std::swap(st.ndirty, st.ndirty2);
        } else {
            pdl_launch(k_project, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, fine.gamma, assign, assign2);
            DHGP_LAUNCHED(c);
        }
    }
    std::swap(assign, assign2);
}

void refine_level(Ctx &c, const DLevel &L, const DWeights &W, RefineState &st, int32_t *assign, int32_t K,
                  int64_t omega, int64_t delta, int32_t max_rounds, int32_t level, std::vector<double> &conns,
                  const RoundObserver *obs, int32_t max_edge_pins) {
    static bool attr = false;
    if (!attr) {
        DHGP_CUDA(cudaFuncSetAttribute(k_propose_warp<unsigned>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       pr_smem<unsigned>()));
        DHGP_CUDA(cudaFuncSetAttribute(k_propose_warp<unsigned long long>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, pr_smem<unsigned long long>()));
        DHGP_CUDA(cudaFuncSetAttribute(k_propose_heavy<unsigned>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)ph_smem<unsigned>(ph_maxk<unsigned>())));
        DHGP_CUDA(cudaFuncSetAttribute(k_propose_heavy<unsigned long long>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)ph_smem<unsigned long long>(ph_maxk<unsigned long long>())));
        DHGP_CUDA(cudaFuncSetAttribute(k_select_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sel_smem()));
        DHGP_CUDA(cudaFuncSetAttribute(k_propose_mid<unsigned>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       pm_smem<unsigned>()));
        DHGP_CUDA(cudaFuncSetAttribute(k_propose_mid<unsigned long long>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       pm_smem<unsigned long long>()));
        attr = true;
    }
    const int32_t N = L.N;
    // ---- state (run lists at the level-0 pin offsets, part counters) -------
    Runs r;
    r.off = st.roff;
    r.pc = st.rpc;
    r.cin = st.rcin;
    r.len = st.rlen;
    int64_t *psizes = st.psizes, *pinbound = st.pinbound;
    int32_t *target = st.target;
    int64_t *gain = st.gain;
    unsigned long long *conn_d = st.conn;
    // ---- per-level buffers (capacities: N moves, 4N events) -----------------
    int32_t *tmp_parts = max_edge_pins > 128 ? c.alloc<int32_t>(L.U) : nullptr;
    uint8_t *flags = c.alloc<uint8_t>(N);
    int64_t *mpos = c.alloc<int64_t>((int64_t)N + 1);
    int32_t *pos = c.alloc<int32_t>(N);
    int32_t *ctr = c.alloc<int32_t>(4);
    int32_t *big = c.alloc<int32_t>(std::max<int64_t>(N, L.E));
    int32_t *big2 = c.alloc<int32_t>(N);
    uint64_t *mk = c.alloc<uint64_t>(N), *mkt = c.alloc<uint64_t>(N);
    uint32_t *mv = c.alloc<uint32_t>(N), *mvt = c.alloc<uint32_t>(N);
    int32_t *node = c.alloc<int32_t>(N), *from = c.alloc<int32_t>(N), *to = c.alloc<int32_t>(N);
    int64_t *giso = c.alloc<int64_t>(N), *gseq = c.alloc<int64_t>(N), *gseq_acc = c.alloc<int64_t>(N);
    int32_t *ev_from = c.alloc<int32_t>(N), *ev_to = c.alloc<int32_t>(N);
    int32_t *ectr = c.alloc<int32_t>(4);  // the event stage's overflow-list counters (ctr is the proposals')
    // sg_ctr [2], [3]: huge-list counts; [4]: the flat kernel's large h-edges (lg_list)
    int32_t *sg_big = c.alloc<int32_t>(L.E), *sg_ctr = c.alloc<int32_t>(8), *lg_list = c.alloc<int32_t>(L.E);
    // h-edges with more movers than shared memory holds (only possible when
    // an h-edge has more than 2048 pins): huge lists + 20 B/pin scratch per CTA
    const int mv_max = std::min(std::min(kSgBlockMax, kEvBlockMax), tiers().mv_block);
    const bool huge_movers = max_edge_pins > mv_max;
    int32_t *hv_sg = nullptr, *hv_ev = nullptr;
    uint8_t *mv_scr = nullptr;
    int mv_grid = 1;
    if (huge_movers) {
        hv_sg = c.alloc<int32_t>(L.E);
        hv_ev = c.alloc<int32_t>(L.E);
        mv_grid = (int)std::max<int64_t>(1, std::min<int64_t>(c.num_sms, (int64_t)(4ll << 30) /
                                                                           (20ll * max_edge_pins + 8)));
        mv_scr = c.alloc<uint8_t>((int64_t)mv_grid * ((20 * (int64_t)max_edge_pins + 15) & ~(int64_t)7));
    }
    const int64_t ecap = 4 * (int64_t)N + 4;  // 2 size + 2 aggregated inbound events per move
    uint64_t *ek = c.alloc<uint64_t>(ecap), *ekt = c.alloc<uint64_t>(ecap);
    uint32_t *evv = c.alloc<uint32_t>(ecap), *evt = c.alloc<uint32_t>(ecap);
    unsigned long long *ecount = c.alloc<unsigned long long>(1);
    long long *sres = c.alloc<long long>(4);
    long long *rsum = c.alloc<long long>(11);
    // dense global tier (K too large for shared memory): per-block rows of K
    // counters + touched lists, as many blocks as ~1 GiB allows (4 per SM max)
    const bool need_dense = K > ph_maxk<unsigned>() && K > std::min(4096, tiers().small_k);
    const int pb_blocks = need_dense ? (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c.num_sms * 4,
                                                                              (int64_t)(1ll << 30) /
                                                                                  std::max<int64_t>(1, 12ll * K)))
                                     : 1;
    long long *pdense = c.alloc<long long>((int64_t)pb_blocks * K);
    int32_t *ptouched = c.alloc<int32_t>((int64_t)pb_blocks * K);
    if (K > 0) {
        pdl_launch(k_fill_ll, (unsigned)cdiv((int64_t)pb_blocks * K, 256), 256, 0, c.stream, pdense, -1ll,
                                                                                   (int64_t)pb_blocks * K);
        DHGP_LAUNCHED(c);
    }
    const int gmax_bits = std::max(1, bitlen((uint64_t)W.wsum));
    const int pbits = std::max(1, bitlen((uint64_t)(K > 0 ? K - 1 : 0)));
    const int ibits_cap = std::max(1, bitlen((uint64_t)N));
    if (1 + ibits_cap + pbits > 64) throw Error{DHGP_ERR_UNSUPPORTED, "event key needs more than 64 bits"};
    int64_t *dM = mpos + N;
    static int g_ru = resident_grid(c, k_runs_update, 256, 0);
    static int g_me = resident_grid(c, k_mover_edges, 256, 0);
    static int g_ap = resident_grid(c, k_apply_inc, 256, 0);
    const bool wide_edges = max_edge_pins > 128;
    // h-edges beyond shared memory: 13 B per pin slot of global scratch per CTA
    uint8_t *huge_scr = nullptr;
    int huge_grid = c.num_sms;
    const int seg_smem = std::min<int>((int)kMaxSegSort, tiers().seg_smem);
    if (max_edge_pins > seg_smem) {
        huge_grid = (int)std::max<int64_t>(1, std::min<int64_t>(c.num_sms, (int64_t)(4ll << 30) /
                                                                             (13ll * max_edge_pins)));
        huge_scr = c.alloc<uint8_t>((int64_t)huge_grid * ((13 * (int64_t)max_edge_pins + 15) & ~(int64_t)15));
    }
    auto runs_update = [&](bool reset) {
        pdl_launch(k_runs_update, g_ru, 256, 0, c.stream, st.elist, st.ctr + CT_ELIST, st.edirty, L.pin_off, L.pin_dat,
                                                 L.dst_off, L.dst_dat, assign, W.wi, r, conn_d, pinbound, K, st.ndirty,
                                                 st.nlist, st.ctr + CT_NLIST, st.wide, st.ctr + CT_WIDE,
                                                 c.work_slot(Ctx::PW_RUNS_UPDATE));
        DHGP_LAUNCHED(c);
        if (wide_edges) {
            static bool wattr = false;
            if (!wattr) {
                DHGP_CUDA(cudaFuncSetAttribute(k_runs_update_wide, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)(13 * kMaxSegSort)));
                wattr = true;
            }
            pdl_launch(k_runs_update_wide, huge_grid, 1024, 13 * kMaxSegSort, c.stream,
                st.wide, st.ctr + CT_WIDE, st.edirty, L.pin_off, L.pin_dat, L.dst_off, L.dst_dat, assign, W.wi, r,
                conn_d, pinbound, st.ndirty, st.nlist, st.ctr + CT_NLIST, huge_scr, (int64_t)max_edge_pins,
                seg_smem);
            DHGP_LAUNCHED(c);
        }
        if (reset) zero_many(c, {{st.ctr + CT_ELIST, 4}, {st.ctr + CT_WIDE, 4}});
    };

    bool need_final = false;
    for (int32_t rnd = 0; rnd < max_rounds; rnd++) {
        const bool full = !st.inc || st.fresh;
        // the round's counters and, for a speculative tail, its per-move
        // accumulators start at zero: one fill at the round's start (the mover
        // count, the mover-edge list, the h-edge terms, the event lists)
        const bool spec_round = gmax_bits <= 32 && tiers().speculate;
        const int64_t mc0 = spec_round ? std::min<int64_t>(kSpecCap, N) : 0;
        const std::initializer_list<ZeroSpan> round_zero = {
            {dM, 8}, {st.ctr + CT_MLIST, 4}, {sg_ctr, 32}, {ectr, 16}, {ecount, 8}, {gseq_acc, 8 * mc0},
            {ev_from, 4 * mc0}, {ev_to, 4 * mc0}};
        if (full) {
            // --- A11/A12/A16 + A13 over everything ----------------------------
            build_runs(c, L, W, assign, r, tmp_parts, pinbound, K, conn_d, max_edge_pins);
            zero_many(c, round_zero, {{psizes, 8 * (int64_t)K}, {ctr, 16}});
            if (N > 0) {
                pdl_launch(k_part_sizes, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, assign, L.size, psizes);
                DHGP_LAUNCHED(c);
            }
        } else {
            // --- only what the last moves / the projection touched -----------
            KScope ks(c, "runs_update");
            runs_update(false);
            const bool mp = st.moved && N > 0;
            if (mp) {
                pdl_launch(k_mark_psize, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, target, st.fsens, st.fpart, st.pflags,
                                                                           psizes, L.size, omega, st.ndirty,
                                                                           st.nlist, st.ctr + CT_NLIST);
                DHGP_LAUNCHED(c);
            }
            // the dirty-edge list is consumed, the shrink flags too; the
            // propose counters start at zero
            zero_many(c, round_zero,
                      {{st.ctr + CT_ELIST, 4}, {st.pflags, mp ? (int64_t)K : 0}, {ctr, 16}, {st.ctr + CT_WIDE, 4}});
        }
        st.moved = false;
        // --- A14 propose (warp tier + block tier, no host sync) -------------
        {
            KScope ks(c, "propose", 0.0, N);
            unsigned long long *work = nullptr;
            if (c.profiling) {
                work = c.alloc<unsigned long long>(1);
                c.zero(work, 1);
            }
            ProposeArgs a{N, K, L.inc_off, L.inc_dat, W.wi, r, assign, psizes, L.size, omega,
                          target, gain, ctr, big, ctr + 1, big2, ctr + 2, tiers(), 0, N};
            a.inc_end = L.inc_e();
            a.fsens = st.fsens;
            a.fpart = st.fpart;
            a.work = work;
            constexpr int kSmallK = 4096;
            const bool small_k = K <= std::min(kSmallK, tiers().small_k);
            if (small_k) {
                a.hub_list = st.hlist;
                a.hub_count = ctr + 3;
                a.hub_max = st.hub_max;
                a.hub_pref = st.hpref;
            }
            if (!full) {
                a.list = st.nlist;
                a.list_count = st.ctr + CT_NLIST;
                a.ndirty = st.ndirty;
            }
            const Shard sh = shard_of(c.comm, N);
            a.lo = (int32_t)sh.lo;
            a.hi = (int32_t)sh.hi;
            const int64_t nmine = full ? std::max<int64_t>(1, sh.hi - sh.lo) : (int64_t)1 << 40;
            if (trace_enabled() && !full) {  // diagnostics: dirty-set sizes
                int32_t hc[8];
                c.d2h(hc, st.ctr, 8);
                c.sync();
                fprintf(stderr, "dirty level %d round %d N %d nodes %d\n", level, rnd, N, hc[CT_NLIST]);
            }
            if (N > 0) {
                const bool narrow = W.wsum < (1ll << 32);
                if (narrow) {
                    static int g32 = resident_grid(c, k_propose_warp<unsigned>, PR_WARPS * 32, pr_smem<unsigned>());
                    int blocks = (int)std::min<int64_t>(cdiv(nmine, PR_WARPS), g32);
                    pdl_launch(k_propose_warp<unsigned>, blocks, PR_WARPS * 32, pr_smem<unsigned>(), c.stream, a);
                } else {
                    static int g64 = resident_grid(c, k_propose_warp<unsigned long long>, PR_WARPS * 32,
                                                   pr_smem<unsigned long long>());
                    int blocks = (int)std::min<int64_t>(cdiv(nmine, PR_WARPS), g64);
                    pdl_launch(k_propose_warp<unsigned long long>, blocks, PR_WARPS * 32, pr_smem<unsigned long long>(), c.stream, a);
                }
                DHGP_LAUNCHED(c);
                KScope kh(c, "propose_heavy");
                if (small_k) {
                    pdl_launch(k_hub_prefix, 1, 1024, 0, c.stream, st.hlist, ctr + 3, st.hub_max, L.inc_off, L.inc_e(),
                               st.hpref);
                    DHGP_LAUNCHED(c);
                    if (narrow) {
                        static int h32 = resident_grid(c, k_propose_hub<unsigned>, 256, 4 * kSmallK);
                        pdl_launch(k_propose_hub<unsigned>, h32, 256, 4 * K, c.stream, a, st.hacc, st.htot, st.hdone);
                    } else {
                        static int h64 = resident_grid(c, k_propose_hub<unsigned long long>, 256, 8 * kSmallK);
                        pdl_launch(k_propose_hub<unsigned long long>, h64, 256, 8 * K, c.stream, a, st.hacc, st.htot, st.hdone);
                    }
                    DHGP_LAUNCHED(c);
                    // few parts: the escalated nodes go straight to dense shared
                    // arrays over the parts (no hashing), 256 threads per node
                    ProposeArgs b = a;
                    b.dense_list = big;
                    b.dense_count = ctr + 1;
                    if (narrow) {
                        static int s32 = resident_grid(c, k_propose_heavy<unsigned, 256>, 256,
                                                       ph_smem<unsigned>(kSmallK));
                        pdl_launch(k_propose_heavy<unsigned, 256>, s32, 256, ph_smem<unsigned>(K), c.stream, b);
                    } else {
                        static int s64 = resident_grid(c, k_propose_heavy<unsigned long long, 256>, 256,
                                                       ph_smem<unsigned long long>(kSmallK));
                        pdl_launch(k_propose_heavy<unsigned long long, 256>, s64, 256, ph_smem<unsigned long long>(K), c.stream, b);
                    }
                    DHGP_LAUNCHED(c);
                } else {
                    // medium tier: reads the escalation count on device, exits when zero
                    if (narrow) {
                        static int m32 = resident_grid(c, k_propose_mid<unsigned>, PM_THREADS, pm_smem<unsigned>());
                        pdl_launch(k_propose_mid<unsigned>, m32, PM_THREADS, pm_smem<unsigned>(), c.stream, a);
                    } else {
                        static int m64 = resident_grid(c, k_propose_mid<unsigned long long>, PM_THREADS,
                                                       pm_smem<unsigned long long>());
                        pdl_launch(k_propose_mid<unsigned long long>, m64, PM_THREADS, pm_smem<unsigned long long>(), c.stream, a);
                    }
                    DHGP_LAUNCHED(c);
                    if (narrow && K <= ph_maxk<unsigned>()) {
                        pdl_launch(k_propose_heavy<unsigned>, c.num_sms, PH_THREADS, ph_smem<unsigned>(K), c.stream, a);
                    } else if (!narrow && K <= ph_maxk<unsigned long long>()) {
                        pdl_launch(k_propose_heavy<unsigned long long>, c.num_sms, PH_THREADS, ph_smem<unsigned long long>(K), c.stream, a);
                    } else {
                        pdl_launch(k_propose_block, pb_blocks, PB_THREADS, 0, c.stream, a, pdense, ptouched);
                    }
                    DHGP_LAUNCHED(c);
                }
            }
            if (work) {  // measured algorithmic bytes: lists read (+ per node assign/size/outputs, full mode)
                ks.stop();
                unsigned long long h = 0;
                c.d2h(&h, work, 1);
                c.sync();
                ks.set_bytes((double)h + 24.0 * (full ? (double)N : 0.0));
                c.free(work);
            }
            if (trace_enabled()) {
                int32_t hc[4];
                c.d2h(hc, ctr, 4);
                c.sync();
                fprintf(stderr, "tiers level %d round %d big %d dense %d hubs %d\n", level, rnd, hc[1], hc[2], hc[3]);
            }
            if (sh.on) {  // complete (target, gain, fsens) from the other ranks' node ranges
                allgather(c, c.comm, target, sizeof(int32_t), sh.chunk);
                allgather(c, c.comm, gain, sizeof(int64_t), sh.chunk);
                allgather(c, c.comm, st.fsens, sizeof(uint8_t), sh.chunk);
                allgather(c, c.comm, st.fpart, 2 * sizeof(int32_t), sh.chunk);
            }
        }
        st.fresh = false;
        // --- sequence: movers by (gain desc, node asc) (refine.py:108-110) --
        // packed (key, node) when the key fits 32 bits: an unordered atomic
        // compaction then sorts correctly; else the ordered flags + scan
        const bool packed = gmax_bits <= 32;
        // algorithmic bytes: target, gain and position per node
        KScope km(c, "movers", 16.0 * (double)N);
        if (packed) {
            if (N > 0) {
                // (the dirty-node list was consumed by the proposals: its count
                // is reset here, incremental rounds only)
                pdl_launch(k_mover_compact, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, target, gain, W.wsum, mk, mv, pos,
                                                                             (unsigned long long *)dM,
                                                                             full ? nullptr : st.ctr + CT_NLIST);
                DHGP_LAUNCHED(c);
            }
        } else {
            if (N > 0) {
                pdl_launch(k_mover_flags, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, target, flags,
                           full ? nullptr : st.ctr + CT_NLIST);
                DHGP_LAUNCHED(c);
            }
            scan_excl<uint8_t>(c, flags, mpos, N);
        }
        km.close();
        // ---- the round's tail (sort, moves, A15, A17 select) is launched
        // before M is on the host: speculatively for up to kSpecCap movers,
        // with M read on device (the kernels are no-ops beyond that, and the
        // host then relaunches it for the real M).  One host sync per round
        // reads M, the connectivity and the selection together.  Unpacked
        // sequence keys need the ordered scan, hence M first.
        const bool spec = packed && tiers().speculate;
        int64_t M = 0;
        unsigned long long conn_h = 0;
        if (!spec) {
            c.d2h(&M, dM, 1);
            c.d2h(&conn_h, conn_d, 1);
            c.sync();
            conns.push_back((double)(int64_t)conn_h * W.unit);
            need_final = false;
            if (M == 0) break;
        }
        int ibits = 1;
        EvArgs ev{};
        int64_t *dlt = nullptr, *act_ex = nullptr, *cum = nullptr;
        auto launch_tail = [&](bool sp, int64_t Mh) {
            // capacity of this launch (the per-move buffers hold N entries)
            const int64_t Mc = sp ? std::min<int64_t>(kSpecCap, N) : Mh;
            if (packed) {
                if (sp)
                    small_sort_packed(c, mk, mv, 0, dM);
                else if (Mh <= kSmallSort)
                    small_sort_packed(c, mk, mv, Mh);
                else
                    (Mh <= kMergeSortMax) ? merge_sort_pairs(c, mk, mv, mkt, mvt, Mh)
                                          : radix_sort_pairs(c, mk, mv, mkt, mvt, Mh, nullptr, gmax_bits + 32);
            } else {
                if (N > 0) {
                    pdl_launch(k_mover_keys, (unsigned)cdiv(N, 256), 256, 0, c.stream, N, flags, mpos, gain, W.wsum, mk, mv);
                    DHGP_LAUNCHED(c);
                }
                if (Mh <= kSmallSort)
                    small_sort_pairs(c, mk, mv, Mh);  // vals (nodes) are distinct and ascend: stable
                else
                    (Mh <= kMergeSortMax) ? merge_sort_pairs(c, mk, mv, mkt, mvt, Mh)
                                          : radix_sort_pairs(c, mk, mv, mkt, mvt, Mh, nullptr, gmax_bits);
                fill_i32(c, pos, -1, N);
            }
            pdl_launch(k_build_moves_dn, (unsigned)std::max<int64_t>(1, cdiv(Mc, 256)), 256, 0, c.stream, 
                dM, mv, assign, target, gain, node, from, to, giso, pos, sp);
            DHGP_LAUNCHED(c);
            // h-edges holding a mover: the only ones with sequence-gain terms or
            // inbound events (incremental mode; the full mode scans every h-edge)
            const int32_t *elist = nullptr, *elist_n = nullptr;
            if (st.inc) {
                pdl_launch(k_mover_edges, g_me, 256, 0, c.stream, dM, node, L.inc_off, L.inc_e(), L.inc_dat, st.emflag, st.mlist,
                                                          st.ctr + CT_MLIST, sp);
                DHGP_LAUNCHED(c);
                elist = st.mlist;
                elist_n = st.ctr + CT_MLIST;
            }
            // --- A15 sequence gains + A17 events (replicated: O(sum |e|), no exchange)
            ibits = std::max(1, bitlen((uint64_t)Mc));
            ev = EvArgs{ibits, pbits, ek, evv, ecount};
            ev.in_from = ev_from;
            ev.in_to = ev_to;
            {
                KScope ks(c, "seq_gains", 0.0);
                unsigned long long *gacc = (unsigned long long *)gseq_acc;
                // (a speculative tail's accumulators were zeroed at the round's start)
                if (!sp) zero_many(c, {{gacc, 8 * Mc}, {sg_ctr, 32}, {ectr, 16}, {ev_from, 4 * Mc}, {ev_to, 4 * Mc},
                                       {ecount, 8}});
                // sharding: each rank takes the mover h-edges of its h-edge id
                // range; a move's terms are then summed across ranks
                const Shard esh = shard_of(c.comm, L.E);
                if (L.E > 0) {
                    {
                        // the flat kernel takes rounds of many mover h-edges
                        // (small ones in warp chunks; the rest listed), the
                        // per-edge kernel the listed ones, or all of a small round
                        const int64_t fe_min = tiers().fe_min;
                        static int g_fe = resident_grid(c, k_round_edges_flat, FE_WARPS * 32, 0);
                        const unsigned gre =
                            (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(L.E, 32 * FE_WARPS), g_fe));
                        pdl_launch(k_round_edges_flat, gre, FE_WARPS * 32, 0, c.stream, L.E, elist, elist_n,
                                   L.pin_off, L.pin_dat, L.dst_off, L.dst_dat, W.wi, r, pos, from, to, gacc, ev,
                                   sg_big, sg_ctr, big, ectr, tiers().edge_movers, sp ? dM : nullptr,
                                   c.work_slot(Ctx::PW_SEQ_GAINS), esh.lo, esh.hi, lg_list, sg_ctr + 4, fe_min);
                        DHGP_LAUNCHED(c);
                        static int g_re = resident_grid(c, k_round_edges, 256, 0);
                        const unsigned gpe = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(L.E, 8), g_re));
                        pdl_launch(k_round_edges, gpe, 256, 0, c.stream, L.E, elist, elist_n, L.pin_off, L.pin_dat,
                                   L.dst_off, L.dst_dat, W.wi, r, pos, from, to, gacc, ev, sg_big, sg_ctr, big, ectr,
                                   tiers().edge_movers, sp ? dM : nullptr, c.work_slot(Ctx::PW_SEQ_GAINS), esh.lo,
                                   esh.hi, lg_list, sg_ctr + 4, fe_min);
                    }
                    DHGP_LAUNCHED(c);
                    pdl_launch(k_seq_gains_edge_block, c.num_sms, 256, 0, c.stream, L.pin_off, L.pin_dat, W.wi, r, pos, from,
                                                                             to, gacc, sg_big, sg_ctr, hv_sg, sg_ctr + 2,
                                                                             mv_max);
                    DHGP_LAUNCHED(c);
                    pdl_launch(k_inbound_events_block, c.num_sms, 256, 0, c.stream, L.dst_off, L.dst_dat, r, pos, from, to,
                                                                             ev, big, ectr, hv_ev, sg_ctr + 3, mv_max);
                    DHGP_LAUNCHED(c);
                    if (huge_movers) {  // exit at once when the huge lists are empty
                        pdl_launch(k_edge_movers_huge, mv_grid, 1024, 0, c.stream, 0, L.pin_off, L.pin_dat, W.wi, r,
                                   pos, from, to, gacc, ev, hv_sg, sg_ctr + 2, mv_scr, (int64_t)max_edge_pins);
                        DHGP_LAUNCHED(c);
                        pdl_launch(k_edge_movers_huge, mv_grid, 1024, 0, c.stream, 1, L.dst_off, L.dst_dat, W.wi, r,
                                   pos, from, to, gacc, ev, hv_ev, sg_ctr + 3, mv_scr, (int64_t)max_edge_pins);
                        DHGP_LAUNCHED(c);
                    }
                }
                if (esh.on) {
                    allreduce_sum_i64(c, c.comm, (long long *)gacc, Mc);
                    allreduce_sum_i32(c, c.comm, ev_from, Mc);
                    allreduce_sum_i32(c, c.comm, ev_to, Mc);
                }
                pdl_launch(k_round_moves, (unsigned)std::max<int64_t>(1, cdiv(Mc, 256)), 256, 0, c.stream, 
                    dM, node, from, to, L.size, ev, giso, gacc, gseq, sp);
                DHGP_LAUNCHED(c);
            }
            // --- A17 select: one CTA for small rounds, T and M read on device
            dlt = c.alloc<int64_t>(Mc + 1);
            act_ex = c.alloc<int64_t>(Mc + 2);
            cum = c.alloc<int64_t>(Mc + 1);
            KScope ks(c, "select", 0.0, N);
            const bool packed_ev = 1 + ibits + pbits <= 32;
            pdl_launch(k_select_small, 1, SEL_THREADS, sel_smem(), c.stream, ecount, dM, ek, evv, gseq, psizes, pinbound,
                                                                    omega, delta, ibits, pbits, act_ex, sres,
                                                                    packed_ev, c.work_slot(Ctx::PW_SELECT));
            DHGP_LAUNCHED(c);
        };
        auto free_tail = [&]() {
            c.free(dlt);
            c.free(act_ex);
            c.free(cum);
            dlt = act_ex = cum = nullptr;
        };
        launch_tail(spec, M);
        int64_t kbest = 0, total_gain = 0;
        {
            // ---- the round's sync: the selected prefix (or "too large"), error flags
            long long hr[3];
            int32_t hc[4];
            int32_t hs[2];
            long long sum[11];
            auto read_round = [&](bool with_m) {
                pdl_launch(k_round_summary, 1, 32, 0, c.stream, (const long long *)sres, (const int32_t *)ctr,
                           (const int32_t *)sg_ctr, with_m ? (const int64_t *)dM : nullptr,
                           with_m ? (const unsigned long long *)conn_d : nullptr, rsum);
                DHGP_LAUNCHED(c);
                c.d2h(sum, rsum, 11);
                c.sync();
                for (int i = 0; i < 3; i++) hr[i] = sum[i];
                if (with_m) {
                    M = sum[3];
                    conn_h = (unsigned long long)sum[4];
                }
                for (int i = 0; i < 4; i++) hc[i] = (int32_t)sum[5 + i];
                hs[0] = (int32_t)sum[9];
                hs[1] = (int32_t)sum[10];
            };
            read_round(spec);
            if (spec) {
                conns.push_back((double)(int64_t)conn_h * W.unit);
                need_final = false;
                if (M == 0) {
                    free_tail();
                    break;
                }
                if (M > kSpecCap) {  // the speculative launch did nothing: relaunch for the real M
                    free_tail();
                    launch_tail(false, M);
                    read_round(false);
                }
            }
            kbest = hr[0];
            total_gain = hr[1];
            if (trace_enabled()) {  // diagnostics: movers and the h-edges holding one
                int32_t hm[CT_MLIST + 1];
                c.d2h(hm, st.ctr, CT_MLIST + 1);
                c.sync();
                fprintf(stderr, "round level %d N %d E %d M %lld elist %d\n", level, N, L.E, (long long)M,
                        st.inc ? hm[CT_MLIST] : L.E);
            }
            if (hr[2]) {  // a large round: the multi-kernel path
                unsigned long long T = 0;
                c.d2h(&T, ecount, 1);
                c.sync();
                if (trace_enabled()) fprintf(stderr, "largeselect level %d M %lld T %llu\n", level, (long long)M, T);
                if ((int64_t)T <= kSmallSort)
                    small_sort_pairs(c, ek, evv, (int64_t)T);  // equal keys only need grouping
                else
                    ((int64_t)T <= kMergeSortMax)
                        ? merge_sort_pairs(c, ek, evv, ekt, evt, (int64_t)T)
                        : radix_sort_pairs(c, ek, evv, ekt, evt, (int64_t)T, nullptr, 1 + ibits + pbits);
                int64_t *gs = c.alloc<int64_t>(T), *ss = c.alloc<int64_t>(T), *dv = c.alloc<int64_t>(T);
                int64_t *ex = c.alloc<int64_t>(T + 1), *gst = c.alloc<int64_t>(T), *sst = c.alloc<int64_t>(T);
                c.zero(dlt, M + 1);
                if (T > 0) {
                    pdl_launch(k_ev_prep, (unsigned)cdiv(T, 256), 256, 0, c.stream, (int64_t)T, ek, evv, ibits, gs, ss, dv);
                    DHGP_LAUNCHED(c);
                    scan_excl<int64_t>(c, dv, ex, T);
                    scan_incl_max(c, gs, gst, T);
                    scan_incl_max(c, ss, sst, T);
                    pdl_launch(k_ev_toggle, (unsigned)cdiv(T, 256), 256, 0, c.stream, (int64_t)T, ek, ex, gst, sst, ibits,
                                                                              pbits, psizes, pinbound, omega, delta,
                                                                              dlt);
                    DHGP_LAUNCHED(c);
                }
                scan_excl<int64_t>(c, dlt, act_ex, M + 1);  // act_ex[j+1] = active[j]
                scan_excl<int64_t>(c, gseq, cum, M);        // cum[j] = sum of the first j gains
                const int nb = (int)std::min<int64_t>(cdiv(M + 1, 256), 256);
                long long *bv = c.alloc<long long>(nb), *bk = c.alloc<long long>(nb), *res = c.alloc<long long>(2);
                pdl_launch(k_best_prefix_partial, nb, 256, 0, c.stream, M + 1, act_ex, cum, bv, bk);
                DHGP_LAUNCHED(c);
                pdl_launch(k_best_prefix_final, 1, 32, 0, c.stream, nb, bv, bk, res);
                DHGP_LAUNCHED(c);
                long long h2[2];
                c.d2h(h2, res, 2);
                c.sync();
                kbest = h2[0];
                total_gain = h2[1];
                c.free(bv);
                c.free(bk);
                c.free(res);
                for (void *q : {(void *)gs, (void *)ss, (void *)dv, (void *)ex, (void *)gst, (void *)sst}) c.free(q);
            }
        }
        if (obs && *obs) {
            RoundRecord rec;
            rec.level = level;
            rec.round = rnd;
            rec.num_parts = K;
            rec.k = (int32_t)kbest;
            rec.total_gain = (double)total_gain * W.unit;
            rec.assign.resize(N);
            rec.node.resize(M);
            rec.from.resize(M);
            rec.to.resize(M);
            std::vector<int64_t> gi(M), gs(M), ae(M + 2);
            c.d2h(rec.assign.data(), assign, N);
            c.d2h(rec.node.data(), node, M);
            c.d2h(rec.from.data(), from, M);
            c.d2h(rec.to.data(), to, M);
            c.d2h(gi.data(), giso, M);
            c.d2h(gs.data(), gseq, M);
            c.d2h(ae.data(), act_ex, M + 2);
            c.sync();
            rec.gain_iso.resize(M);
            rec.gain_seq.resize(M);
            for (int64_t i = 0; i < M; i++) {
                rec.gain_iso[i] = (double)gi[i] * W.unit;
                rec.gain_seq[i] = (double)gs[i] * W.unit;
            }
            rec.active.assign(ae.begin() + 1, ae.begin() + 2 + M);
            (*obs)(rec);
        }
        // algorithmic bytes (lower bound): the applied moves (node, from, to, size) and their assignment
        KScope kap(c, "apply", 24.0 * (double)kbest);
        if (st.inc) {
            // apply + record the dirt; clears the mover-edge flags either way
            pdl_launch(k_apply_inc, g_ap, 256, 0, c.stream, kbest, node, from, to, L.size, L.inc_off, L.inc_e(), L.inc_dat, assign,
                                                    psizes, st.pflags, st.edirty, st.elist, st.ctr + CT_ELIST,
                                                    st.emflag, st.mlist, st.ctr + CT_MLIST, st.ndirty, st.nlist,
                                                    st.ctr + CT_NLIST);
            DHGP_LAUNCHED(c);
            if (kbest > 0) st.moved = true;
        } else if (kbest > 0) {
            pdl_launch(k_apply, (unsigned)cdiv(kbest, 256), 256, 0, c.stream, kbest, node, to, assign);
            DHGP_LAUNCHED(c);
        }
        kap.close();
        c.free(dlt);
        c.free(act_ex);
        c.free(cum);
        if (kbest == 0) break;
        need_final = true;
    }
    if (need_final) {
        // connectivity after the last applied round
        if (st.inc) {
            runs_update(true);
            unsigned long long h = 0;
            c.d2h(&h, conn_d, 1);
            c.sync();
            conns.push_back((double)(int64_t)h * W.unit);
        } else {
            double v;
            evaluate_assign(c, L, W, assign, K, nullptr, nullptr, &v);
            conns.push_back(v);
        }
    }
    for (void *p : {(void *)tmp_parts, (void *)flags, (void *)mpos, (void *)pos, (void *)ctr, (void *)big,
                    (void *)big2, (void *)mk, (void *)mkt, (void *)mv, (void *)mvt, (void *)node, (void *)from,
                    (void *)to, (void *)giso, (void *)gseq, (void *)gseq_acc, (void *)ev_from, (void *)ev_to,
                    (void *)sg_big, (void *)sg_ctr, (void *)lg_list,
                    (void *)ek, (void *)ekt, (void *)evv, (void *)evt, (void *)ecount, (void *)ectr, (void *)sres, (void *)rsum, (void *)pdense,
                    (void *)ptouched, (void *)huge_scr, (void *)hv_sg,
                    (void *)hv_ev, (void *)mv_scr})
        c.free(p);
}

void evaluate_assign(Ctx &c, const DLevel &L, const DWeights &W, const int32_t *assign, int32_t K,
                     int64_t *d_sizes, int64_t *d_inbound, double *h_conn) {
    Runs r;
    r.off = L.pin_off;
    r.pc = c.alloc<int32_t>(2 * L.U);
    r.cin = c.alloc<int32_t>(L.U);
    r.len = c.alloc<int32_t>(L.E);
    int32_t *tmp = c.alloc<int32_t>(L.U);
    seg_sort(c, L.E, L.pin_off, L.pin_dat, assign, tmp);
    unsigned long long *conn = c.alloc<unsigned long long>(1);
    c.zero(conn, 1);
    if (d_inbound) c.zero(d_inbound, K);
    if (L.E > 0) {
        pdl_launch(k_edge_runs, (unsigned)cdiv(L.E, 256), 256, 0, c.stream, L.E, L.pin_off, tmp, L.dst_off, L.dst_dat, assign,
                                                                   W.wi, r, conn, d_inbound);
        DHGP_LAUNCHED(c);
    }
    if (d_sizes) {
        c.zero(d_sizes, K);
        if (L.N > 0) {
            pdl_launch(k_part_sizes, (unsigned)cdiv(L.N, 256), 256, 0, c.stream, L.N, assign, L.size, d_sizes);
            DHGP_LAUNCHED(c);
        }
    }
    if (h_conn) {
        unsigned long long h = 0;
        c.d2h(&h, conn, 1);
        c.sync();
        *h_conn = (double)(int64_t)h * W.unit;
    }
    c.free(conn);
    c.free(r.pc);
    c.free(r.cin);
    c.free(r.len);
    c.free(tmp);
}

}  // namespace dhgp
