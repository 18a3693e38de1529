// prims.cu — scans, radix sort, per-segment sorts, sorted-set merges.
#include <climits>

#include <cmath>

#include "prims.cuh"

namespace dhgp {

// ===========================================================================
// exclusive scan (single pass, decoupled look-back; tile = 256 threads x 16 items)
// ===========================================================================
namespace {
constexpr int SC_BT = 256;
constexpr int SC_IPT = 16;
constexpr int SC_TILE = SC_BT * SC_IPT;

// One tile, warp-striped: warp w owns elements [w*512, (w+1)*512) of the
// tile, lane l holds element r*32 + l of it in v[r] (coalesced loads); the
// scan runs over registers with shuffles (no shared-memory transpose).
// v[] becomes the exclusive prefix within the tile; returns the tile total.
template <class T>
__device__ __forceinline__ int64_t tile_excl_scan(const T *in, int64_t n, int64_t base, int64_t (&v)[SC_IPT],
                                                  int64_t *sh) {
    const int lane = lane_id(), w = warp_id();
    const int64_t wb = base + (int64_t)w * (SC_IPT * 32);
#pragma unroll
    for (int r = 0; r < SC_IPT; r++) {
        const int64_t idx = wb + r * 32 + lane;
        v[r] = idx < n ? (int64_t)in[idx] : 0;
    }
    int64_t carry = 0;
#pragma unroll
    for (int r = 0; r < SC_IPT; r++) {
        const int64_t x = warp_incl_scan(v[r]);
        const int64_t e = x - v[r] + carry;
        carry += __shfl_sync(FULL_MASK, x, 31);
        v[r] = e;
    }
    if (lane == 0) sh[w] = carry;
    __syncthreads();
    int64_t before = 0, tot = 0;
#pragma unroll
    for (int j = 0; j < SC_BT / 32; j++) {
        const int64_t t = sh[j];
        if (j < w) before += t;
        tot += t;
    }
#pragma unroll
    for (int r = 0; r < SC_IPT; r++) v[r] += before;
    return tot;
}
__device__ __forceinline__ void tile_store(int64_t *out, int64_t n, int64_t base, const int64_t (&v)[SC_IPT],
                                           int64_t add) {
    const int lane = lane_id(), w = warp_id();
    const int64_t wb = base + (int64_t)w * (SC_IPT * 32);
#pragma unroll
    for (int r = 0; r < SC_IPT; r++) {
        const int64_t idx = wb + r * 32 + lane;
        if (idx < n) out[idx] = v[r] + add;
    }
}

// up to three independent scans of the same length in one launch (blockIdx.y)
template <class T>
struct ScanSet {
    const T *in[3];
    int64_t *out[3];
};

template <class T>
__global__ void __launch_bounds__(SC_BT) k_scan_final(ScanSet<T> set, int64_t n, const int64_t *partial) {
    pdl_entry();
    const T *in = set.in[blockIdx.y];
    int64_t *out = set.out[blockIdx.y];
    __shared__ int64_t sh[SC_BT / 32];
    const int64_t base = (int64_t)blockIdx.x * SC_TILE;
    int64_t v[SC_IPT];
    const int64_t tot = tile_excl_scan(in, n, base, v, sh);
    const int64_t add = partial ? partial[blockIdx.x] : 0;
    tile_store(out, n, base, v, add);
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = add + tot;
}
// Single-pass exclusive scan with decoupled look-back: each tile publishes
// its aggregate, then its inclusive prefix once known; a tile's prefix is
// found by walking back over its predecessors' published values (32 at a
// time, one warp).  Tile status words carry an epoch so the scratch is never
// cleared between calls (calls on a device are serialised).
constexpr uint32_t kAggBit = 1u, kIncBit = 2u;
template <class T>
__global__ void __launch_bounds__(SC_BT) k_scan_onepass(ScanSet<T> set, int64_t n, uint32_t *flag0, int64_t *agg0,
                                                        int64_t *inc0, int64_t stride, uint32_t epoch) {
    pdl_entry();
    const T *in = set.in[blockIdx.y];
    int64_t *out = set.out[blockIdx.y];
    uint32_t *flag = flag0 + blockIdx.y * stride;
    int64_t *agg = agg0 + blockIdx.y * stride, *inc = inc0 + blockIdx.y * stride;
    __shared__ int64_t sh[SC_BT / 32];
    __shared__ int64_t s_prefix;
    const int64_t tile = blockIdx.x;
    const int64_t base = tile * SC_TILE;
    int64_t v[SC_IPT];
    const int64_t tot = tile_excl_scan(in, n, base, v, sh);
    if (threadIdx.x < 32) {
        const int lane = lane_id();
        int64_t prefix = 0;
        if (tile == 0) {
            if (lane == 0) {
                inc[0] = tot;
                __threadfence();
                atomicExch(&flag[0], (epoch << 2) | kIncBit);
            }
        } else {
            if (lane == 0) {
                agg[tile] = tot;
                __threadfence();
                atomicExch(&flag[tile], (epoch << 2) | kAggBit);
            }
            // look back: predecessors tile-1-lane, 32 per step
            int64_t j = tile - 1;
            while (true) {
                const int64_t t = j - lane;
                uint32_t f = 0;
                if (t >= 0) {
                    do {
                        f = *(volatile uint32_t *)&flag[t];
                    } while ((f >> 2) != epoch);  // not yet published in this call
                }
                __threadfence();
                const bool has_inc = t >= 0 && (f & kIncBit);
                const uint32_t incmask = __ballot_sync(FULL_MASK, has_inc);
                // lanes up to (and including) the first with an inclusive value
                const int stop = incmask ? __ffs(incmask) - 1 : 31;
                int64_t v = 0;
                if (t >= 0 && lane <= stop) v = has_inc ? *(volatile int64_t *)&inc[t] : *(volatile int64_t *)&agg[t];
                prefix += warp_sum(v);
                if (incmask || j - 31 < 0) break;
                j -= 32;
            }
            if (lane == 0) {
                inc[tile] = prefix + tot;
                __threadfence();
                atomicExch(&flag[tile], (epoch << 2) | kIncBit);
            }
        }
        if (lane == 0) s_prefix = prefix;
    }
    __syncthreads();
    tile_store(out, n, base, v, s_prefix);
    if (tile == gridDim.x - 1 && threadIdx.x == 0) out[n] = s_prefix + tot;
}

// persistent per-device look-back scratch (grown on demand)
struct ScanScratch {
    uint32_t *flag = nullptr;
    int64_t *agg = nullptr, *inc = nullptr;
    int64_t cap = 0;
    uint32_t epoch = 0;
};
ScanScratch g_scan[64];
}  // namespace

template <class T>
static void scan_set(Ctx &c, const ScanSet<T> &set, int k, int64_t n) {
    if (n <= 0) {
        for (int q = 0; q < k; q++) c.zero(set.out[q], 1);
        return;
    }
    const int64_t ntiles = cdiv(n, SC_TILE);
    if (ntiles == 1) {
        pdl_launch(k_scan_final<T>, dim3(1, k), SC_BT, 0, c.stream, set, n, nullptr);
        DHGP_LAUNCHED(c);
        return;
    }
    ScanSet<T> s2 = set;
    ScanScratch &ss = g_scan[c.device];
    const int64_t need = 3 * ntiles;
    if (ss.cap < need) {
        // stream-ordered: earlier kernels on this stream are done with the old buffers
        if (ss.flag) {
            c.free(ss.flag);
            c.free(ss.agg);
            c.free(ss.inc);
        }
        ss.cap = std::max<int64_t>(need, 3 * 4096);
        ss.flag = c.alloc<uint32_t>(ss.cap);
        ss.agg = c.alloc<int64_t>(ss.cap);
        ss.inc = c.alloc<int64_t>(ss.cap);
        DHGP_CUDA(cudaMemsetAsync(ss.flag, 0, sizeof(uint32_t) * ss.cap, c.stream));
        ss.epoch = 0;
    }
    ss.epoch = (ss.epoch + 1) & 0x3fffffffu;
    if (ss.epoch == 0) {  // wrapped: clear so no stale word matches
        DHGP_CUDA(cudaMemsetAsync(ss.flag, 0, sizeof(uint32_t) * ss.cap, c.stream));
        ss.epoch = 1;
    }
    pdl_launch(k_scan_onepass<T>, dim3((unsigned)ntiles, k), SC_BT, 0, c.stream, s2, n, ss.flag, ss.agg, ss.inc, ntiles,
                                                                         ss.epoch);
    DHGP_LAUNCHED(c);
}

template <class T>
void scan_excl(Ctx &c, const T *in, int64_t *out, int64_t n) {
    ScanSet<T> set{{in, nullptr, nullptr}, {out, nullptr, nullptr}};
    scan_set(c, set, 1, n);
}
template <class T>
void scan_excl3(Ctx &c, const T *in0, int64_t *out0, const T *in1, int64_t *out1, const T *in2, int64_t *out2,
                int64_t n) {
    ScanSet<T> set{{in0, in1, in2}, {out0, out1, out2}};
    scan_set(c, set, in2 ? 3 : 2, n);
}
template void scan_excl3<int32_t>(Ctx &, const int32_t *, int64_t *, const int32_t *, int64_t *, const int32_t *,
                                  int64_t *, int64_t);
template void scan_excl3<int64_t>(Ctx &, const int64_t *, int64_t *, const int64_t *, int64_t *, const int64_t *,
                                  int64_t *, int64_t);
// running maximum: per-tile maxima, a single-block max-scan over them,
// then per-tile inclusive max with the carry
namespace {
__device__ __forceinline__ int64_t warp_incl_max(int64_t v) {
    const int lane = lane_id();
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int64_t o = __shfl_up_sync(FULL_MASK, v, d);
        if (lane >= d && o > v) v = o;
    }
    return v;
}
// block inclusive max-scan of one value per thread; carry-in applied
__device__ __forceinline__ int64_t block_incl_max(int64_t v, int64_t *sh, int64_t *total) {
    const int lane = lane_id(), w = warp_id(), nw = blockDim.x >> 5;
    int64_t incl = warp_incl_max(v);
    if (lane == 31) sh[w] = incl;
    __syncthreads();
    if (w == 0) {
        int64_t x = lane < nw ? sh[lane] : LLONG_MIN;
        int64_t xi = warp_incl_max(x);
        int64_t prev = __shfl_up_sync(FULL_MASK, xi, 1);
        if (lane < nw) sh[lane] = lane == 0 ? LLONG_MIN : prev;
        if (lane == nw - 1) sh[32] = xi;
    }
    __syncthreads();
    int64_t r = incl > sh[w] ? incl : sh[w];
    *total = sh[32];
    __syncthreads();
    return r;
}
__global__ void k_max_reduce(const int64_t *in, int64_t n, int64_t *partial) {
    pdl_entry();
    __shared__ int64_t sh[33];
    int64_t base = (int64_t)blockIdx.x * SC_TILE, m = LLONG_MIN;
    for (int i = 0; i < SC_IPT; i++) {
        int64_t idx = base + (int64_t)i * SC_BT + threadIdx.x;
        if (idx < n && in[idx] > m) m = in[idx];
    }
    int64_t t;
    block_incl_max(m, sh, &t);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}
__global__ void k_max_partials(int64_t *partial, int64_t ntiles) {
    pdl_entry();
    // exclusive running max over tiles: the carry into each tile
    __shared__ int64_t sh[33];
    __shared__ int64_t incl_s[1024];
    int64_t carry = LLONG_MIN;
    for (int64_t base = 0; base < ntiles; base += blockDim.x) {
        int64_t idx = base + threadIdx.x;
        int64_t v = idx < ntiles ? partial[idx] : LLONG_MIN;
        int64_t tot;
        int64_t incl = block_incl_max(v, sh, &tot);
        incl_s[threadIdx.x] = incl;
        __syncthreads();
        int64_t ex = threadIdx.x ? incl_s[threadIdx.x - 1] : LLONG_MIN;
        if (carry > ex) ex = carry;
        __syncthreads();
        if (idx < ntiles) partial[idx] = ex;
        if (tot > carry) carry = tot;
    }
}
__global__ void k_max_final(const int64_t *in, int64_t n, const int64_t *partial, int64_t *out) {
    pdl_entry();
    __shared__ int64_t sh[33];
    __shared__ int64_t buf[SC_TILE];
    int64_t base = (int64_t)blockIdx.x * SC_TILE;
    for (int i = 0; i < SC_IPT; i++) {
        int64_t idx = base + (int64_t)i * SC_BT + threadIdx.x;
        buf[i * SC_BT + threadIdx.x] = idx < n ? in[idx] : LLONG_MIN;
    }
    __syncthreads();
    int64_t loc[SC_IPT];
    int64_t m = LLONG_MIN;
    for (int i = 0; i < SC_IPT; i++) {
        loc[i] = buf[threadIdx.x * SC_IPT + i];
        if (loc[i] > m) m = loc[i];
    }
    int64_t tot;
    int64_t incl = block_incl_max(m, sh, &tot);
    // exclusive max for this thread = inclusive max of the previous thread
    __shared__ int64_t prev_of[SC_BT];
    prev_of[threadIdx.x] = incl;
    __syncthreads();
    int64_t run = threadIdx.x ? prev_of[threadIdx.x - 1] : LLONG_MIN;
    if (partial && partial[blockIdx.x] > run) run = partial[blockIdx.x];
    for (int i = 0; i < SC_IPT; i++) {
        if (loc[i] > run) run = loc[i];
        buf[threadIdx.x * SC_IPT + i] = run;
    }
    __syncthreads();
    for (int i = 0; i < SC_IPT; i++) {
        int64_t idx = base + (int64_t)i * SC_BT + threadIdx.x;
        if (idx < n) out[idx] = buf[i * SC_BT + threadIdx.x];
    }
}
}  // namespace

void scan_incl_max(Ctx &c, const int64_t *in, int64_t *out, int64_t n) {
    if (n <= 0) return;
    int64_t ntiles = cdiv(n, SC_TILE);
    if (ntiles == 1) {
        pdl_launch(k_max_final, 1, SC_BT, 0, c.stream, in, n, nullptr, out);
        DHGP_LAUNCHED(c);
        return;
    }
    int64_t *partial = c.alloc<int64_t>(ntiles + 1);
    pdl_launch(k_max_reduce, (unsigned)ntiles, SC_BT, 0, c.stream, in, n, partial);
    DHGP_LAUNCHED(c);
    pdl_launch(k_max_partials, 1, 1024, 0, c.stream, partial, ntiles);
    DHGP_LAUNCHED(c);
    pdl_launch(k_max_final, (unsigned)ntiles, SC_BT, 0, c.stream, in, n, partial, out);
    DHGP_LAUNCHED(c);
    c.free(partial);
}

template void scan_excl<int32_t>(Ctx &, const int32_t *, int64_t *, int64_t);
template void scan_excl<int64_t>(Ctx &, const int64_t *, int64_t *, int64_t);
template void scan_excl<uint8_t>(Ctx &, const uint8_t *, int64_t *, int64_t);

// ===========================================================================
// stable LSD radix sort, 8-bit digits, tile = 8 warps x 8 steps x 32 lanes
// ===========================================================================
namespace {
constexpr int RS_BT = 256;
constexpr int RS_STEPS = 8;
constexpr int RS_TILE = RS_BT * RS_STEPS;

__global__ void k_rs_up(const uint64_t *kin, int64_t ncap, const int64_t *dn, int shift, int64_t *counts,
                        int64_t ntiles) {
    pdl_entry();
    __shared__ uint32_t cnt[256];
    const int64_t n = dn ? *dn : ncap;
    cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
    if (base < n) {
#pragma unroll
        for (int s = 0; s < RS_STEPS; s++) {
            int64_t idx = base + (int64_t)s * RS_BT + threadIdx.x;
            if (idx < n) atomicAdd(&cnt[(kin[idx] >> shift) & 255u], 1u);
        }
    }
    __syncthreads();
    counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = cnt[threadIdx.x];
}

__global__ void k_rs_down(const uint64_t *kin, const uint32_t *vin, uint64_t *kout, uint32_t *vout, int64_t ncap,
                          const int64_t *dn, int shift, const int64_t *offs, int64_t ntiles) {
    pdl_entry();
    __shared__ uint32_t wcnt[RS_BT / 32][256];
    const int64_t n = dn ? *dn : ncap;
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
    if (base >= n) return;
    const int w = warp_id(), lane = lane_id();
    for (int i = threadIdx.x; i < (RS_BT / 32) * 256; i += RS_BT) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    uint64_t k[RS_STEPS];
    uint32_t v[RS_STEPS];
    int dig[RS_STEPS];
    uint32_t rank[RS_STEPS];
    const uint32_t lt_mask = (1u << lane) - 1u;
    // warp w owns the contiguous range [base + w*256, base + (w+1)*256)
#pragma unroll
    for (int s = 0; s < RS_STEPS; s++) {
        int64_t idx = base + (int64_t)w * (32 * RS_STEPS) + s * 32 + lane;
        bool valid = idx < n;
        k[s] = valid ? kin[idx] : ~0ull;
        v[s] = valid ? vin[idx] : 0u;
        dig[s] = valid ? (int)((k[s] >> shift) & 255u) : 256;
        uint32_t peers = __match_any_sync(FULL_MASK, dig[s]);
        uint32_t before = valid ? wcnt[w][dig[s]] : 0u;
        rank[s] = before + __popc(peers & lt_mask);
        __syncwarp();
        if (valid && (peers & lt_mask) == 0) wcnt[w][dig[s]] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {
        const int d = threadIdx.x;  // RS_BT == 256 digits
        uint32_t run = 0;
#pragma unroll
        for (int ww = 0; ww < RS_BT / 32; ww++) {
            uint32_t cc = wcnt[ww][d];
            wcnt[ww][d] = run;
            run += cc;
        }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < RS_STEPS; s++) {
        if (dig[s] < 256) {
            int64_t pos = offs[(int64_t)dig[s] * ntiles + blockIdx.x] + wcnt[w][dig[s]] + rank[s];
            kout[pos] = k[s];
            vout[pos] = v[s];
        }
    }
}
}  // namespace

namespace {
__global__ void __launch_bounds__(1024) k_small_sort(uint64_t *keys, uint32_t *vals, int n) {
    pdl_entry();
    __shared__ uint64_t sk[kSmallSort];
    __shared__ uint32_t sv[kSmallSort];
    int np = 1;
    while (np < n) np <<= 1;
    for (int i = threadIdx.x; i < np; i += blockDim.x) {
        sk[i] = i < n ? keys[i] : ~0ull;
        sv[i] = i < n ? vals[i] : 0xffffffffu;
    }
    for (int size = 2; size <= np; size <<= 1) {
        for (int j = size >> 1; j > 0; j >>= 1) {
            __syncthreads();
            for (int t = threadIdx.x; t < (np >> 1); t += blockDim.x) {
                const int lo = 2 * j * (t / j) + (t % j), hi = lo + j;
                const bool asc = (lo & size) == 0;
                const uint64_t a = sk[lo], b = sk[hi];
                const uint32_t va = sv[lo], vb = sv[hi];
                const bool gt = a > b || (a == b && va > vb);
                if (gt == asc) {
                    sk[lo] = b;
                    sk[hi] = a;
                    sv[lo] = vb;
                    sv[hi] = va;
                }
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        keys[i] = sk[i];
        vals[i] = sv[i];
    }
}
// unique u64 keys whose low 32 bits are the value (the packed mover keys)
__global__ void __launch_bounds__(1024) k_small_sort_packed(uint64_t *keys, uint32_t *vals, int n,
                                                            const int64_t *dn) {
    pdl_entry();
    if (dn) {  // count on device: a no-op when it does not fit
        const int64_t m = *dn;
        if (m <= 1 || m > kSmallSort) return;
        n = (int)m;
    }
    extern __shared__ unsigned long long sm[];
    uint64_t *a = (uint64_t *)sm, *b = a + kSmallSort;
    for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = keys[i];
    __syncthreads();
    block_sort_u64_4096(a, b, n);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        keys[i] = a[i];
        vals[i] = (uint32_t)a[i];
    }
}
}  // namespace

void small_sort_pairs(Ctx &c, uint64_t *keys, uint32_t *vals, int64_t n) {
    if (n <= 1) return;
    KScope ks(c, "radix_sort");
    pdl_launch(k_small_sort, 1, 1024, 0, c.stream, keys, vals, (int)n);
    DHGP_LAUNCHED(c);
}
void small_sort_packed(Ctx &c, uint64_t *keys, uint32_t *vals, int64_t n, const int64_t *dn) {
    if (!dn && n <= 1) return;
    KScope ks(c, "radix_sort");
    static bool attr = false;
    if (!attr) {
        DHGP_CUDA(cudaFuncSetAttribute(k_small_sort_packed, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(2 * kSmallSort * sizeof(uint64_t))));
        attr = true;
    }
    pdl_launch(k_small_sort_packed, 1, 1024, 2 * kSmallSort * sizeof(uint64_t), c.stream, keys, vals, (int)n, dn);
    DHGP_LAUNCHED(c);
}

// ===========================================================================
// merge sort of (key, val) pairs by (key, val) for mid-size arrays: chunks of
// MS_CHUNK sorted in shared memory (one CTA each, bitonic), then merge passes
// that double the run width (merge path: each thread finds its co-rank once
// and emits MS_PER consecutive outputs).  A handful of launches instead of
// three per 8-bit radix pass.
// ===========================================================================
namespace {
constexpr int MS_CHUNK = 512, MS_THREADS = 256, MS_PER = 8;
__device__ __forceinline__ bool pair_less(uint64_t ka, uint32_t va, uint64_t kb, uint32_t vb) {
    return ka < kb || (ka == kb && va < vb);
}
__global__ void __launch_bounds__(MS_THREADS) k_chunk_sort(uint64_t *keys, uint32_t *vals, int64_t n) {
    pdl_entry();
    __shared__ uint64_t sk[MS_CHUNK];
    __shared__ uint32_t sv[MS_CHUNK];
    const int64_t base = (int64_t)blockIdx.x * MS_CHUNK;
    const int m = (int)min((int64_t)MS_CHUNK, n - base);
    for (int i = threadIdx.x; i < MS_CHUNK; i += MS_THREADS) {
        sk[i] = i < m ? keys[base + i] : ~0ull;
        sv[i] = i < m ? vals[base + i] : 0xffffffffu;
    }
    for (int size = 2; size <= MS_CHUNK; size <<= 1) {
        for (int j = size >> 1; j > 0; j >>= 1) {
            __syncthreads();
            for (int t = threadIdx.x; t < MS_CHUNK / 2; t += MS_THREADS) {
                const int lo = 2 * j * (t / j) + (t % j), hi = lo + j;
                const bool asc = (lo & size) == 0;
                const uint64_t a = sk[lo], b = sk[hi];
                const uint32_t va = sv[lo], vb = sv[hi];
                if (pair_less(b, vb, a, va) == asc) {
                    sk[lo] = b;
                    sk[hi] = a;
                    sv[lo] = vb;
                    sv[hi] = va;
                }
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += MS_THREADS) {
        keys[base + i] = sk[i];
        vals[base + i] = sv[i];
    }
}
// merge of the sorted runs [r0, r0 + w) and [r0 + w, r0 + 2w) (clipped to n)
__global__ void k_merge_pass(const uint64_t *ki, const uint32_t *vi, uint64_t *ko, uint32_t *vo, int64_t n,
                             int64_t w) {
    pdl_entry();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t o = t * MS_PER;
    if (o >= n) return;
    const int64_t r0 = (o / (2 * w)) * (2 * w);
    const int64_t a0 = r0, a1 = min(n, r0 + w), b0 = a1, b1 = min(n, r0 + 2 * w);
    const int64_t na = a1 - a0, nb = b1 - b0, k = o - r0;  // output rank within the merged run
    // co-rank: i elements from A, k - i from B, with A[i-1] <= B[k-i] and B[k-i-1] < A[i]
    int64_t lo = max((int64_t)0, k - nb), hi = min(k, na);
    while (lo < hi) {
        const int64_t i = (lo + hi) >> 1;  // take i from A: is A[i] <= B[k-i-1]? then more from A
        if (!pair_less(ki[b0 + k - i - 1], vi[b0 + k - i - 1], ki[a0 + i], vi[a0 + i])) lo = i + 1;
        else hi = i;
    }
    int64_t i = lo, j = k - lo;
    const int64_t end = min(n, o + MS_PER);
    for (int64_t q = o; q < end; q++) {
        const bool takeA = j >= nb || (i < na && !pair_less(ki[b0 + j], vi[b0 + j], ki[a0 + i], vi[a0 + i]));
        if (takeA) {
            ko[q] = ki[a0 + i];
            vo[q] = vi[a0 + i];
            i++;
        } else {
            ko[q] = ki[b0 + j];
            vo[q] = vi[b0 + j];
            j++;
        }
    }
}
}  // namespace

void merge_sort_pairs(Ctx &c, uint64_t *keys, uint32_t *vals, uint64_t *ktmp, uint32_t *vtmp, int64_t n) {
    if (n <= 1) return;
    KScope ks(c, "radix_sort", 24.0 * (double)n * (1.0 + std::max(0.0, std::ceil(std::log2((double)n / MS_CHUNK)))));
    pdl_launch(k_chunk_sort, (unsigned)cdiv(n, MS_CHUNK), MS_THREADS, 0, c.stream, keys, vals, n);
    DHGP_LAUNCHED(c);
    uint64_t *ka = keys, *kb = ktmp;
    uint32_t *va = vals, *vb = vtmp;
    for (int64_t w = MS_CHUNK; w < n; w *= 2) {
        pdl_launch(k_merge_pass, (unsigned)cdiv(cdiv(n, MS_PER), 256), 256, 0, c.stream, (const uint64_t *)ka,
                   (const uint32_t *)va, kb, vb, n, w);
        DHGP_LAUNCHED(c);
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    if (ka != keys) {
        c.d2d(keys, ka, n);
        c.d2d(vals, va, n);
    }
}

void radix_sort_pairs(Ctx &c, uint64_t *keys, uint32_t *vals, uint64_t *ktmp, uint32_t *vtmp, int64_t n_cap,
                      const int64_t *d_n, int bits) {
    if (n_cap <= 1 || bits <= 0) return;
    // algorithmic bytes: every pass reads and writes the (key, value) pairs
    KScope ks(c, "radix_sort", 24.0 * (double)n_cap * (double)((bits + 7) / 8));
    const int64_t ntiles = cdiv(n_cap, RS_TILE);
    int64_t *counts = c.alloc<int64_t>(256 * ntiles);
    int64_t *offs = c.alloc<int64_t>(256 * ntiles + 1);
    uint64_t *ka = keys, *kb = ktmp;
    uint32_t *va = vals, *vb = vtmp;
    const int passes = (bits + 7) / 8;
    for (int p = 0; p < passes; p++) {
        const int shift = 8 * p;
        pdl_launch(k_rs_up, (unsigned)ntiles, RS_BT, 0, c.stream, ka, n_cap, d_n, shift, counts, ntiles);
        DHGP_LAUNCHED(c);
        scan_excl<int64_t>(c, counts, offs, 256 * ntiles);
        pdl_launch(k_rs_down, (unsigned)ntiles, RS_BT, 0, c.stream, ka, va, kb, vb, n_cap, d_n, shift, offs, ntiles);
        DHGP_LAUNCHED(c);
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    if (ka != keys) {
        // odd number of passes: result sits in the scratch buffers
        c.d2d(keys, ka, n_cap);
        c.d2d(vals, va, n_cap);
    }
    c.free(counts);
    c.free(offs);
}

// ===========================================================================
// per-segment sort (three tiers: thread <= 16, warp <= 128, block <= 8192)
// ===========================================================================
namespace {
constexpr int kThreadTier = 16;
constexpr int kWarpTier = 128;

__global__ void k_seg_sort_thread(int64_t nseg, const int64_t *off, const int32_t *dat, const int32_t *map,
                                  int32_t *tmp, int32_t *warp_list, int32_t *block_list, int32_t *counts) {
    pdl_entry();
    int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nseg) return;
    int64_t lo = off[s], len = off[s + 1] - lo;
    if (len > kThreadTier) {
        if (len <= kWarpTier)
            warp_list[atomicAdd(&counts[0], 1)] = (int32_t)s;
        else
            block_list[atomicAdd(&counts[1], 1)] = (int32_t)s;
        return;
    }
    uint32_t a[kThreadTier];
#pragma unroll
    for (int i = 0; i < kThreadTier; i++) {
        if (i < len) {
            int32_t x = dat[lo + i];
            a[i] = (uint32_t)(map ? map[x] : x);
        }
    }
    // insertion sort
    for (int i = 1; i < len; i++) {
        uint32_t x = a[i];
        int j = i - 1;
        while (j >= 0 && a[j] > x) {
            a[j + 1] = a[j];
            j--;
        }
        a[j + 1] = x;
    }
    for (int i = 0; i < len; i++) tmp[lo + i] = (int32_t)a[i];
}

template <int K>
__device__ __forceinline__ void warp_sort_segment(int64_t lo, int len, const int32_t *dat, const int32_t *map,
                                                  int32_t *tmp) {
    const int lane = lane_id();
    uint32_t v[K];
    bool sorted = true;
#pragma unroll
    for (int k = 0; k < K; k++) {
        int i = k * 32 + lane;
        if (i < len) {
            int32_t x = dat[lo + i];
            v[k] = (uint32_t)(map ? map[x] : x);
        } else {
            v[k] = 0xffffffffu;
        }
    }
    // fast path: already strictly ascending (e.g. gamma is monotone on this edge)
#pragma unroll
    for (int k = 0; k < K; k++) {
        const int i = k * 32 + lane;
        uint32_t up = __shfl_up_sync(FULL_MASK, v[k], 1);
        uint32_t wrap = __shfl_sync(FULL_MASK, v[k > 0 ? k - 1 : 0], 31);
        uint32_t prev = lane == 0 ? wrap : up;
        if (i > 0 && i < len && !(prev < v[k])) sorted = false;
    }
    if (!__all_sync(FULL_MASK, sorted)) warp_bitonic_sort<K>(v);
#pragma unroll
    for (int k = 0; k < K; k++) {
        int i = k * 32 + lane;
        if (i < len) tmp[lo + i] = (int32_t)v[k];
    }
}

__global__ void k_seg_sort_warp(const int64_t *off, const int32_t *dat, const int32_t *map, int32_t *tmp,
                                const int32_t *list, const int32_t *counts) {
    pdl_entry();
    const int nw = gridDim.x * (blockDim.x >> 5);
    const int n = counts[0];
    for (int t = blockIdx.x * (blockDim.x >> 5) + warp_id(); t < n; t += nw) {
        int64_t s = list[t];
        int64_t lo = off[s];
        int len = (int)(off[s + 1] - lo);
        if (len <= 32)
            warp_sort_segment<1>(lo, len, dat, map, tmp);
        else if (len <= 64)
            warp_sort_segment<2>(lo, len, dat, map, tmp);
        else
            warp_sort_segment<4>(lo, len, dat, map, tmp);
    }
}

__global__ void k_seg_sort_block(const int64_t *off, const int32_t *dat, const int32_t *map, int32_t *tmp,
                                 const int32_t *list, const int32_t *counts, int smem_max) {
    pdl_entry();
    extern __shared__ uint32_t sbuf[];
    const int n = counts[1];
    for (int t = blockIdx.x; t < n; t += gridDim.x) {
        int64_t s = list[t];
        int64_t lo = off[s];
        int len = (int)(off[s + 1] - lo);
        if (len > smem_max) {  // in place in global memory (tmp is the segment's own output)
            __syncthreads();
            for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
                const int32_t x = dat[lo + i];
                tmp[lo + i] = map ? map[x] : x;
            }
            block_sort_asc_any<uint32_t>((uint32_t *)(tmp + lo), len);
            continue;
        }
        int np = next_pow2(len);
        __syncthreads();
        for (int i = threadIdx.x; i < np; i += blockDim.x) {
            if (i < len) {
                int32_t x = dat[lo + i];
                sbuf[i] = (uint32_t)(map ? map[x] : x);
            } else {
                sbuf[i] = 0xffffffffu;
            }
        }
        block_bitonic_sort32(sbuf, np);
        for (int i = threadIdx.x; i < len; i += blockDim.x) tmp[lo + i] = (int32_t)sbuf[i];
        __syncthreads();
    }
}
}  // namespace

void seg_sort(Ctx &c, int64_t nseg, const int64_t *off, const int32_t *dat, const int32_t *map, int32_t *tmp) {
    if (nseg <= 0) return;
    KScope ks(c, "seg_sort");  // (bytes: only as part of an enclosing class)
    int32_t *wl = c.alloc<int32_t>(nseg);
    int32_t *bl = c.alloc<int32_t>(nseg);
    int32_t *cnt = c.alloc<int32_t>(3);
    c.zero(cnt, 3);
    pdl_launch(k_seg_sort_thread, (unsigned)cdiv(nseg, 256), 256, 0, c.stream, nseg, off, dat, map, tmp, wl, bl, cnt);
    DHGP_LAUNCHED(c);
    pdl_launch(k_seg_sort_warp, (unsigned)(c.num_sms * 8), 256, 0, c.stream, off, dat, map, tmp, wl, cnt);
    DHGP_LAUNCHED(c);
    // segments above kMaxSegSort (shared memory) sort in place in global memory
    pdl_launch(k_seg_sort_block, (unsigned)(c.num_sms), 1024, kMaxSegSort * sizeof(uint32_t), c.stream, off, dat, map, tmp,
                                                                                                 bl, cnt,
               std::min<int>((int)kMaxSegSort, tiers().seg_smem));
    DHGP_LAUNCHED(c);
    c.free(wl);
    c.free(bl);
    c.free(cnt);
}

namespace {
__global__ void k_seg_unique_count(int64_t nseg, const int64_t *off, const int32_t *tmp, int64_t *cnt) {
    pdl_entry();
    int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nseg) return;
    int64_t lo = off[s], hi = off[s + 1];
    int64_t k = 0;
    int32_t prev = 0;
    for (int64_t p = lo; p < hi; p++) {
        int32_t x = tmp[p];
        if (p == lo || x != prev) k++;
        prev = x;
    }
    cnt[s] = k;
}
__global__ void k_seg_unique_write(int64_t nseg, const int64_t *off, const int32_t *tmp, const int64_t *out_off,
                                   int32_t *out) {
    pdl_entry();
    int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nseg) return;
    int64_t lo = off[s], hi = off[s + 1];
    int64_t w = out_off[s];
    int32_t prev = 0;
    for (int64_t p = lo; p < hi; p++) {
        int32_t x = tmp[p];
        if (p == lo || x != prev) out[w++] = x;
        prev = x;
    }
}
}  // namespace

void seg_unique_count(Ctx &c, int64_t nseg, const int64_t *off, const int32_t *tmp, int64_t *cnt) {
    if (nseg <= 0) return;
    pdl_launch(k_seg_unique_count, (unsigned)cdiv(nseg, 256), 256, 0, c.stream, nseg, off, tmp, cnt);
    DHGP_LAUNCHED(c);
}
void seg_unique_write(Ctx &c, int64_t nseg, const int64_t *off, const int32_t *tmp, const int64_t *out_off,
                      int32_t *out) {
    if (nseg <= 0) return;
    pdl_launch(k_seg_unique_write, (unsigned)cdiv(nseg, 256), 256, 0, c.stream, nseg, off, tmp, out_off, out);
    DHGP_LAUNCHED(c);
}

// ===========================================================================
// sorted-set union of member lists (warp per coarse node)
// ===========================================================================
namespace {
constexpr int64_t kMergeBig = 2048;
// two node families (in, inc) per launch: blockIdx.y picks one
struct MergeFam {
    const int64_t *off;
    const int32_t *dat;
    int64_t *cnt;            // count pass
    const int64_t *out_off;  // write pass
    int32_t *out;
    int32_t *big_list;
    int32_t *big_count;
};
struct MergeFams {
    MergeFam f[2];
};
__device__ __forceinline__ void merge_count_body(int64_t nc_cap, const int64_t *d_nc, const int32_t *ma,
                                                 const int32_t *mb, const int64_t *off, const int32_t *dat,
                                                 int64_t *cnt, int32_t *big_list, int32_t *big_count);
__global__ void k_merge_count2(int64_t nc_cap, const int64_t *d_nc, const int32_t *ma, const int32_t *mb,
                               MergeFams fs) {
    pdl_entry();
    const MergeFam &f = fs.f[blockIdx.y];
    merge_count_body(nc_cap, d_nc, ma, mb, f.off, f.dat, f.cnt, f.big_list, f.big_count);
}
__device__ __forceinline__ void merge_count_body(int64_t nc_cap, const int64_t *d_nc, const int32_t *ma,
                                                 const int32_t *mb, const int64_t *off, const int32_t *dat,
                                                 int64_t *cnt, int32_t *big_list, int32_t *big_count) {
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int lane = lane_id();
    const int64_t nc = d_nc ? *d_nc : nc_cap;
    for (int64_t cn = nc + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; cn < nc_cap;
         cn += (int64_t)gridDim.x * blockDim.x)
        cnt[cn] = 0;
    for (int64_t cn = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id(); cn < nc; cn += nw) {
        int32_t a = ma[cn], b = mb[cn];
        int64_t alo = off[a], na = off[a + 1] - alo;
        if (b < 0) {
            if (lane == 0) {
                cnt[cn] = na;
                // a long list is copied by a block (a warp would serialise on it)
                if (big_list && na > kMergeBig) big_list[atomicAdd(big_count, 1)] = (int32_t)cn;
            }
            continue;
        }
        int64_t blo = off[b], nb = off[b + 1] - blo;
        if (big_list && na + nb > kMergeBig) {  // a block takes it
            if (lane == 0) big_list[atomicAdd(big_count, 1)] = (int32_t)cn;
            continue;
        }
        // common elements: search the shorter list in the longer
        const int32_t *sp = dat + (na <= nb ? alo : blo);
        const int32_t *lp = dat + (na <= nb ? blo : alo);
        int64_t ns = na <= nb ? na : nb, nl = na <= nb ? nb : na;
        int64_t common = 0;
        for (int64_t i = lane; i < ns; i += 32) common += bsearch_dev(lp, 0, nl, sp[i]) >= 0;
        common = warp_sum(common);
        if (lane == 0) cnt[cn] = na + nb - common;
    }
}

__device__ __forceinline__ void merge_write_body(int64_t nc, const int32_t *ma, const int32_t *mb, const int64_t *off,
                                                 const int32_t *dat, const int64_t *out_off, int32_t *out,
                                                 bool skip_big);
__global__ void k_merge_write2(int64_t nc, const int32_t *ma, const int32_t *mb, MergeFams fs, bool skip_big) {
    pdl_entry();
    const MergeFam &f = fs.f[blockIdx.y];
    merge_write_body(nc, ma, mb, f.off, f.dat, f.out_off, f.out, skip_big);
}
__device__ __forceinline__ void merge_write_body(int64_t nc, const int32_t *ma, const int32_t *mb, const int64_t *off,
                                                 const int32_t *dat, const int64_t *out_off, int32_t *out,
                                                 bool skip_big) {
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int lane = lane_id();
    const uint32_t lt = (1u << lane) - 1u;
    for (int64_t cn = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp_id(); cn < nc; cn += nw) {
        int32_t a = ma[cn], b = mb[cn];
        int64_t alo = off[a], na = off[a + 1] - alo;
        int32_t *o = out + out_off[cn];
        const int32_t *A = dat + alo;
        if (b < 0) {
            if (skip_big && na > kMergeBig) continue;
            // four loads in flight per lane before the stores
            int64_t i = lane;
            for (; i + 96 < na; i += 128) {
                const int32_t x0 = A[i], x1 = A[i + 32], x2 = A[i + 64], x3 = A[i + 96];
                o[i] = x0;
                o[i + 32] = x1;
                o[i + 64] = x2;
                o[i + 96] = x3;
            }
            for (; i < na; i += 32) o[i] = A[i];
            continue;
        }
        int64_t blo = off[b], nb = off[b + 1] - blo;
        if (skip_big && na + nb > kMergeBig) continue;
        const int32_t *B = dat + blo;
        // x = A[i]: pos = i + lb_B(x) - #{A[k], k < i : A[k] in B}
        int64_t run = 0;
        for (int64_t base = 0; base < na; base += 32) {
            int64_t i = base + lane;
            int64_t lb = 0;
            bool in_other = false;
            int32_t x = 0;
            if (i < na) {
                x = A[i];
                lb = lower_bound_dev<int32_t>(B, 0, nb, x);
                in_other = lb < nb && B[lb] == x;
            }
            uint32_t bal = __ballot_sync(FULL_MASK, in_other);
            if (i < na) o[i + lb - (run + __popc(bal & lt))] = x;
            run += __popc(bal);
        }
        // y = B[j] not in A: pos = lb_A(y) + j - #{B[k], k < j : B[k] in A}
        run = 0;
        for (int64_t base = 0; base < nb; base += 32) {
            int64_t j = base + lane;
            int64_t lb = 0;
            bool in_other = false;
            int32_t y = 0;
            if (j < nb) {
                y = B[j];
                lb = lower_bound_dev<int32_t>(A, 0, na, y);
                in_other = lb < na && A[lb] == y;
            }
            uint32_t bal = __ballot_sync(FULL_MASK, in_other);
            if (j < nb && !in_other) o[lb + j - (run + __popc(bal & lt))] = y;
            run += __popc(bal);
        }
    }
}

// block-per-node union for large member lists (hubs), same formulas as the
// warp version with a block-wide prefix over the "in the other list" flags
__device__ __forceinline__ int64_t block_excl_flags(bool f, int64_t *sh_w, int64_t *total) {
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
__device__ __forceinline__ void merge_count_big_body(const int32_t *list, const int32_t *count, const int32_t *ma,
                                                     const int32_t *mb, const int64_t *off, const int32_t *dat,
                                                     int64_t *cnt);
__global__ void k_merge_count_big2(const int32_t *ma, const int32_t *mb, MergeFams fs) {
    pdl_entry();
    const MergeFam &f = fs.f[blockIdx.y];
    merge_count_big_body(f.big_list, f.big_count, ma, mb, f.off, f.dat, f.cnt);
}
__device__ __forceinline__ void merge_count_big_body(const int32_t *list, const int32_t *count, const int32_t *ma,
                                                     const int32_t *mb, const int64_t *off, const int32_t *dat,
                                                     int64_t *cnt) {
    __shared__ int64_t sh[32];
    const int n = *count;
    for (int t = blockIdx.x; t < n; t += gridDim.x) {
        const int32_t cn = list[t], a = ma[cn], b = mb[cn];
        if (b < 0) continue;  // a long unmerged list: counted by the warp kernel
        const int64_t alo = off[a], na = off[a + 1] - alo, blo = off[b], nb = off[b + 1] - blo;
        const int32_t *sp = dat + (na <= nb ? alo : blo), *lp = dat + (na <= nb ? blo : alo);
        const int64_t ns = na <= nb ? na : nb, nl = na <= nb ? nb : na;
        int64_t common = 0;
        for (int64_t i = threadIdx.x; i < ns; i += blockDim.x) common += bsearch_dev(lp, 0, nl, sp[i]) >= 0;
        int64_t tot = block_sum<int64_t>(common, sh);
        if (threadIdx.x == 0) cnt[cn] = na + nb - tot;
        __syncthreads();
    }
}
__device__ __forceinline__ void merge_write_big_body(const int32_t *list, const int32_t *count, const int32_t *ma,
                                                     const int32_t *mb, const int64_t *off, const int32_t *dat,
                                                     const int64_t *out_off, int32_t *out);
__global__ void k_merge_write_big2(const int32_t *ma, const int32_t *mb, MergeFams fs) {
    pdl_entry();
    const MergeFam &f = fs.f[blockIdx.y];
    merge_write_big_body(f.big_list, f.big_count, ma, mb, f.off, f.dat, f.out_off, f.out);
}
__device__ __forceinline__ void merge_write_big_body(const int32_t *list, const int32_t *count, const int32_t *ma,
                                                     const int32_t *mb, const int64_t *off, const int32_t *dat,
                                                     const int64_t *out_off, int32_t *out) {
    __shared__ int64_t sh[32];
    const int n = *count;
    for (int t = blockIdx.x; t < n; t += gridDim.x) {
        const int32_t cn = list[t], a = ma[cn], b = mb[cn];
        if (b < 0) {  // a long unmerged list: block copy
            const int64_t alo = off[a], na = off[a + 1] - alo;
            int32_t *o = out + out_off[cn];
            for (int64_t i = threadIdx.x; i < na; i += blockDim.x) o[i] = dat[alo + i];
            continue;
        }
        const int64_t alo = off[a], na = off[a + 1] - alo, blo = off[b], nb = off[b + 1] - blo;
        const int32_t *A = dat + alo, *B = dat + blo;
        int32_t *o = out + out_off[cn];
        int64_t run = 0;
        for (int64_t base = 0; base < na; base += blockDim.x) {
            const int64_t i = base + threadIdx.x;
            int64_t lb = 0;
            bool in_other = false;
            int32_t x = 0;
            if (i < na) {
                x = A[i];
                lb = lower_bound_dev<int32_t>(B, 0, nb, x);
                in_other = lb < nb && B[lb] == x;
            }
            int64_t tot;
            const int64_t ex = block_excl_flags(in_other, sh, &tot);
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
                y = B[j];
                lb = lower_bound_dev<int32_t>(A, 0, na, y);
                in_other = lb < na && A[lb] == y;
            }
            int64_t tot;
            const int64_t ex = block_excl_flags(in_other, sh, &tot);
            if (j < nb && !in_other) o[lb + j - (run + ex)] = y;
            run += tot;
        }
        __syncthreads();
    }
}
}  // namespace

void merge_union_count2(Ctx &c, int64_t nc, const int32_t *ma, const int32_t *mb, const int64_t *off0,
                        const int32_t *dat0, int64_t *cnt0, int32_t *big0, int32_t *bigc0, const int64_t *off1,
                        const int32_t *dat1, int64_t *cnt1, int32_t *big1, int32_t *bigc1, const int64_t *d_nc) {
    if (nc <= 0) return;
    MergeFams fs{{MergeFam{off0, dat0, cnt0, nullptr, nullptr, big0, bigc0},
                  MergeFam{off1, dat1, cnt1, nullptr, nullptr, big1, bigc1}}};
    const int64_t blocks = std::min<int64_t>(cdiv(nc, 8), (int64_t)c.num_sms * 16);
    pdl_launch(k_merge_count2, dim3((unsigned)blocks, 2), 256, 0, c.stream, nc, d_nc, ma, mb, fs);
    DHGP_LAUNCHED(c);
    pdl_launch(k_merge_count_big2, dim3(c.num_sms, 2), 1024, 0, c.stream, ma, mb, fs);
    DHGP_LAUNCHED(c);
}
void merge_union_write2(Ctx &c, int64_t nc, const int32_t *ma, const int32_t *mb, const int64_t *off0,
                        const int32_t *dat0, const int64_t *out_off0, int32_t *out0, int32_t *big0, int32_t *bigc0,
                        const int64_t *off1, const int32_t *dat1, const int64_t *out_off1, int32_t *out1,
                        int32_t *big1, int32_t *bigc1) {
    if (nc <= 0) return;
    MergeFams fs{{MergeFam{off0, dat0, nullptr, out_off0, out0, big0, bigc0},
                  MergeFam{off1, dat1, nullptr, out_off1, out1, big1, bigc1}}};
    const int64_t blocks = std::min<int64_t>(cdiv(nc, 8), (int64_t)c.num_sms * 16);
    pdl_launch(k_merge_write2, dim3((unsigned)blocks, 2), 256, 0, c.stream, nc, ma, mb, fs, true);
    DHGP_LAUNCHED(c);
    pdl_launch(k_merge_write_big2, dim3(c.num_sms, 2), 1024, 0, c.stream, ma, mb, fs);
    DHGP_LAUNCHED(c);
}

// ===========================================================================
// several small zero-fills in one launch (blockIdx.y = buffer)
// ===========================================================================
namespace {
constexpr int kZeroMax = 16;
struct ZeroSet {
    void *p[kZeroMax];
    int64_t bytes[kZeroMax];
};
__global__ void k_zero_many(ZeroSet z) {
    pdl_entry();
    char *p = (char *)z.p[blockIdx.y];
    const int64_t nb = z.bytes[blockIdx.y];
    const int64_t nw = nb >> 2;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += (int64_t)gridDim.x * blockDim.x)
        ((uint32_t *)p)[i] = 0u;
    if (blockIdx.x == 0 && threadIdx.x < (nb & 3)) p[nw * 4 + threadIdx.x] = 0;
}
// 16-byte stores over the aligned body, single bytes only for the head up to
// the first 16-byte boundary and the tail after the last one
__global__ void k_fill(uint8_t *p, uint32_t word, size_t bytes) {
    pdl_entry();
    const size_t stride = (size_t)gridDim.x * blockDim.x, t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t head = std::min<size_t>(bytes, (16 - ((uintptr_t)p & 15)) & 15);
    const size_t body = (bytes - head) >> 4;
    const uint4 v = make_uint4(word, word, word, word);
    uint4 *q = (uint4 *)(p + head);
    for (size_t i = t; i < body; i += stride) q[i] = v;
    const size_t tail0 = head + (body << 4);
    if (t < head) p[t] = (uint8_t)word;
    if (t < bytes - tail0) p[tail0 + t] = (uint8_t)word;
}
// 16-byte loads and stores when source and destination share their offset
// within 16 bytes (the arena's blocks always do), bytes otherwise
__global__ void k_copy(uint8_t *d, const uint8_t *s, size_t bytes) {
    pdl_entry();
    const size_t stride = (size_t)gridDim.x * blockDim.x, t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if ((((uintptr_t)d ^ (uintptr_t)s) & 15) == 0) {
        const size_t head = std::min<size_t>(bytes, (16 - ((uintptr_t)d & 15)) & 15);
        const size_t body = (bytes - head) >> 4;
        const uint4 *sq = (const uint4 *)(s + head);
        uint4 *dq = (uint4 *)(d + head);
        for (size_t i = t; i < body; i += stride) dq[i] = sq[i];
        const size_t tail0 = head + (body << 4);
        if (t < head) d[t] = s[t];
        if (t < bytes - tail0) d[tail0 + t] = s[tail0 + t];
    } else {
        for (size_t i = t; i < bytes; i += stride) d[i] = s[i];
    }
}
unsigned fill_grid(size_t bytes) { return (unsigned)std::max<size_t>(1, std::min<size_t>((bytes / 16 + 255) / 256, 148 * 8)); }
}  // namespace

void dev_fill(void *p, int byte, size_t bytes, cudaStream_t s) {
    const uint32_t w = (uint32_t)(byte & 0xff) * 0x01010101u;
    pdl_launch(k_fill, fill_grid(bytes), 256, 0, s, (uint8_t *)p, w, bytes);
}
void dev_copy(void *dst, const void *src, size_t bytes, cudaStream_t s) {
    pdl_launch(k_copy, fill_grid(bytes), 256, 0, s, (uint8_t *)dst, (const uint8_t *)src, bytes);
}

void zero_many(Ctx &c, std::initializer_list<std::pair<void *, int64_t>> bufs,
               std::initializer_list<std::pair<void *, int64_t>> more) {
    ZeroSet z;
    int n = 0;
    int64_t mx = 0;
    for (const auto *set : {&bufs, &more})
        for (const auto &b : *set) {
            if (b.second <= 0 || !b.first) continue;
            if (n == kZeroMax) throw Error{DHGP_ERR_CUDA, "zero_many: too many buffers"};
            z.p[n] = b.first;
            z.bytes[n] = b.second;
            mx = std::max(mx, b.second);
            n++;
        }
    if (n == 0) return;
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(mx / 4, 256), 64));
    pdl_launch(k_zero_many, dim3(gx, n), 256, 0, c.stream, z);
    DHGP_LAUNCHED(c);
}

// ===========================================================================
// fills and the stable transpose
// ===========================================================================
namespace {
__global__ void k_iota(int32_t *p, int64_t n) {
    pdl_entry();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = (int32_t)i;
}
__global__ void k_fill32(int32_t *p, int32_t v, int64_t n) {
    pdl_entry();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}
__global__ void k_fill64(int64_t *p, int64_t v, int64_t n) {
    pdl_entry();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}
// per pin: key = node id, val = edge id (pins enumerated in edge order)
__global__ void k_expand_pairs(int64_t nseg, const int64_t *off, const int32_t *dat, uint64_t *keys,
                               uint32_t *vals, int32_t *node_count) {
    pdl_entry();
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nseg) return;
    int64_t lo = off[e] - off[0], hi = off[e + 1] - off[0];
    for (int64_t p = lo; p < hi; p++) {
        int32_t n = dat[p];
        keys[p] = (uint64_t)(uint32_t)n;
        vals[p] = (uint32_t)e;
        atomicAdd(&node_count[n], 1);
    }
}
__global__ void k_u32_to_i32(const uint32_t *a, int32_t *b, int64_t n) {
    pdl_entry();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = (int32_t)a[i];
}
}  // namespace

void iota_i32(Ctx &c, int32_t *p, int64_t n) {
    if (n <= 0) return;
    pdl_launch(k_iota, (unsigned)cdiv(n, 256), 256, 0, c.stream, p, n);
    DHGP_LAUNCHED(c);
}
void fill_i32(Ctx &c, int32_t *p, int32_t v, int64_t n) {
    if (n <= 0) return;
    pdl_launch(k_fill32, (unsigned)cdiv(n, 256), 256, 0, c.stream, p, v, n);
    DHGP_LAUNCHED(c);
}
void fill_i64(Ctx &c, int64_t *p, int64_t v, int64_t n) {
    if (n <= 0) return;
    pdl_launch(k_fill64, (unsigned)cdiv(n, 256), 256, 0, c.stream, p, v, n);
    DHGP_LAUNCHED(c);
}

void transpose_csr(Ctx &c, int64_t nseg, int32_t N, const int64_t *off, const int32_t *dat, int64_t nnz,
                   int64_t *out_off, int32_t *out_dat) {
    KScope ks(c, "transpose");
    int32_t *cnt = c.alloc<int32_t>(N > 0 ? N : 1);
    c.zero(cnt, N);
    if (nnz == 0) {
        scan_excl<int32_t>(c, cnt, out_off, N);
        c.free(cnt);
        return;
    }
    uint64_t *k = c.alloc<uint64_t>(nnz), *kt = c.alloc<uint64_t>(nnz);
    uint32_t *v = c.alloc<uint32_t>(nnz), *vt = c.alloc<uint32_t>(nnz);
    pdl_launch(k_expand_pairs, (unsigned)cdiv(nseg, 256), 256, 0, c.stream, nseg, off, dat, k, v, cnt);
    DHGP_LAUNCHED(c);
    radix_sort_pairs(c, k, v, kt, vt, nnz, nullptr, bitlen((uint64_t)(N > 0 ? N - 1 : 0)));
    pdl_launch(k_u32_to_i32, (unsigned)cdiv(nnz, 256), 256, 0, c.stream, v, out_dat, nnz);
    DHGP_LAUNCHED(c);
    scan_excl<int32_t>(c, cnt, out_off, N);
    c.free(cnt);
    c.free(k);
    c.free(kt);
    c.free(v);
    c.free(vt);
}

}  // namespace dhgp
