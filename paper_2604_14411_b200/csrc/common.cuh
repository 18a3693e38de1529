// common.cuh — shared device/host utilities for libdhgp (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "../../include/dhgp.h"

namespace dhgp {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
struct Error {
    int code;
    std::string msg;
};

void set_error(int code, const std::string &msg);
const char *last_error();

#define DHGP_CUDA(call)                                                                              \
    do {                                                                                             \
        cudaError_t _e = (call);                                                                     \
        if (_e != cudaSuccess) {                                                                     \
            throw ::dhgp::Error{DHGP_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e) + \
                                                   " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"}; \
        }                                                                                            \
    } while (0)

#define DHGP_LAUNCHED(ctx)                                                                           \
    do {                                                                                             \
        cudaError_t _e = cudaGetLastError();                                                         \
        if (_e != cudaSuccess)                                                                       \
            throw ::dhgp::Error{DHGP_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(_e) + \
                                                   " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"}; \
        (ctx).launches++;                                                                            \
    } while (0)

// ---------------------------------------------------------------------------
// Programmatic dependent launch.  Every kernel is launched with programmatic
// stream serialization, so the next kernel's launch is processed while this
// one drains (hiding part of the launch gap of the short dependent kernels
// that make up a level / round).  Each kernel's first statement is
// pdl_entry(): griddepcontrol.wait blocks until the previous grid has
// completed and its writes are visible, so stream order is unchanged for
// every memory access.  No kernel triggers its dependents early
// (griddepcontrol.launch_dependents): a CTA's exit is the trigger.  Triggering
// at entry let the next kernel's CTAs sit resident, waiting, on SMs the
// running kernel still needed — measured 3% slower on C2 and C3.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_entry() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... P, typename... A>
inline void pdl_launch(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, A &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    DHGP_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...));
}
// byte fill / device copy as PDL kernels (prims.cu), so a cudaMemsetAsync /
// cudaMemcpyAsync node does not break the launch overlap of the kernel chain
void dev_fill(void *p, int byte, size_t bytes, cudaStream_t s);
void dev_copy(void *dst, const void *src, size_t bytes, cudaStream_t s);

// ---------------------------------------------------------------------------
// execution context: one stream per call, stream-ordered pool allocations
// ---------------------------------------------------------------------------
struct KernelStat {
    const char *name;
    int64_t launches;
    double ms;
    double bytes;
};

struct Comm;

// Device memory: one arena per device over large cudaMalloc chunks, with a
// best-fit free list (address-ordered, coalescing).  All library work on a
// device runs on one stream in issue order, so a block freed on the host can
// be handed out again at once — the stream orders the old and the new use
// (the semantics of cudaMallocAsync on one stream).  Growing by cudaMalloc
// chunks is ~100x cheaper than growing a stream-ordered pool (measured:
// tests/micro/pool_growth.cu), and the chunks are kept for the process.
void *arena_alloc(int device, size_t bytes);
void arena_free(int device, void *p);

struct Ctx {
    Comm *comm = nullptr;  // node-range sharding across ranks (comm.cuh); null = single GPU
    int device = 0;
    cudaStream_t stream = nullptr;
    // a second stream for independent work forked from `stream` and joined
    // back (fork / join events); see contract_write
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int64_t launches = 0;
    int num_sms = 148;
    // optional per-kernel event timing (bench/profiling only); only the
    // outermost scope of a nest is recorded, so the classes are disjoint
    bool profiling = false;
    int prof_depth = 0;
    // device counters of algorithmic bytes for data-dependent classes
    // (profiling only; slots below), added to their class at flush_profile
    unsigned long long *prof_work = nullptr;
    enum { PW_SEQ_GAINS = 0, PW_RUNS_UPDATE = 1, PW_SELECT = 2, PW_SLOTS = 4 };
    unsigned long long *work_slot(int k) {
        if (!profiling) return nullptr;
        if (!prof_work) {
            prof_work = alloc<unsigned long long>(PW_SLOTS);
            DHGP_CUDA(cudaMemsetAsync(prof_work, 0, PW_SLOTS * sizeof(unsigned long long), stream));
        }
        return prof_work + k;
    }
    std::vector<KernelStat> kstats;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending_ev;
    std::vector<int> pending_idx;
    std::vector<double> pending_bytes;
    // Small device -> host reads (status words, counts) go through a pinned
    // bounce buffer: a cudaMemcpyAsync into pageable memory is staged by the
    // driver and costs several microseconds each, and the refinement round
    // does five of them.  The values land at their destinations in sync().
    static constexpr size_t kPinnedBytes = 1 << 16;
    char *pinned = nullptr;
    size_t pin_used = 0;
    struct PinnedRead {
        void *dst;
        size_t off, bytes;
    };
    std::vector<PinnedRead> pin_reads;

    template <class T>
    T *alloc(int64_t n) {
        const size_t bytes = (size_t)(n > 0 ? n : 1) * sizeof(T);
        return (T *)arena_alloc(device, bytes);
    }
    template <class T>
    void free(T *p) {
        if (p) arena_free(device, (void *)p);
    }
    template <class T>
    void zero(T *p, int64_t n) {
        if (n > 0) {
            dev_fill(p, 0, (size_t)n * sizeof(T), stream);
            launches++;
        }
    }
    template <class T>
    void fill_bytes(T *p, int v, int64_t n) {
        if (n > 0) {
            dev_fill(p, v, (size_t)n * sizeof(T), stream);
            launches++;
        }
    }
    template <class T>
    void h2d(T *d, const T *h, int64_t n) {
        if (n > 0) DHGP_CUDA(cudaMemcpyAsync(d, h, (size_t)n * sizeof(T), cudaMemcpyHostToDevice, stream));
    }
    template <class T>
    void d2h(T *h, const T *d, int64_t n) {
        if (n <= 0) return;
        const size_t bytes = (size_t)n * sizeof(T);
        if (pinned && bytes <= 4096) {
            if (pin_used + bytes > kPinnedBytes) sync();
            DHGP_CUDA(cudaMemcpyAsync(pinned + pin_used, d, bytes, cudaMemcpyDeviceToHost, stream));
            pin_reads.push_back(PinnedRead{(void *)h, pin_used, bytes});
            pin_used += (bytes + 15) & ~(size_t)15;
            return;
        }
        DHGP_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, stream));
    }
    template <class T>
    void d2d(T *dst, const T *src, int64_t n) {
        if (n > 0) {
            dev_copy(dst, src, (size_t)n * sizeof(T), stream);
            launches++;
        }
    }
    // diagnostics: host time blocked in sync() and the number of syncs
    double sync_wait_ms = 0.0;
    int64_t syncs = 0;
    void sync() {
        const auto t0 = std::chrono::steady_clock::now();
        DHGP_CUDA(cudaStreamSynchronize(stream));
        sync_wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        syncs++;
        for (const PinnedRead &r : pin_reads) memcpy(r.dst, pinned + r.off, r.bytes);
        pin_reads.clear();
        pin_used = 0;
    }

    // profiling brackets: kbegin(name) ... kend(bytes)
    int kbegin(const char *name);
    void kend(int idx, double bytes);
    void flush_profile();
};

// DHGP_TRACE=1: every scope is synchronised and printed to stderr as
// "trace <name> <ms> <tag>" (diagnostics only; serialises the stream)
bool trace_enabled();
void trace_print(const char *name, double ms, long long tag);

struct KScope {
    Ctx &c;
    int idx;
    double bytes;
    const char *name;
    long long tag;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    bool nested = false;  // counted in the profiling depth
    KScope(Ctx &ctx, const char *nm, double b = 0, long long tg = -1) : c(ctx), idx(-1), bytes(b), name(nm), tag(tg) {
        if (c.profiling) {
            if (c.prof_depth == 0) idx = c.kbegin(name);
            c.prof_depth++;
            nested = true;
        }
        if (trace_enabled()) {
            cudaEventCreate(&t0);
            cudaEventCreate(&t1);
            cudaEventRecord(t0, c.stream);
        }
    }
    ~KScope() { close(); }
    // records the end now (before a profiling readback that syncs); the
    // measured bytes can be set afterwards with set_bytes
    int stopped = -1;
    void stop() {
        if (idx >= 0) c.kend(idx, bytes);
        stopped = idx;
        idx = -1;
    }
    void set_bytes(double b) {
        if (stopped >= 0)
            c.pending_bytes[stopped] = b;
        else
            bytes = b;
    }
    // ends the scope early (the destructor then does nothing)
    void close() {
        if (idx >= 0) c.kend(idx, bytes);
        idx = -1;
        if (nested) {
            c.prof_depth--;
            nested = false;
        }
        if (t0) {
            cudaEventRecord(t1, c.stream);
            cudaEventSynchronize(t1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, t0, t1);
            trace_print(name, ms, tag);
            cudaEventDestroy(t0);
            cudaEventDestroy(t1);
            t0 = t1 = nullptr;
        }
    }
};

// Escalation thresholds of the tiered per-node kernels (warp -> block ->
// dense).  DHGP_FORCE_TIERS=1 shrinks them so that small parity tests drive
// every tier (=2 keeps the small-K dense path, =1 disables it); results
// never depend on them.
struct Tiers {
    int ss_limit = 720;       // score: distinct neighbours per warp table
    int ss_heavy_inc = 192;   // score: incident h-edges above which a CTA takes the node (full scoring)
    int sm_limit = 2816;      // score: distinct neighbours per 256-thread CTA table (4096 slots)
    int sm_heavy_inc = 512;   // score: incident h-edges above which the 1024-thread tier takes the node
    int ss_list_inc = 80;     // score, list mode (incremental levels): incident h-edges above which a CTA takes the node
    int sh_limit = 12288;     // score: distinct neighbours per block table
    int pr_limit = 400;       // propose: distinct parts per warp table
    int pr_heavy_inc = 64;    // propose: incident h-edges above which a block takes the node
    int pm_limit = 3072;      // propose: distinct parts per medium-tier table
    int small_k = 4096;       // propose: K up to which escalated nodes use dense shared arrays
    int pr_hub_inc = 128;     // propose: incident h-edges above which a node is split over many CTAs
    int edge_movers = 64;     // events / sequence gains: movers per h-edge for the warp tier (<= 64; 2 per lane above 32)
    int seg_smem = 8192;      // per-segment sorts / wide run updates: longest list kept in shared memory
    int mv_block = 2048;      // events / sequence gains: movers per h-edge for the shared-memory block tier
    int speculate = 1;        // refinement: launch a round's tail before its mover count is on the host
    long long fe_min = 32768; // sequence gains / events: mover h-edges from which the flat kernel takes a round
};
const Tiers &tiers();

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
__device__ __forceinline__ int64_t cdiv_dev(int64_t a, int64_t b) { return (a + b - 1) / b; }

// grid for a persistent / grid-stride kernel: resident blocks per SM x SMs
template <class K>
inline int resident_grid(const Ctx &c, K kernel, int threads, size_t smem) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    return per_sm * c.num_sms;
}
inline int bitlen(uint64_t x) {
    int b = 0;
    while (x) {
        b++;
        x >>= 1;
    }
    return b;
}

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
#define FULL_MASK 0xffffffffu

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(FULL_MASK, v, d);
    return v;
}
template <class T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        T o = __shfl_xor_sync(FULL_MASK, v, d);
        v = o > v ? o : v;
    }
    return v;
}
template <class T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        T o = __shfl_xor_sync(FULL_MASK, v, d);
        v = o < v ? o : v;
    }
    return v;
}
// inclusive prefix sum across the warp
template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
    const int lane = lane_id();
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T o = __shfl_up_sync(FULL_MASK, v, d);
        if (lane >= d) v += o;
    }
    return v;
}

// lower bound in sorted a[lo, hi)
template <class T>
__device__ __forceinline__ int64_t lower_bound_dev(const T *a, int64_t lo, int64_t hi, T key) {
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// index of key in strictly increasing a[lo, hi) or -1 (_kernels.pyx:22-32)
__device__ __forceinline__ int64_t bsearch_dev(const int32_t *a, int64_t lo, int64_t hi, int32_t key) {
    int64_t p = lower_bound_dev<int32_t>(a, lo, hi, key);
    return (p < hi && a[p] == key) ? p : -1;
}

// In-register warp bitonic sort of 32*K unsigned keys (ascending); element
// index of v[k] on lane l is k*32 + l.
template <int K>
__device__ __forceinline__ void warp_bitonic_sort(uint32_t (&v)[K]) {
    const int lane = lane_id();
#pragma unroll
    for (int size = 2; size <= 32 * K; size <<= 1) {
#pragma unroll
        for (int j = size >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                const int jk = j >> 5;
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const int partner = k ^ jk;
                    if (partner > k) {
                        const int idx = k * 32 + lane;
                        const bool asc = (idx & size) == 0;
                        uint32_t a = v[k], b = v[partner];
                        if ((a > b) == asc) {
                            v[k] = b;
                            v[partner] = a;
                        }
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const int idx = k * 32 + lane;
                    uint32_t o = __shfl_xor_sync(FULL_MASK, v[k], j);
                    const bool asc = (idx & size) == 0;
                    const bool lower = (idx & j) == 0;
                    v[k] = (lower == asc) ? min(v[k], o) : max(v[k], o);
                }
            }
        }
    }
}

// 64-bit keyed variant (key in high bits, payload in low bits of one u64)
template <int K>
__device__ __forceinline__ void warp_bitonic_sort64(uint64_t (&v)[K]) {
    const int lane = lane_id();
#pragma unroll
    for (int size = 2; size <= 32 * K; size <<= 1) {
#pragma unroll
        for (int j = size >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                const int jk = j >> 5;
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const int partner = k ^ jk;
                    if (partner > k) {
                        const int idx = k * 32 + lane;
                        const bool asc = (idx & size) == 0;
                        uint64_t a = v[k], b = v[partner];
                        if ((a > b) == asc) {
                            v[k] = b;
                            v[partner] = a;
                        }
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < K; k++) {
                    const int idx = k * 32 + lane;
                    uint64_t o = __shfl_xor_sync(FULL_MASK, v[k], j);
                    const bool asc = (idx & size) == 0;
                    const bool lower = (idx & j) == 0;
                    v[k] = (lower == asc) ? (v[k] < o ? v[k] : o) : (v[k] > o ? v[k] : o);
                }
            }
        }
    }
}

// Sorts n <= 4096 u64 keys ascending with one 1024-thread CTA: each warp
// sorts a 128-key run in registers, then runs of 128..2048 are merged
// pairwise by co-ranks — a key's output slot is its offset in its run plus
// its rank in the partner run (lower bound for the first run's keys, upper
// bound for the second's, so ties keep run order).  `a` holds the input and
// receives the output; `b` is scratch; both have room for 4096 keys.
__device__ __forceinline__ int rank_in_run(const uint64_t *r, int len, uint64_t x, bool upper) {
    int lo = 0, hi = len;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (upper ? (r[mid] <= x) : (r[mid] < x))
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}
__device__ __forceinline__ void block_sort_u64_4096(uint64_t *a, uint64_t *b, int n) {
    const int t = threadIdx.x, lane = lane_id(), w = warp_id();
    int np = 128;
    while (np < n) np <<= 1;
    if (w * 128 < np) {
        uint64_t v[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int idx = w * 128 + k * 32 + lane;
            v[k] = idx < n ? a[idx] : ~0ull;
        }
        warp_bitonic_sort64<4>(v);
#pragma unroll
        for (int k = 0; k < 4; k++) b[w * 128 + k * 32 + lane] = v[k];
    }
    __syncthreads();
    uint64_t *src = b, *dst = a;
    for (int run = 128; run < np; run <<= 1) {
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int i = q * 1024 + t;
            if (i < np) {
                const int ps = i & ~(2 * run - 1);
                const bool first = (i & run) == 0;
                const uint64_t x = src[i];
                const int r = first ? rank_in_run(src + ps + run, run, x, false) : rank_in_run(src + ps, run, x, true);
                dst[ps + (i - ps - (first ? 0 : run)) + r] = x;
            }
        }
        __syncthreads();
        uint64_t *tmp = src;
        src = dst;
        dst = tmp;
    }
    if (src != a) {
        for (int i = t; i < np; i += blockDim.x) a[i] = src[i];
        __syncthreads();
    }
}

// block-wide bitonic sort of n_pow2 u64 keys in shared memory (ascending)
__device__ __forceinline__ void block_bitonic_sort64(uint64_t *s, int n_pow2) {
    for (int size = 2; size <= n_pow2; size <<= 1) {
        for (int j = size >> 1; j > 0; j >>= 1) {
            __syncthreads();
            for (int t = threadIdx.x; t < (n_pow2 >> 1); t += blockDim.x) {
                int lo = 2 * j * (t / j) + (t % j);
                int hi = lo + j;
                bool asc = (lo & size) == 0;
                uint64_t a = s[lo], b = s[hi];
                if ((a > b) == asc) {
                    s[lo] = b;
                    s[hi] = a;
                }
            }
        }
    }
    __syncthreads();
}
__device__ __forceinline__ void block_bitonic_sort32(uint32_t *s, int n_pow2) {
    for (int size = 2; size <= n_pow2; size <<= 1) {
        for (int j = size >> 1; j > 0; j >>= 1) {
            __syncthreads();
            for (int t = threadIdx.x; t < (n_pow2 >> 1); t += blockDim.x) {
                int lo = 2 * j * (t / j) + (t % j);
                int hi = lo + j;
                bool asc = (lo & size) == 0;
                uint32_t a = s[lo], b = s[hi];
                if ((a > b) == asc) {
                    s[lo] = b;
                    s[hi] = a;
                }
            }
        }
    }
    __syncthreads();
}

// In-place ascending sort of s[0..n) for any n, by the block, in any memory
// (segments too long for shared memory sort in global memory).  The network
// is the bitonic sorter written with ascending comparators only (each merge
// first compares i with its mirror in the block, then half-cleans), so a
// virtual +inf padding up to the next power of two never moves and every
// comparator touching an index >= n is skipped.
template <class T>
__device__ __forceinline__ void block_sort_asc_any(T *s, int64_t n) {
    int64_t np = 1;
    while (np < n) np <<= 1;
    for (int64_t size = 2; size <= np; size <<= 1) {
        for (int64_t j = size >> 1; j > 0; j >>= 1) {
            __syncthreads();
            for (int64_t t = threadIdx.x; t < (np >> 1); t += blockDim.x) {
                const int64_t blk = t / j, off = t % j;
                const int64_t lo = 2 * j * blk + off;
                // first step of a merge: mirror partner; later steps: +j
                const int64_t hi = (j == (size >> 1)) ? (lo - off) + (2 * j - 1 - off) : lo + j;
                if (hi >= n) continue;
                const T a = s[lo], b = s[hi];
                if (b < a) {
                    s[lo] = b;
                    s[hi] = a;
                }
            }
        }
    }
    __syncthreads();
}

// Early-exit flags shared by the threads of a block (a table overflowed):
// set and polled with atomic read-modify-writes (race-free, and seen as such
// by compute-sanitizer racecheck).  The hash loops poll only on a long probe
// chain — the case a full table produces — so the common insert pays
// nothing; the authoritative read follows a barrier.
__device__ __forceinline__ int32_t flag_get(int32_t *f) { return atomicOr(f, 0); }
__device__ __forceinline__ void flag_set(int32_t *f) { atomicExch(f, 1); }
constexpr int kFlagPoll = 16;  // probes between polls of the overflow flag

__host__ __device__ __forceinline__ int next_pow2(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

// block reduce (sum) helpers; `sh` must hold >= 32 elements
template <class T>
__device__ __forceinline__ T block_sum(T v, T *sh) {
    v = warp_sum(v);
    __syncthreads();
    if (lane_id() == 0) sh[warp_id()] = v;
    __syncthreads();
    T r = 0;
    if (warp_id() == 0) {
        r = (lane_id() < (int)(blockDim.x >> 5)) ? sh[lane_id()] : (T)0;
        r = warp_sum(r);
    }
    return r;  // valid in thread 0
}

}  // namespace dhgp
