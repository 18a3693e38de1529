// baselines.cu — the reference's comparison partitioners on the GPU
// (baselines.py:16-91): `one_pass` and `overlap_greedy`, bit-identical.
//
// Both are greedy and sequential by definition (each decision depends on the
// running partition), so each runs as ONE persistent kernel — a warp for
// one_pass, a 1024-thread CTA for overlap_greedy — with no host round trips;
// the parallelism is inside a decision (a node's inbound list, the frontier
// of candidates).  State lives in HBM as bitmaps over h-edges plus lists of
// the set bits, so resetting a partition costs its own size, not E.
//   one_pass: O(N + S_in) work, N sequential steps.
//   overlap_greedy: overlap counts are maintained incrementally — when an
//   h-edge joins the partition's incident set, every free pin of it gains 1
//   (ov = |inc(m) ∩ inc_u|, baselines.py:74) — and the next node is the
//   frontier's argmax by (overlap desc, id asc) that passes the size and
//   inbound-union bounds (a node failing them keeps failing: both only grow).
#include <mutex>

#include "graph.cuh"
#include "prims.cuh"

namespace dhgp {

void seams_setup(Ctx &c, int device);
std::recursive_mutex &device_mutex(int device);

namespace {

__device__ __forceinline__ bool bit_get(const uint32_t *b, int32_t e) { return (b[e >> 5] >> (e & 31)) & 1u; }
// sets the bit; true when it was clear
__device__ __forceinline__ bool bit_set(uint32_t *b, int32_t e) {
    const uint32_t m = 1u << (e & 31);
    return !(atomicOr(&b[e >> 5], m) & m);
}

// one_pass (baselines.py:16-40): nodes in id order fill one open partition;
// a node that would break the size bound or the distinct-inbound bound
// opens the next one.  One warp; the inbound union is a bitmap over h-edges.
__global__ void k_one_pass(int32_t N, const int32_t *size, const int64_t *in_off, const int32_t *in_dat,
                           int64_t omega, int64_t delta, uint32_t *bits, int32_t *list, int32_t *assign,
                           int32_t *num_parts) {
    pdl_entry();
    const int lane = lane_id();
    const uint32_t lt = (1u << lane) - 1u;
    int32_t cur = -1;
    int64_t cur_size = 0, cur_cnt = 0;
    int64_t nlist = 0;
    for (int32_t v = 0; v < N; v++) {
        const int64_t s = size[v];
        const int64_t lo = in_off[v], hi = in_off[v + 1];
        int64_t fresh = 0;  // |in(v) \ cur_in| (in(v) is sorted unique)
        for (int64_t j = lo + lane; j < hi; j += 32) fresh += !bit_get(bits, in_dat[j]);
        fresh = warp_sum(fresh);
        const bool fits = cur >= 0 && cur_size + s <= omega && cur_cnt + fresh <= delta;
        if (!fits) {  // open the next partition: clear the union
            for (int64_t j = lane; j < nlist; j += 32) {
                const int32_t e = list[j];
                bits[e >> 5] = 0u;
            }
            __syncwarp();
            nlist = 0;
            cur++;
            cur_size = 0;
            cur_cnt = 0;
            fresh = hi - lo;
        }
        cur_size += s;
        cur_cnt += fresh;
        for (int64_t b = lo; b < hi; b += 32) {
            const int64_t j = b + lane;
            bool added = false;
            int32_t e = 0;
            if (j < hi) {
                e = in_dat[j];
                added = bit_set(bits, e);
            }
            const uint32_t bal = __ballot_sync(FULL_MASK, added);
            if (added) list[nlist + __popc(bal & lt)] = e;
            nlist += __popc(bal);
        }
        __syncwarp();
        if (lane == 0) assign[v] = cur;
    }
    if (lane == 0) *num_parts = cur + 1;
}

// overlap_greedy (baselines.py:43-91), one CTA.  Per partition: inc_u /
// in_u as bitmaps (+ lists of their set bits for the reset), ov[m] for the
// frontier (free nodes with an incident h-edge in inc_u, listed in `front`),
// `excl` for frontier nodes that failed a bound.
constexpr int OG_T = 1024;
struct OgState {
    uint32_t *inc_bits, *in_bits;
    int32_t *inc_list, *in_list;
    int32_t *ov, *front;
    uint8_t *excl;
};
__global__ void __launch_bounds__(OG_T) k_overlap_greedy(int32_t N, const int32_t *size, const int64_t *in_off,
                                                         const int32_t *in_dat, const int64_t *inc_off,
                                                         const int32_t *inc_dat, const int64_t *pin_off,
                                                         const int32_t *pin_dat, int64_t omega, int64_t delta,
                                                         OgState s, int32_t *assign, int32_t *num_parts) {
    pdl_entry();
    __shared__ int64_t s_in_cnt;
    __shared__ int32_t s_ninc, s_nin, s_nfront;
    __shared__ long long r_key[OG_T / 32];
    __shared__ int64_t r_cnt[OG_T / 32];
    __shared__ int s_ok;
    const int t = threadIdx.x, lane = lane_id(), w = warp_id();
    if (t == 0) {
        s_in_cnt = 0;
        s_ninc = s_nin = s_nfront = 0;
    }
    __syncthreads();
    // adds node b to the open partition: its in-edges to in_u, its incident
    // h-edges to inc_u and their free pins' overlaps (+1 per new h-edge)
    auto add = [&](int32_t b) {
        for (int64_t j = in_off[b] + t; j < in_off[b + 1]; j += OG_T) {
            const int32_t e = in_dat[j];
            if (bit_set(s.in_bits, e)) {
                s.in_list[atomicAdd(&s_nin, 1)] = e;
                atomicAdd((unsigned long long *)&s_in_cnt, 1ull);
            }
        }
        for (int64_t j = inc_off[b] + t; j < inc_off[b + 1]; j += OG_T) {
            const int32_t e = inc_dat[j];
            if (!bit_set(s.inc_bits, e)) continue;
            s.inc_list[atomicAdd(&s_ninc, 1)] = e;
            for (int64_t q = pin_off[e]; q < pin_off[e + 1]; q++) {
                const int32_t m = pin_dat[q];
                if (assign[m] >= 0) continue;
                if (atomicAdd(&s.ov[m], 1) == 0) s.front[atomicAdd(&s_nfront, 1)] = m;
            }
        }
        __syncthreads();
    };
    int32_t part = -1;
    for (int32_t seed = 0; seed < N; seed++) {
        if (assign[seed] >= 0) continue;  // uniform: written by thread 0 before a barrier
        part++;
        __syncthreads();
        if (t == 0) assign[seed] = part;
        __syncthreads();
        int64_t psize = size[seed];
        add(seed);
        while (true) {
            // best frontier candidate by (overlap desc, id asc) within the size bound
            const int nf = s_nfront;
            long long key = -1;  // ov << 32 | (2^31 - 1 - m): larger = better
            for (int i = t; i < nf; i += OG_T) {
                const int32_t m = s.front[i];
                if (assign[m] >= 0 || s.excl[m]) continue;
                const int32_t o = s.ov[m];
                if (o <= 0 || psize + size[m] > omega) continue;
                const long long k = ((long long)o << 32) | (long long)(0x7fffffff - m);
                if (k > key) key = k;
            }
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                const long long o = __shfl_xor_sync(FULL_MASK, key, d);
                if (o > key) key = o;
            }
            if (lane == 0) r_key[w] = key;
            __syncthreads();
            long long best = r_key[0];
            for (int j = 1; j < OG_T / 32; j++) best = max(best, r_key[j]);
            __syncthreads();
            if (best < 0) break;
            const int32_t m = 0x7fffffff - (int32_t)(best & 0xffffffffll);
            // inbound union |in_u ∪ in(m)| <= delta (baselines.py:80)
            int64_t fresh = 0;
            for (int64_t j = in_off[m] + t; j < in_off[m + 1]; j += OG_T) fresh += !bit_get(s.in_bits, in_dat[j]);
            fresh = warp_sum(fresh);
            if (lane == 0) r_cnt[w] = fresh;
            __syncthreads();
            if (t == 0) {
                int64_t tot = 0;
                for (int j = 0; j < OG_T / 32; j++) tot += r_cnt[j];
                s_ok = s_in_cnt + tot <= delta;
                if (s_ok)
                    assign[m] = part;
                else
                    s.excl[m] = 1;  // in_u and the size only grow: it stays out
            }
            __syncthreads();
            if (s_ok) {
                psize += size[m];
                add(m);
            }
        }
        // reset the partition's state through its lists
        const int nf = s_nfront, ni = s_ninc, nn = s_nin;
        for (int i = t; i < nf; i += OG_T) {
            const int32_t m = s.front[i];
            s.ov[m] = 0;
            s.excl[m] = 0;
        }
        for (int i = t; i < ni; i += OG_T) s.inc_bits[s.inc_list[i] >> 5] = 0u;
        for (int i = t; i < nn; i += OG_T) s.in_bits[s.in_list[i] >> 5] = 0u;
        __syncthreads();
        if (t == 0) {
            s_in_cnt = 0;
            s_ninc = s_nin = s_nfront = 0;
        }
        __syncthreads();
    }
    if (t == 0) *num_parts = part + 1;
}

}  // namespace

}  // namespace dhgp

using namespace dhgp;

extern "C" {

int dhgp_baseline(const dhgp_graph *g, int64_t max_size, int64_t max_inbound, int32_t method, int32_t device,
                  int32_t *assign_out, int32_t *num_parts_out) {
    std::lock_guard<std::recursive_mutex> lk(device_mutex(device));
    try {
        Ctx c;
        seams_setup(c, device);
        if (!g || !assign_out || !num_parts_out || (method != 0 && method != 1))
            throw Error{DHGP_ERR_ARG, "bad arguments to dhgp_baseline"};
        // check_feasibility (hgraph.py:376-401), as both baselines start with it
        if (max_size < 1) throw Error{DHGP_ERR_INFEASIBLE, "max_size must be >= 1, got " + std::to_string(max_size)};
        if (max_inbound < 0)
            throw Error{DHGP_ERR_INFEASIBLE, "max_inbound must be >= 0, got " + std::to_string(max_inbound)};
        DInput in;
        upload_input(c, *g, in);
        DLevel L;
        build_level0(c, in, L);
        const int32_t N = L.N, E = L.E;
        if (N > 0) {
            int32_t bs = -1, bi = -1;
            feasibility(c, L, max_size, max_inbound, &bs, &bi);
            if (bs >= 0 || bi >= 0) {
                std::string msg;
                if (bs >= 0) {
                    int32_t sz;
                    c.d2h(&sz, L.size + bs, 1);
                    c.sync();
                    msg = "node " + std::to_string(bs) + " has size " + std::to_string(sz) + " > max_size " +
                          std::to_string(max_size);
                } else {
                    int64_t o[2];
                    c.d2h(o, L.in_off + bi, 2);
                    c.sync();
                    msg = "node " + std::to_string(bi) + " has " + std::to_string(o[1] - o[0]) +
                          " inbound edges > max_inbound " + std::to_string(max_inbound);
                }
                L.release(c);
                in.release(c);
                throw Error{DHGP_ERR_INFEASIBLE, msg};
            }
        }
        int32_t *assign = c.alloc<int32_t>(N), *np = c.alloc<int32_t>(1);
        const int64_t words = (int64_t)E / 32 + 1;
        c.zero(np, 1);
        if (N > 0 && method == 0) {
            uint32_t *bits = c.alloc<uint32_t>(words);
            int32_t *list = c.alloc<int32_t>(E);
            c.zero(bits, words);
            pdl_launch(k_one_pass, 1, 32, 0, c.stream, N, L.size, L.in_off, L.in_dat, max_size, max_inbound, bits, list,
                                               assign, np);
            DHGP_LAUNCHED(c);
            c.free(bits);
            c.free(list);
        } else if (N > 0) {
            OgState s;
            s.inc_bits = c.alloc<uint32_t>(words);
            s.in_bits = c.alloc<uint32_t>(words);
            s.inc_list = c.alloc<int32_t>(E);
            s.in_list = c.alloc<int32_t>(E);
            s.ov = c.alloc<int32_t>(N);
            s.front = c.alloc<int32_t>(N);
            s.excl = c.alloc<uint8_t>(N);
            c.zero(s.inc_bits, words);
            c.zero(s.in_bits, words);
            c.zero(s.ov, N);
            c.zero(s.excl, N);
            fill_i32(c, assign, -1, N);
            pdl_launch(k_overlap_greedy, 1, OG_T, 0, c.stream, N, L.size, L.in_off, L.in_dat, L.inc_off, L.inc_dat, L.pin_off,
                                                     L.pin_dat, max_size, max_inbound, s, assign, np);
            DHGP_LAUNCHED(c);
            for (void *p : {(void *)s.inc_bits, (void *)s.in_bits, (void *)s.inc_list, (void *)s.in_list,
                            (void *)s.ov, (void *)s.front, (void *)s.excl})
                c.free(p);
        }
        if (N > 0) c.d2h(assign_out, assign, N);
        c.d2h(num_parts_out, np, 1);
        c.sync();
        c.free(assign);
        c.free(np);
        L.release(c);
        in.release(c);
        c.sync();
    } catch (const Error &e) {
        set_error(e.code, e.msg);
        return e.code;
    } catch (const std::exception &e) {
        set_error(DHGP_ERR_CUDA, e.what());
        return DHGP_ERR_CUDA;
    }
    return DHGP_OK;
}

}  // extern "C"
