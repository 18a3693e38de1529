// prims.cuh — hand-written sm_100a building blocks: scans, a stable LSD radix
// sort, tiered per-segment sorts and sorted-set merges.  All integer, all
// deterministic.
#pragma once
#include <initializer_list>
#include <utility>
#include "common.cuh"

namespace dhgp {

// out[0..n]: exclusive prefix sums of in[0..n-1]; out[n] = total.
template <class T>
void scan_excl(Ctx &c, const T *in, int64_t *out, int64_t n);
// two or three independent exclusive scans of length n in one launch
// (in2 == nullptr: two)
template <class T>
void scan_excl3(Ctx &c, const T *in0, int64_t *out0, const T *in1, int64_t *out1, const T *in2, int64_t *out2,
                int64_t n);
// out[k] = max(in[0..k]) (inclusive running maximum), int64.
void scan_incl_max(Ctx &c, const int64_t *in, int64_t *out, int64_t n);

// Stable LSD radix sort of (key, val) pairs on key bits [0, bits).
// n = *d_n when d_n != nullptr (device-resident count, <= n_cap), else n_cap.
// Sorted output ends in (keys, vals); (ktmp, vtmp) are scratch of n_cap.
void radix_sort_pairs(Ctx &c, uint64_t *keys, uint32_t *vals, uint64_t *ktmp, uint32_t *vtmp, int64_t n_cap,
                      const int64_t *d_n, int bits);

// Sort of (key, val) pairs by (key, val) (for distinct vals ascending in the
// input this is the stable key order): CTA chunk sorts + merge-path passes,
// for the mid-size sorts of the refinement rounds (n up to ~1M).
void merge_sort_pairs(Ctx &c, uint64_t *keys, uint32_t *vals, uint64_t *ktmp, uint32_t *vtmp, int64_t n);
constexpr int64_t kMergeSortMax = 1 << 20;

// Single-CTA sort of (key, val) pairs by (key, val) for n <= kSmallSort
// (one launch; not stable in general, stable when vals ascend in input order
// and are distinct).
constexpr int64_t kSmallSort = 4096;
// up to eight zero-fills (pointer, bytes; 4-byte aligned) in one launch
using ZeroSpan = std::pair<void *, int64_t>;  // (pointer, bytes)
void zero_many(Ctx &c, std::initializer_list<ZeroSpan> bufs, std::initializer_list<ZeroSpan> more = {});
// the same for unique keys carrying their value in the low 32 bits
// dn != null: the count is read on device (n ignored); no-op above kSmallSort
void small_sort_packed(Ctx &c, uint64_t *keys, uint32_t *vals, int64_t n, const int64_t *dn = nullptr);
void small_sort_pairs(Ctx &c, uint64_t *keys, uint32_t *vals, int64_t n);

// Per-segment ascending sort of (map ? map[dat[i]] : dat[i]) into tmp (same
// layout as dat).  Segments longer than kMaxSegSort raise DHGP_ERR_UNSUPPORTED.
constexpr int64_t kMaxSegSort = 8192;
void seg_sort(Ctx &c, int64_t nseg, const int64_t *off, const int32_t *dat, const int32_t *map, int32_t *tmp);

// cnt[s] = number of distinct values in sorted segment s of tmp.
void seg_unique_count(Ctx &c, int64_t nseg, const int64_t *off, const int32_t *tmp, int64_t *cnt);
// out[out_off[s]..] = distinct values of sorted segment s.
void seg_unique_write(Ctx &c, int64_t nseg, const int64_t *off, const int32_t *tmp, const int64_t *out_off,
                      int32_t *out);

// Sorted-set union of two member lists per coarse node.  The count variant
// takes the node count from device memory (d_nc) when given; nc is then the
// capacity and cnt[d_nc..nc) is zeroed.
// Unions of more than 2048 elements go to a block-per-node kernel through
// big_list (filled by the count call, reused by the write call).
void merge_union_count2(Ctx &c, int64_t nc, const int32_t *ma, const int32_t *mb, const int64_t *off0,
                        const int32_t *dat0, int64_t *cnt0, int32_t *big0, int32_t *bigc0, const int64_t *off1,
                        const int32_t *dat1, int64_t *cnt1, int32_t *big1, int32_t *bigc1, const int64_t *d_nc);
void merge_union_write2(Ctx &c, int64_t nc, const int32_t *ma, const int32_t *mb, const int64_t *off0,
                        const int32_t *dat0, const int64_t *out_off0, int32_t *out0, int32_t *big0, int32_t *bigc0,
                        const int64_t *off1, const int32_t *dat1, const int64_t *out_off1, int32_t *out1,
                        int32_t *big1, int32_t *bigc1);

// Simple fills.
void iota_i32(Ctx &c, int32_t *p, int64_t n);
void fill_i32(Ctx &c, int32_t *p, int32_t v, int64_t n);
void fill_i64(Ctx &c, int64_t *p, int64_t v, int64_t n);

// Transpose edge -> node lists into node -> ascending edge lists (stable).
// out_off[N+1], out_dat[nnz].
void transpose_csr(Ctx &c, int64_t nseg, int32_t N, const int64_t *off, const int32_t *dat, int64_t nnz,
                   int64_t *out_off, int32_t *out_dat);

}  // namespace dhgp
