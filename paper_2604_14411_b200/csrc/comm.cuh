// comm.cuh — node-range sharding across ranks.
//
// One process per GPU.  Every rank holds a replica of every level (the
// contraction, the sequence gains and the event pipeline run replicated and
// are deterministic); the per-node phases — candidate scoring (A4-A6) and
// move proposals (A14) — are computed for this rank's contiguous node range
// only and completed by an in-place allgather of their outputs.
// The exchanged values are exact integers / f64 and every later tie-break is
// the reference's global total order, so the result is bit-identical to the
// single-GPU run at any world size.
#pragma once
#include "common.cuh"

namespace dhgp {

struct Comm {
    int world = 1, rank = 0, device = 0;
    int kind = 0;                 // DHGP_COMM_NCCL or DHGP_COMM_HOST
    void *nccl = nullptr;         // ncclComm_t (libnccl.so.2, resolved at run time)
    dhgp_allgather_fn fn = nullptr;
    void *user = nullptr;
    void *pinned = nullptr;       // host staging for DHGP_COMM_HOST
    size_t pinned_cap = 0;
    int64_t min_units = 1 << 16;  // phases over fewer units run replicated (no exchange)
    bool exercise = false;        // world 1: still issue the exchanges (DHGP_COMM_EXERCISE=1, tests)
    int64_t calls = 0;            // allgathers issued
    double bytes = 0;             // bytes received per rank
};

// This rank's share [lo, hi) of n units; chunk = ceil(n / world).  `on` is
// false (lo = 0, hi = n) when there is no communicator or n < min_units.
struct Shard {
    bool on = false;
    int64_t lo = 0, hi = 0, chunk = 0;
};
Shard shard_of(const Comm *cm, int64_t n);
// capacity a buffer exchanged over n units needs (world * chunk >= n)
int64_t shard_capacity(const Comm *cm, int64_t n);

// In-place allgather over buf[world * chunk] elements of `elem` bytes; rank r
// contributes buf[r*chunk, (r+1)*chunk).  Stream-ordered on c.stream for
// NCCL; the host mode synchronises and calls the user's allgather.
void allgather(Ctx &c, Comm *cm, void *buf, size_t elem, int64_t chunk);

// Element-wise reduction across ranks of buf[0..n) (every rank ends with the
// result), as an allgather of every rank's whole array followed by an on-device
// reduction in rank order (exact: integer max / sum).  Used for the phases whose
// per-rank outputs overlap: the incremental scoring's per-node best tuple key
// (max) and the in-sequence gain / inbound-crossing terms of each move (sum).
void allreduce_max_u64(Ctx &c, Comm *cm, unsigned long long *buf, int64_t n);
void allreduce_sum_i64(Ctx &c, Comm *cm, long long *buf, int64_t n);
void allreduce_sum_i32(Ctx &c, Comm *cm, int32_t *buf, int64_t n);
// is the communicator live (world > 1, or exercised at world 1)?
inline bool comm_active(const Comm *cm) { return cm && (cm->world > 1 || cm->exercise); }

}  // namespace dhgp
