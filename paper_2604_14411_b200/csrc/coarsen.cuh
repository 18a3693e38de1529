// coarsen.cuh — one coarsening level on device.
#pragma once
#include <vector>

#include "graph.cuh"

namespace dhgp {

// A4+A5+A6 fused: per node, shared-edge-weight histogram over the pins of
// its incident h-edges (never written to HBM), candidates in (hist desc,
// id desc) order, first one passing the size and inbound-union checks.
// coarsen.py:93-132, _kernels.pyx:47-103.  Requires exact-integer weights.
// Scratch for the block tier (nodes with too many distinct neighbours for a
// warp's shared-memory table): dense per-block histograms over all node ids,
// allocated once per partition for the level-0 node count.
struct ScoreScratch {
    int64_t cap = 0;
    int blocks = 0;
    long long *dense = nullptr, *cval = nullptr;
    int32_t *touched = nullptr, *big = nullptr, *heavy = nullptr, *mid = nullptr, *ctr = nullptr;
};
void score_scratch_init(Ctx &c, ScoreScratch &s, int64_t n_cap);
void score_scratch_release(Ctx &c, ScoreScratch &s);
void score_select(Ctx &c, const DLevel &L, const DWeights &W, int64_t omega, int64_t delta, int32_t *pair,
                  double *score, ScoreScratch &s);

// Incremental scoring of the next level.  A node that did not merge keeps
// its histogram entries for every neighbour that did not merge (same h-edges,
// same members) and the size / inbound verdicts for them, so its first valid
// candidate can only change through the new clusters: each merged cluster is
// rescored and its histogram emits (neighbour, cluster, hist) when that
// outranks the neighbour's carried (score, pair); the best such tuple passing
// the inbound-union bound wins, else the carried pair stands.  When the
// carried pair itself merged and no cluster outranks it, the node is
// rescored (its next candidate is unknown).  Bit-identical to score_select.
struct ScoreCarry {
    const int32_t *prev_pair = nullptr;   // previous level's pair / score (previous-level ids)
    const double *prev_score = nullptr;
    const int32_t *gamma_prev = nullptr;  // previous level -> this level
    const int32_t *ma = nullptr;          // this level's node -> its min member (previous-level id)
    const int32_t *mb = nullptr;          // ... -> the other member, -1 if not merged
};
bool score_inc_supported(const Ctx &c, const DWeights &W);
void score_select_inc(Ctx &c, const DLevel &L, const DWeights &W, int64_t omega, int64_t delta, int32_t *pair,
                      double *score, ScoreScratch &s, const ScoreCarry &carry);

// Per-level status words, filled on device and read with ONE host sync.
struct LevelStatus {
    int64_t moved;     // nodes with match != self (= 2 x matched pairs)
    int64_t bad_cert;  // (score, id) monotonicity certificate failed somewhere
    int64_t long_run;  // a run of won claims longer than the walk limit
    int64_t nc, ps, pd, u, sin, uinc;  // coarse sizes
    int64_t pool_top[2];               // node pool: slots in use after this level's unions (pooled mode)
};
constexpr int kStatusWords = 11;

// A7: pseudo-forest -> involution (_kernels.pyx:106-181), no host sync:
// status->moved / bad_cert / long_run are written on device.
void launch_matching(Ctx &c, int32_t N, const int32_t *pair, const double *score, int32_t *match, uint8_t *isrep,
                     int32_t *claim, int64_t *d_status);
// Rare exact fallbacks after the sync (pointer jumping for long runs, the
// reference's sequential cycle check); throws DHGP_ERR_MATCHING on a cycle
// of length != 2.  Returns true when match/isrep were recomputed.
bool matching_fallbacks(Ctx &c, int32_t N, const int32_t *pair, const double *score, int32_t *match,
                        uint8_t *isrep, const int32_t *claim, LevelStatus &st);
// Synchronous form for the kernel seam: returns matched pairs.
int64_t resolve_matching(Ctx &c, int32_t N, const int32_t *pair, const double *score, int32_t *match,
                         uint8_t *isrep);

// A9: contraction (coarsen.py:141-173) in two phases around one host sync:
// contract_count fills fine.gamma, the coarse offsets/sizes and the status
// totals; contract_write materialises the coarse lists once the sizes are
// known on the host.
struct ContractScratch {
    int32_t *ma = nullptr, *mb = nullptr;
    int32_t *tmp_src = nullptr, *tmp_dst = nullptr, *tmp_pin = nullptr;
    int64_t *rank = nullptr;
    int32_t *mlist = nullptr, *mcount = nullptr;  // merged coarse nodes (any order) and their count
    uint8_t *emark = nullptr;  // [E] h-edges holding an absorbed (non-minimum) member
    bool fused = false;  // h-edge lists of <= 128 slots: warp kernels + the linear gap map (no sorted temporaries)
    int32_t *elist = nullptr;  // marked h-edges (emark), ascending ...
    int32_t *ecount = nullptr; // ... and their count
    int64_t *epos = nullptr;   // [E+1] exclusive scan of emark
    unsigned long long *pool_ctr = nullptr;  // pooled mode: pool tops + union shrink (count pass)
};
// With a node pool, the coarse level's per-node lists are pooled: an
// unmerged node keeps its list, a merged cluster's union is appended to the
// pool (reserved in the count pass; the host grows the pool with
// node_pool_fit when the status words show it overflowed); otherwise
// (pool == nullptr) the coarse level gets its own CSR node lists.
void contract_count(Ctx &c, DLevel &fine, const int32_t *match, const uint8_t *isrep, DLevel &coarse,
                    ContractScratch &s, int64_t *d_status, NodePool *pool = nullptr);
void contract_write(Ctx &c, DLevel &fine, DLevel &coarse, ContractScratch &s, const LevelStatus &st,
                    NodePool *pool = nullptr);
// node pool: create from level 0 (its lists move into the pool) and grow so
// that the reserved slots fit (levels' data pointers follow)
void node_pool_init(Ctx &c, NodePool &pool, DLevel &level0, double factor);
void node_pool_fit(Ctx &c, NodePool &pool, const int64_t top[2], std::vector<DLevel> &levels, DLevel *extra);
void contract_release(Ctx &c, ContractScratch &s);
// contract_write leaves s.ma / s.mb (cluster members, for ScoreCarry); the
// caller frees them with this
void contract_release_members(Ctx &c, ContractScratch &s);

// match / isrep of a stored contraction, recovered from its gamma (coarse
// ids are ranks of each cluster's minimum member): used to rebuild levels
// that were not kept during coarsening.
void match_from_gamma(Ctx &c, int32_t N, int32_t nc, const int32_t *gamma, int32_t *match, uint8_t *isrep);
// Drops a level's lists, keeping gamma and the size metadata.
void level_to_stub(Ctx &c, DLevel &L);

}  // namespace dhgp
