// driver.cu — multi-level orchestration and the C-ABI (driver.py:76-163).
#include <chrono>
#include <climits>
#include <cstdlib>
#include <map>
#include <mutex>
#include <unordered_map>

#include "coarsen.cuh"
#include "comm.cuh"
#include "prims.cuh"
#include "ordered.cuh"
#include "refine.cuh"

namespace dhgp {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_last_error;
void set_error(int code, const std::string &msg) {
    (void)code;
    g_last_error = msg;
}
const char *last_error() { return g_last_error.c_str(); }

bool trace_enabled() {
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("DHGP_TRACE");
        on = (e && e[0] == '1') ? 1 : 0;
    }
    return on == 1;
}
const Tiers &tiers() {
    static Tiers t = [] {
        Tiers x;
        const char *e = getenv("DHGP_FORCE_TIERS");
        if (e && (e[0] == '1' || e[0] == '2')) {
            if (e[0] == '1') x.small_k = 0;
            x.ss_limit = 3;
            x.ss_heavy_inc = 2;
            x.sh_limit = 6;
            x.sm_limit = 4;
            x.sm_heavy_inc = 3;
            x.pr_limit = 2;
            x.pr_heavy_inc = 1;
            x.pr_hub_inc = 6;
            x.pm_limit = 3;
            x.edge_movers = e[0] == '1' ? 2 : 40;  // =2: the 33-64 two-per-lane tier up to 40, block above
            x.seg_smem = 48;
            x.mv_block = 6;
            x.speculate = 0;
            x.fe_min = 0;  // every round through the flat kernel (and its deferrals)
        }
        const char *h = getenv("DHGP_HUB_INC");  // tuning: propose hub-tier threshold
        if (h) x.pr_hub_inc = atoi(h);
        if (const char *v = getenv("DHGP_SM_HEAVY_INC")) x.sm_heavy_inc = atoi(v);  // tuning: mid -> 1024-thread tier
        if (const char *v = getenv("DHGP_SS_HEAVY_INC")) x.ss_heavy_inc = atoi(v);  // tuning: warp -> CTA (full scoring)
        if (const char *v = getenv("DHGP_SS_LIST_INC")) x.ss_list_inc = atoi(v);    // tuning: warp -> CTA (list mode)
        if (const char *v = getenv("DHGP_FE_MIN")) x.fe_min = atoll(v);  // tuning: flat round-edges threshold
        return x;
    }();
    return t;
}
void trace_print(const char *name, double ms, long long tag) { fprintf(stderr, "trace %s %.4f %lld\n", name, ms, tag); }

// ---------------------------------------------------------------------------
// per-kernel event timing (bench / profiling only)
// ---------------------------------------------------------------------------
int Ctx::kbegin(const char *name) {
    int idx = -1;
    for (size_t i = 0; i < kstats.size(); i++)
        if (kstats[i].name == name) idx = (int)i;
    if (idx < 0) {
        kstats.push_back(KernelStat{name, 0, 0.0, 0.0});
        idx = (int)kstats.size() - 1;
    }
    cudaEvent_t a, b;
    DHGP_CUDA(cudaEventCreate(&a));
    DHGP_CUDA(cudaEventCreate(&b));
    DHGP_CUDA(cudaEventRecord(a, stream));
    pending_ev.push_back({a, b});
    pending_idx.push_back(idx);
    pending_bytes.push_back(0.0);
    return (int)pending_ev.size() - 1;
}
void Ctx::kend(int p, double bytes) {
    DHGP_CUDA(cudaEventRecord(pending_ev[p].second, stream));
    pending_bytes[p] = bytes;
}
void Ctx::flush_profile() {
    if (prof_work) {  // device-counted bytes of the data-dependent classes
        unsigned long long h[PW_SLOTS];
        DHGP_CUDA(cudaMemcpyAsync(h, prof_work, sizeof h, cudaMemcpyDeviceToHost, stream));
        DHGP_CUDA(cudaStreamSynchronize(stream));
        const char *names[PW_SLOTS] = {"seq_gains", "runs_update", "select", nullptr};
        for (int k = 0; k < PW_SLOTS; k++)
            if (names[k] && h[k])
                for (size_t i = 0; i < pending_idx.size(); i++)
                    if (kstats[pending_idx[i]].name == std::string(names[k])) {
                        pending_bytes[i] += (double)h[k];  // the class total, carried by its first launch
                        break;
                    }
        free(prof_work);
        prof_work = nullptr;
    }
    if (pending_ev.empty()) return;
    DHGP_CUDA(cudaStreamSynchronize(stream));
    for (size_t i = 0; i < pending_ev.size(); i++) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, pending_ev[i].first, pending_ev[i].second);
        KernelStat &k = kstats[pending_idx[i]];
        k.launches++;
        k.ms += ms;
        k.bytes += pending_bytes[i];
        cudaEventDestroy(pending_ev[i].first);
        cudaEventDestroy(pending_ev[i].second);
    }
    pending_ev.clear();
    pending_idx.clear();
    pending_bytes.clear();
}

// ---------------------------------------------------------------------------
// one in-flight call per device: calls on different devices run concurrently;
// the mutex is recursive so that an observer (run on the calling thread while
// the partition is paused at a synchronised point) may call back into the
// library, as the reference allows (its observer gets live objects).
// ---------------------------------------------------------------------------
static std::recursive_mutex g_dev_mu[65];
std::recursive_mutex &device_mutex(int device) { return g_dev_mu[(device >= 0 && device < 64) ? device : 64]; }

// ---------------------------------------------------------------------------
// device arena (common.cuh)
// ---------------------------------------------------------------------------
namespace {
struct Arena {
    std::mutex mu;
    std::map<char *, size_t> chunks;            // base -> bytes
    std::map<char *, size_t> free_by_addr;      // free block -> bytes
    std::multimap<size_t, char *> free_by_size;  // bytes -> free block
    std::unordered_map<char *, size_t> used;     // allocated block -> bytes
    size_t reserved = 0;

    void insert_free(char *p, size_t n) {
        free_by_addr[p] = n;
        free_by_size.emplace(n, p);
    }
    void erase_free(std::map<char *, size_t>::iterator it) {
        auto r = free_by_size.equal_range(it->second);
        for (auto j = r.first; j != r.second; ++j)
            if (j->second == it->first) {
                free_by_size.erase(j);
                break;
            }
        free_by_addr.erase(it);
    }
    char *chunk_end(char *p) {
        auto it = chunks.upper_bound(p);
        --it;
        return it->first + it->second;
    }
    void *alloc(int device, size_t bytes) {
        bytes = (bytes + 255) & ~(size_t)255;
        std::lock_guard<std::mutex> lk(mu);
        auto it = free_by_size.lower_bound(bytes);
        if (it == free_by_size.end()) {
            // grow: at least 1 GiB, at least the reserve so far (doubling), capped at 32 GiB per chunk
            size_t want = std::max<size_t>(bytes, std::min<size_t>(std::max<size_t>(1ull << 30, reserved),
                                                                   32ull << 30));
            char *base = nullptr;
            cudaError_t e = cudaMalloc((void **)&base, want);
            if (e != cudaSuccess && want > bytes) {
                cudaGetLastError();
                want = bytes;
                e = cudaMalloc((void **)&base, want);
            }
            if (e != cudaSuccess) {
                cudaGetLastError();
                throw Error{DHGP_ERR_CUDA, "device memory exhausted: cannot allocate " + std::to_string(bytes) +
                                               " bytes (" + std::to_string(reserved) + " held by libdhgp on device " +
                                               std::to_string(device) + ")"};
            }
            chunks[base] = want;
            reserved += want;
            insert_free(base, want);
            it = free_by_size.lower_bound(bytes);
        }
        char *p = it->second;
        const size_t have = it->first;
        erase_free(free_by_addr.find(p));
        if (have > bytes) insert_free(p + bytes, have - bytes);
        used[p] = bytes;
        return p;
    }
    void release(void *vp) {
        char *p = (char *)vp;
        std::lock_guard<std::mutex> lk(mu);
        auto u = used.find(p);
        if (u == used.end()) throw Error{DHGP_ERR_CUDA, "arena: free of an unknown pointer"};
        size_t n = u->second;
        used.erase(u);
        char *end = chunk_end(p);
        // coalesce with the following and the preceding free blocks of the same chunk
        auto nx = free_by_addr.find(p + n);
        if (nx != free_by_addr.end() && p + n < end) {
            n += nx->second;
            erase_free(nx);
        }
        auto pv = free_by_addr.lower_bound(p);
        if (pv != free_by_addr.begin()) {
            --pv;
            if (pv->first + pv->second == p && chunk_end(pv->first) == end) {
                p = pv->first;
                n += pv->second;
                erase_free(pv);
            }
        }
        insert_free(p, n);
    }
};
Arena g_arena[64];
}  // namespace

void *arena_alloc(int device, size_t bytes) { return g_arena[device].alloc(device, bytes); }
static size_t arena_reserved(int device) {
    std::lock_guard<std::mutex> lk(g_arena[device].mu);
    return g_arena[device].reserved;
}
void arena_free(int device, void *p) { g_arena[device].release(p); }
static cudaStream_t g_streams[64], g_side[64];
static cudaEvent_t g_fork[64], g_join[64];
static int g_sms[64];
static char *g_pinned[64];

static void setup(Ctx &c, int device) {
    if (device < 0 || device >= 64) throw Error{DHGP_ERR_ARG, "bad device ordinal"};
    c.device = device;
    DHGP_CUDA(cudaSetDevice(device));
    if (!g_streams[device]) {
        DHGP_CUDA(cudaStreamCreateWithFlags(&g_streams[device], cudaStreamNonBlocking));
        DHGP_CUDA(cudaStreamCreateWithFlags(&g_side[device], cudaStreamNonBlocking));
        DHGP_CUDA(cudaEventCreateWithFlags(&g_fork[device], cudaEventDisableTiming));
        DHGP_CUDA(cudaEventCreateWithFlags(&g_join[device], cudaEventDisableTiming));
        DHGP_CUDA(cudaDeviceGetAttribute(&g_sms[device], cudaDevAttrMultiProcessorCount, device));
        DHGP_CUDA(cudaHostAlloc((void **)&g_pinned[device], Ctx::kPinnedBytes, cudaHostAllocDefault));
    }
    c.stream = g_streams[device];
    c.side = g_side[device];
    c.ev_fork = g_fork[device];
    c.ev_join = g_join[device];
    c.num_sms = g_sms[device];
    c.pinned = g_pinned[device];
}

void seams_setup(Ctx &c, int device) { setup(c, device); }

namespace {
__global__ void k_used(int32_t N, const int32_t *assign, uint8_t *used) {
    pdl_entry();
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < N) used[assign[v]] = 1;
}
__global__ void k_remap(int32_t N, const int64_t *rank, int32_t *assign) {
    pdl_entry();
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < N) assign[v] = (int32_t)rank[assign[v]];
}
}  // namespace

struct PartitionResult {
    std::vector<int32_t> assign;
    int32_t num_parts = 0;
    std::vector<DLevel> levels_meta;  // N/E/Ps/Pd only
    std::vector<std::vector<double>> trace;
    double phase_ms[3] = {0, 0, 0};
    double device_ms = 0;
};

constexpr size_t kCheckpoint = 16;

// device bytes of one level's lists (what level_to_stub would release)
static size_t level_bytes(const DLevel &L) {
    if (L.pooled)  // the node lists live in the pool: only their (begin, end) arrays are the level's
        return 8 * (3 * (size_t)L.E + 4 * (size_t)L.N + 5) + 4 * ((size_t)L.Ps + L.Pd + L.U + L.N);
    return 8 * (3 * (size_t)L.E + 2 * (size_t)L.N + 5) + 4 * ((size_t)L.Ps + L.Pd + L.U + L.Sin + L.U + L.N);
}

// Rebuilds stub levels (lo, hi] by re-running the contraction from the
// nearest full level below, using the stored gammas (bit-identical).
static void rebuild_levels(Ctx &c, std::vector<DLevel> &levels, size_t hi, NodePool *pool) {
    size_t lo = hi;
    while (levels[lo].stub) lo--;
    int64_t *status = c.alloc<int64_t>(kStatusWords);
    for (size_t j = lo; j < hi; j++) {
        DLevel &f = levels[j];
        DLevel &next = levels[j + 1];
        const int32_t n = f.N;
        int32_t *match = c.alloc<int32_t>(n);
        uint8_t *isrep = c.alloc<uint8_t>(n);
        match_from_gamma(c, n, next.N, f.gamma, match, isrep);
        c.free(f.gamma);
        f.gamma = nullptr;
        DLevel coarse;
        ContractScratch cs;
        c.zero(status, kStatusWords);
        contract_count(c, f, match, isrep, coarse, cs, status, pool);
        LevelStatus st;
        c.d2h((int64_t *)&st, status, kStatusWords);
        c.sync();
        if (pool) node_pool_fit(c, *pool, st.pool_top, levels, &coarse);
        contract_write(c, f, coarse, cs, st, pool);
        contract_release_members(c, cs);
        coarse.gamma = next.gamma;  // the stored map to the level above
        next.gamma = nullptr;
        next.release(c);
        next = coarse;
        c.free(match);
        c.free(isrep);
    }
    c.free(status);
}

// the "level" observer payload (driver.py:106-116) from device arrays; the
// scores are scaled-integer histograms times `unit` (the reference's f64)
static void emit_level_event(Ctx &c, dhgp_observer_fn obs, void *user, int32_t level, const DLevel &f,
                             const DLevel &cl, int32_t n, const int32_t *pair, const double *score,
                             const int32_t *match, double unit) {
    std::vector<int32_t> hp(n), hm(n), hg(n), hsd(cl.Ps), hdd(cl.Pd), hsz(cl.N);
    std::vector<double> hs(n);
    std::vector<int64_t> hso((int64_t)cl.E + 1), hdo((int64_t)cl.E + 1);
    c.d2h(hp.data(), pair, n);
    c.d2h(hs.data(), score, n);
    c.d2h(hm.data(), match, n);
    c.d2h(hg.data(), f.gamma, n);
    c.d2h(hso.data(), cl.src_off, (int64_t)cl.E + 1);
    c.d2h(hsd.data(), cl.src_dat, cl.Ps);
    c.d2h(hdo.data(), cl.dst_off, (int64_t)cl.E + 1);
    c.d2h(hdd.data(), cl.dst_dat, cl.Pd);
    c.d2h(hsz.data(), cl.size, cl.N);
    c.sync();
    if (unit != 1.0)
        for (auto &x : hs) x *= unit;
    dhgp_event ev;
    memset(&ev, 0, sizeof ev);
    ev.kind = DHGP_EVENT_LEVEL;
    ev.level = level;
    ev.num_nodes = n;
    ev.num_edges = cl.E;
    ev.num_coarse = cl.N;
    ev.pair = hp.data();
    ev.score = hs.data();
    ev.match = hm.data();
    ev.gamma = hg.data();
    ev.c_src_off = hso.data();
    ev.c_src_dat = hsd.data();
    ev.c_dst_off = hdo.data();
    ev.c_dst_dat = hdd.data();
    ev.c_node_size = hsz.data();
    obs(&ev, user);
}

static RoundObserver round_observer(dhgp_observer_fn obs, void *user, int32_t E) {
    if (!obs) return RoundObserver();
    return [obs, user, E](const RoundRecord &r) {
        dhgp_event ev;
        memset(&ev, 0, sizeof ev);
        ev.kind = DHGP_EVENT_ROUND;
        ev.level = r.level;
        ev.round = r.round;
        ev.num_nodes = (int32_t)r.assign.size();
        ev.num_edges = E;
        ev.num_parts = r.num_parts;
        ev.assign = r.assign.data();
        ev.num_moves = (int32_t)r.node.size();
        ev.mv_node = r.node.data();
        ev.mv_from = r.from.data();
        ev.mv_to = r.to.data();
        ev.mv_gain_iso = r.gain_iso.data();
        ev.mv_gain_seq = r.gain_seq.data();
        ev.k = r.k;
        ev.total_gain = r.total_gain;
        ev.active = r.active.data();
        obs(&ev, user);
    };
}

// compaction (driver.py:137-143) + check_validity (144-146) of the level-0
// assignment; fills res.assign / res.num_parts
static void finish_partition(Ctx &c, const DLevel &L0, const DWeights &W, int32_t *assign, int32_t K, int64_t omega,
                             int64_t delta, PartitionResult &res) {
    const int32_t N0 = L0.N;
    int32_t final_parts = 0;
    if (N0 > 0) {
        uint8_t *used = c.alloc<uint8_t>(K);
        int64_t *rank = c.alloc<int64_t>((int64_t)K + 1);
        c.zero(used, K);
        pdl_launch(k_used, (unsigned)cdiv(N0, 256), 256, 0, c.stream, N0, assign, used);
        DHGP_LAUNCHED(c);
        scan_excl<uint8_t>(c, used, rank, K);
        pdl_launch(k_remap, (unsigned)cdiv(N0, 256), 256, 0, c.stream, N0, rank, assign);
        DHGP_LAUNCHED(c);
        int64_t fp = 0;
        c.d2h(&fp, rank + K, 1);
        c.sync();
        final_parts = (int32_t)fp;
        c.free(used);
        c.free(rank);
        int64_t *sz = c.alloc<int64_t>(final_parts), *ib = c.alloc<int64_t>(final_parts);
        evaluate_assign(c, L0, W, assign, final_parts, sz, ib, nullptr);
        std::vector<int64_t> hsz(final_parts), hib(final_parts);
        c.d2h(hsz.data(), sz, final_parts);
        c.d2h(hib.data(), ib, final_parts);
        res.assign.resize(N0);
        c.d2h(res.assign.data(), assign, N0);
        c.sync();
        c.free(sz);
        c.free(ib);
        for (int32_t p = 0; p < final_parts; p++) {
            if (hsz[p] > omega || hib[p] > delta) {
                std::string kind = hsz[p] > omega ? "size" : "inbound";
                int64_t actual = hsz[p] > omega ? hsz[p] : hib[p];
                int64_t limit = hsz[p] > omega ? omega : delta;
                throw Error{DHGP_ERR_INVALID_RESULT,
                            "internal error: produced an invalid partitioning: [Violation(part=" + std::to_string(p) +
                                ", kind='" + kind + "', actual=" + std::to_string(actual) +
                                ", limit=" + std::to_string(limit) + ")]"};
            }
        }
    }
    res.num_parts = final_parts;
}

static double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// partition for weights outside the exact-integer contract: the same level
// loop with the reference-order f64 scoring and refinement of ordered.cuh
// (weight-independent phases — incidence, matching, contraction — are the
// production kernels).  Every level is kept (no checkpoint / rebuild).
static void run_partition_ordered(Ctx &c, const DInput &in, const dhgp_config &cfg, DWeights &W,
                                  PartitionResult &res, dhgp_observer_fn obs, void *user) {
    const int64_t omega = cfg.max_size, delta = cfg.max_inbound;
    const int32_t N0 = in.N;
    std::vector<DLevel> levels(1);
    int64_t *status = nullptr;
    int32_t *assign = nullptr, *assign2 = nullptr;
    try {
        build_level0(c, in, levels[0]);
        const double t0 = now_ms();
        const int64_t target = (N0 + omega - 1) / omega;
        status = c.alloc<int64_t>(kStatusWords);
        while (levels.back().N > target) {
            if ((int64_t)levels.size() - 1 >= cfg.max_levels)
                throw Error{DHGP_ERR_MAX_LEVELS, "coarsening exceeded max_levels=" + std::to_string(cfg.max_levels) +
                                                     " (" + std::to_string(levels.back().N) + " nodes, target " +
                                                     std::to_string(target) + ")"};
            const int32_t n = levels.back().N;
            int32_t *pair = c.alloc<int32_t>(n), *match = c.alloc<int32_t>(n), *claim = c.alloc<int32_t>(n);
            double *score = c.alloc<double>(n);
            uint8_t *isrep = c.alloc<uint8_t>(n);
            c.zero(status, kStatusWords);
            ord_score(c, levels.back(), W.w, omega, delta, pair, score);
            launch_matching(c, n, pair, score, match, isrep, claim, status);
            DLevel coarse;
            ContractScratch cs;
            contract_count(c, levels.back(), match, isrep, coarse, cs, status);
            LevelStatus st;
            c.d2h((int64_t *)&st, status, kStatusWords);
            c.sync();
            if ((st.bad_cert || st.long_run) && matching_fallbacks(c, n, pair, score, match, isrep, claim, st)) {
                contract_release(c, cs);
                coarse.release(c);
                c.free(levels.back().gamma);
                levels.back().gamma = nullptr;
                c.zero(status, kStatusWords);
                contract_count(c, levels.back(), match, isrep, coarse, cs, status);
                const int64_t moved = st.moved;
                c.d2h((int64_t *)&st, status, kStatusWords);
                c.sync();
                st.moved = moved;
            }
            const bool stop = st.moved == 0;
            if (stop) {
                contract_release(c, cs);
                coarse.release(c);
                c.free(levels.back().gamma);
                levels.back().gamma = nullptr;
            } else {
                contract_write(c, levels.back(), coarse, cs, st);
                levels.push_back(coarse);
                if (obs)
                    emit_level_event(c, obs, user, (int32_t)levels.size() - 2, levels[levels.size() - 2],
                                     levels.back(), n, pair, score, match, 1.0);
            }
            contract_release_members(c, cs);
            for (void *q : {(void *)pair, (void *)match, (void *)claim, (void *)score, (void *)isrep}) c.free(q);
            if (stop) break;
        }
        c.free(status);
        status = nullptr;
        const double t1 = now_ms();
        // ---- initial partitioning + uncoarsening (driver.py:121-134) -----------
        const int32_t K = levels.back().N;
        assign = c.alloc<int32_t>(std::max(N0, 1));
        assign2 = c.alloc<int32_t>(std::max(N0, 1));
        iota_i32(c, assign, K);
        res.trace.assign(levels.size(), {});
        for (auto &L : levels) {
            DLevel m;
            m.N = L.N;
            m.E = L.E;
            m.Ps = L.Ps;
            m.Pd = L.Pd;
            res.levels_meta.push_back(m);
        }
        RoundObserver robs = round_observer(obs, user, in.E);
        const int64_t nl = (int64_t)levels.size();
        for (int64_t li = nl - 1; li >= 0; li--) {
            if (li < nl - 1) {
                ord_project(c, levels[li].N, levels[li].gamma, assign, assign2);
                std::swap(assign, assign2);
                levels[li + 1].release(c);
            }
            ord_refine_level(c, levels[li], W.w, assign, K, omega, delta, cfg.max_rounds, (int32_t)li,
                             res.trace[nl - 1 - li], obs ? &robs : nullptr);
        }
        const double t2 = now_ms();
        finish_partition(c, levels[0], W, assign, K, omega, delta, res);
        const double t3 = now_ms();
        res.phase_ms[0] = t1 - t0;
        res.phase_ms[1] = t2 - t1;
        res.phase_ms[2] = t3 - t0;
    } catch (...) {
        c.free(status);
        c.free(assign);
        c.free(assign2);
        for (auto &L : levels) L.release(c);
        W.release(c);
        throw;
    }
    c.free(assign);
    c.free(assign2);
    for (auto &L : levels) L.release(c);
    W.release(c);
    c.sync();
}

// partition (driver.py:76-163) over a resident input
static void run_partition(Ctx &c, const DInput &in, const dhgp_config &cfg, PartitionResult &res,
                          dhgp_observer_fn obs, void *user) {
    const int64_t omega = cfg.max_size, delta = cfg.max_inbound;
    if (cfg.max_rounds < 1 || cfg.batch_size < 1 || cfg.max_levels < 1)
        throw Error{DHGP_ERR_ARG, "max_rounds, batch_size and max_levels must be >= 1"};
    // check_feasibility order (hgraph.py:382-401)
    if (omega < 1) throw Error{DHGP_ERR_INFEASIBLE, "max_size must be >= 1, got " + std::to_string(omega)};
    if (delta < 0) throw Error{DHGP_ERR_INFEASIBLE, "max_inbound must be >= 0, got " + std::to_string(delta)};
    const int32_t N0 = in.N;
    {
        int32_t bs, bi, sz = 0, deg = 0;
        feasibility_input(c, in, omega, delta, &bs, &bi, &sz, &deg);
        if (bs >= 0)
            throw Error{DHGP_ERR_INFEASIBLE, "node " + std::to_string(bs) + " has size " + std::to_string(sz) +
                                                 " > max_size " + std::to_string(omega)};
        if (bi >= 0)
            throw Error{DHGP_ERR_INFEASIBLE, "node " + std::to_string(bi) + " has " + std::to_string(deg) +
                                                 " inbound edges > max_inbound " + std::to_string(delta)};
    }
    DWeights W;
    prepare_weights(c, in, W);
    if (!W.integral) {  // the reference-order f64 path (ordered.cuh)
        run_partition_ordered(c, in, cfg, W, res, obs, user);
        return;
    }
    std::vector<DLevel> levels(1);
    build_level0(c, in, levels[0]);
    // per-node lists of every level in one pool (room for three times level 0's)
    NodePool pool;
    node_pool_init(c, pool, levels[0], 3.0);

    const double t0 = now_ms();
    c.sync_wait_ms = 0.0;
    c.syncs = 0;
    const int64_t launches0 = c.launches;
    const int64_t target = (N0 + omega - 1) / omega;
    // ---- coarsening (driver.py:97-118) -----------------------------------
    // One host sync per level: scoring, matching and the counting half of the
    // contraction are queued back to back; the sync reads the matched-pair
    // count, the fallback flags and the coarse sizes together.  A level with
    // no pair is discarded (driver.py:104-105).
    ScoreScratch sscr;
    int64_t *status = nullptr;
    // incremental scoring carries the previous level's choices and clusters
    const char *fs = getenv("DHGP_FULL_SCORE");  // tests: the full rescoring every level
    const bool inc_score = score_inc_supported(c, W) && !(fs && fs[0] == '1');
    int32_t *prev_pair = nullptr, *cma = nullptr, *cmb = nullptr;
    double *prev_score = nullptr;
    auto free_carry = [&]() {
        c.free(prev_pair);
        c.free(prev_score);
        c.free(cma);
        c.free(cmb);
        prev_pair = cma = cmb = nullptr;
        prev_score = nullptr;
    };
    // bytes of non-checkpoint levels kept whole (no rebuild during
    // uncoarsening): up to 65% of the memory free at this point
    size_t kept = 0, keep_budget = 0;
    {
        size_t freeb = 0, total = 0;
        DHGP_CUDA(cudaMemGetInfo(&freeb, &total));
        keep_budget = (size_t)(0.80 * (double)(freeb + arena_reserved(c.device)));
        const char *e = getenv("DHGP_KEEP_LEVELS_BYTES");  // tests: force the checkpoint/rebuild path
        if (e) keep_budget = (size_t)strtoull(e, nullptr, 10);
    }
    try {
        score_scratch_init(c, sscr, N0);
        status = c.alloc<int64_t>(kStatusWords);
        while (levels.back().N > target) {
            if ((int64_t)levels.size() - 1 >= cfg.max_levels)
                throw Error{DHGP_ERR_MAX_LEVELS, "coarsening exceeded max_levels=" + std::to_string(cfg.max_levels) +
                                                     " (" + std::to_string(levels.back().N) + " nodes, target " +
                                                     std::to_string(target) + ")"};
            const int32_t n = levels.back().N;
            const int64_t ncap = shard_capacity(c.comm, n);  // room for the allgather of (pair, score)
            int32_t *pair = c.alloc<int32_t>(ncap), *match = c.alloc<int32_t>(n), *claim = c.alloc<int32_t>(n);
            double *score = c.alloc<double>(ncap);
            uint8_t *isrep = c.alloc<uint8_t>(n);
            c.zero(status, kStatusWords);
            if (inc_score && prev_pair) {
                ScoreCarry cy;
                cy.prev_pair = prev_pair;
                cy.prev_score = prev_score;
                cy.gamma_prev = levels[levels.size() - 2].gamma;
                cy.ma = cma;
                cy.mb = cmb;
                score_select_inc(c, levels.back(), W, omega, delta, pair, score, sscr, cy);
            } else {
                score_select(c, levels.back(), W, omega, delta, pair, score, sscr);
            }
            launch_matching(c, n, pair, score, match, isrep, claim, status);
            DLevel coarse;
            ContractScratch cs;
            contract_count(c, levels.back(), match, isrep, coarse, cs, status, &pool);
            LevelStatus st;
            c.d2h((int64_t *)&st, status, kStatusWords);
            c.sync();
            if (st.bad_cert || st.long_run) {
                if (matching_fallbacks(c, n, pair, score, match, isrep, claim, st)) {
                    contract_release(c, cs);
                    coarse.release(c);
                    c.free(levels.back().gamma);
                    levels.back().gamma = nullptr;
                    c.zero(status, kStatusWords);
                    contract_count(c, levels.back(), match, isrep, coarse, cs, status, &pool);
                    int64_t moved = st.moved;
                    c.d2h((int64_t *)&st, status, kStatusWords);
                    c.sync();
                    st.moved = moved;
                }
            }
            const bool stop = st.moved == 0;
            if (stop) {
                contract_release(c, cs);
                coarse.release(c);
                c.free(levels.back().gamma);
                levels.back().gamma = nullptr;
            } else {
                node_pool_fit(c, pool, st.pool_top, levels, &coarse);
                contract_write(c, levels.back(), coarse, cs, st, &pool);
                levels.push_back(coarse);
            }
            if (!stop && obs)
                emit_level_event(c, obs, user, (int32_t)levels.size() - 2, levels[levels.size() - 2], levels.back(),
                                 n, pair, score, match, W.unit);
            free_carry();
            if (!stop && inc_score) {  // this level's choices and clusters feed the next scoring
                prev_pair = pair;
                prev_score = score;
                cma = cs.ma;
                cmb = cs.mb;
                cs.ma = cs.mb = nullptr;
            } else {
                c.free(pair);
                c.free(score);
                contract_release_members(c, cs);
            }
            c.free(match);
            c.free(claim);
            c.free(isrep);
            if (stop) break;
            // memory: every kCheckpoint-th level stays whole; the others stay
            // whole while they fit the level budget, else keep only gamma and
            // are rebuilt from their checkpoint on the way up
            const size_t fi = levels.size() - 2;
            if (fi % kCheckpoint != 0) {
                const size_t lb = level_bytes(levels[fi]);
                if (kept + lb <= keep_budget)
                    kept += lb;
                else
                    level_to_stub(c, levels[fi]);
            }
        }
    } catch (...) {
        free_carry();
        for (auto &L : levels) L.release(c);
        pool.release(c);
        W.release(c);
        score_scratch_release(c, sscr);
        c.free(status);
        throw;
    }
    free_carry();
    score_scratch_release(c, sscr);
    c.free(status);
    const double t1 = now_ms();
    // ---- initial partitioning + uncoarsening (driver.py:121-134) -----------
    const int32_t K = levels.back().N;
    int32_t *assign = c.alloc<int32_t>(N0), *assign2 = c.alloc<int32_t>(N0);
    iota_i32(c, assign, K);
    res.trace.assign(levels.size(), {});
    for (auto &L : levels) {
        DLevel m;
        m.N = L.N;
        m.E = L.E;
        m.Ps = L.Ps;
        m.Pd = L.Pd;
        res.levels_meta.push_back(m);
    }
    RoundObserver robs = round_observer(obs, user, in.E);
    // incremental refinement (refine.cuh) unless DHGP_FULL_REFINE=1 (tests:
    // both modes)
    RefineState rst;
    {
        const char *fe = getenv("DHGP_FULL_REFINE");
        const bool inc = !(fe && fe[0] == '1');
        refine_state_init(c, rst, levels[0], K, inc);
    }
    try {
        const int64_t L = (int64_t)levels.size();
        refine_level(c, levels[L - 1], W, rst, assign, K, omega, delta, cfg.max_rounds, (int32_t)(L - 1),
                     res.trace[0], obs ? &robs : nullptr, in.max_edge_pins);
        for (int64_t li = L - 2; li >= 0; li--) {
            if (levels[li].stub) rebuild_levels(c, levels, (size_t)li, &pool);
            DLevel &f = levels[li];
            refine_project(c, rst, f, levels[li + 1].N, assign, assign2);
            levels[li + 1].release(c);
            refine_level(c, f, W, rst, assign, K, omega, delta, cfg.max_rounds, (int32_t)li, res.trace[L - 1 - li],
                         obs ? &robs : nullptr, in.max_edge_pins);
        }
        refine_state_release(c, rst);
        const double t2 = now_ms();
        // ---- compaction (driver.py:137-143) + check_validity (144-146) ------
        finish_partition(c, levels[0], W, assign, K, omega, delta, res);
        const double t3 = now_ms();
        res.phase_ms[0] = t1 - t0;
        res.phase_ms[1] = t2 - t1;
        res.phase_ms[2] = t3 - t0;
        if (getenv("DHGP_SYNCSTAT"))
            fprintf(stderr, "syncstat wall_ms %.1f sync_wait_ms %.1f syncs %lld launches %lld\n", t3 - t0,
                    c.sync_wait_ms, (long long)c.syncs, (long long)(c.launches - launches0));
    } catch (...) {
        refine_state_release(c, rst);
        for (auto &L : levels) L.release(c);
        pool.release(c);
        W.release(c);
        c.free(assign);
        c.free(assign2);
        throw;
    }
    for (auto &L : levels) L.release(c);
    pool.release(c);
    W.release(c);
    c.free(assign);
    c.free(assign2);
    c.sync();
}

static void fill_stats(const PartitionResult &r, dhgp_stats *s, int64_t launches) {
    if (!s) return;
    memset(s, 0, sizeof *s);
    const int64_t nl = (int64_t)r.levels_meta.size();
    s->num_levels = nl;
    s->level_nodes = (int64_t *)malloc(sizeof(int64_t) * (nl ? nl : 1));
    s->level_edges = (int64_t *)malloc(sizeof(int64_t) * (nl ? nl : 1));
    s->level_pins = (int64_t *)malloc(sizeof(int64_t) * (nl ? nl : 1));
    s->trace_off = (int64_t *)malloc(sizeof(int64_t) * (nl + 1));
    int64_t tot = 0;
    for (auto &t : r.trace) tot += (int64_t)t.size();
    s->trace_val = (double *)malloc(sizeof(double) * (tot ? tot : 1));
    s->trace_off[0] = 0;
    for (int64_t l = 0; l < nl; l++) {
        s->level_nodes[l] = r.levels_meta[l].N;
        s->level_edges[l] = r.levels_meta[l].E;
        s->level_pins[l] = r.levels_meta[l].Ps + r.levels_meta[l].Pd;
        const auto &t = r.trace[l];
        for (size_t i = 0; i < t.size(); i++) s->trace_val[s->trace_off[l] + i] = t[i];
        s->trace_off[l + 1] = s->trace_off[l] + (int64_t)t.size();
    }
    s->num_partitions = r.num_parts;
    for (int i = 0; i < 3; i++) s->phase_ms[i] = r.phase_ms[i];
    s->gpu_launches = launches;
    s->device_ms = r.device_ms;
}

}  // namespace dhgp

// ===========================================================================
// C-ABI
// ===========================================================================
using namespace dhgp;

Comm *comm_of(dhgp_comm *cm);

struct dhgp_session {
    dhgp_comm *comm = nullptr;
    int device = 0;
    DInput in;
    bool profiling = false;
    std::vector<KernelStat> kstats;
};

#define DHGP_GUARD_BEGIN(dev) \
    std::lock_guard<std::recursive_mutex> _lk(device_mutex(dev)); \
    try {
#define DHGP_GUARD_END                      \
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

static void check_graph(const dhgp_graph *g) {
    if (!g || g->num_nodes < 0 || g->num_edges < 0 || !g->src_off || !g->dst_off ||
        (g->num_edges > 0 && !g->edge_weight))
        throw Error{DHGP_ERR_ARG, "malformed dhgp_graph"};
}

extern "C" {

const char *dhgp_last_error(void) { return last_error(); }

const char *dhgp_build_info(void) {
    static std::string s = std::string("libdhgp sm_100a, nvcc ") + std::to_string(__CUDACC_VER_MAJOR__) + "." +
                           std::to_string(__CUDACC_VER_MINOR__);
    return s.c_str();
}

int dhgp_device_count(int32_t *count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        set_error(DHGP_ERR_CUDA, cudaGetErrorString(e));
        *count = 0;
        return DHGP_ERR_CUDA;
    }
    *count = n;
    return DHGP_OK;
}

static int partition_impl(const dhgp_graph *g, const dhgp_config *cfg, dhgp_comm *cm, int32_t *assign_out,
                          int32_t *num_parts_out, dhgp_stats *stats_out, dhgp_observer_fn obs, void *user) {
    DHGP_GUARD_BEGIN(cfg ? cfg->device : 0)
    check_graph(g);
    Ctx c;
    setup(c, cfg->device);
    c.comm = comm_of(cm);
    DInput in;
    upload_input(c, *g, in);
    PartitionResult r;
    try {
        run_partition(c, in, *cfg, r, obs, user);
    } catch (...) {
        in.release(c);
        c.sync();
        throw;
    }
    in.release(c);
    if (r.assign.size()) memcpy(assign_out, r.assign.data(), sizeof(int32_t) * r.assign.size());
    *num_parts_out = r.num_parts;
    fill_stats(r, stats_out, c.launches);
    DHGP_GUARD_END
}

int dhgp_partition(const dhgp_graph *g, const dhgp_config *cfg, int32_t *assign_out, int32_t *num_parts_out,
                   dhgp_stats *stats_out, dhgp_observer_fn obs, void *user) {
    return partition_impl(g, cfg, nullptr, assign_out, num_parts_out, stats_out, obs, user);
}

int dhgp_partition_sharded(const dhgp_graph *g, const dhgp_config *cfg, dhgp_comm *cm, int32_t *assign_out,
                           int32_t *num_parts_out, dhgp_stats *stats_out) {
    return partition_impl(g, cfg, cm, assign_out, num_parts_out, stats_out, nullptr, nullptr);
}

int dhgp_session_set_comm(dhgp_session *s, dhgp_comm *cm) {
    if (!s) return DHGP_ERR_ARG;
    s->comm = cm;
    return DHGP_OK;
}

void dhgp_stats_free(dhgp_stats *s) {
    if (!s) return;
    free(s->level_nodes);
    free(s->level_edges);
    free(s->level_pins);
    free(s->trace_off);
    free(s->trace_val);
    memset(s, 0, sizeof *s);
}

int dhgp_session_create(const dhgp_graph *g, int32_t device, dhgp_session **out) {
    DHGP_GUARD_BEGIN(device)
    check_graph(g);
    Ctx c;
    setup(c, device);
    dhgp_session *s = new dhgp_session();
    s->device = device;
    upload_input(c, *g, s->in);
    c.sync();
    *out = s;
    DHGP_GUARD_END
}

int dhgp_session_partition(dhgp_session *s, const dhgp_config *cfg, int32_t *assign_out, int32_t *num_parts_out,
                           dhgp_stats *stats_out) {
    DHGP_GUARD_BEGIN(s->device)
    Ctx c;
    setup(c, s->device);
    c.comm = comm_of(s->comm);
    c.profiling = s->profiling;
    dhgp_config cc = *cfg;
    cc.device = s->device;
    PartitionResult r;
    cudaEvent_t ev0, ev1;
    DHGP_CUDA(cudaEventCreate(&ev0));
    DHGP_CUDA(cudaEventCreate(&ev1));
    DHGP_CUDA(cudaEventRecord(ev0, c.stream));
    run_partition(c, s->in, cc, r, nullptr, nullptr);
    DHGP_CUDA(cudaEventRecord(ev1, c.stream));
    DHGP_CUDA(cudaEventSynchronize(ev1));
    float dms = 0.f;
    DHGP_CUDA(cudaEventElapsedTime(&dms, ev0, ev1));
    r.device_ms = dms;
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    if (c.profiling) {
        c.flush_profile();
        s->kstats = c.kstats;
    }
    if (assign_out && r.assign.size()) memcpy(assign_out, r.assign.data(), sizeof(int32_t) * r.assign.size());
    if (num_parts_out) *num_parts_out = r.num_parts;
    fill_stats(r, stats_out, c.launches);
    DHGP_GUARD_END
}

void dhgp_session_destroy(dhgp_session *s) {
    if (!s) return;
    std::lock_guard<std::recursive_mutex> lk(device_mutex(s->device));
    try {
        Ctx c;
        setup(c, s->device);
        s->in.release(c);
        c.sync();
    } catch (...) {
    }
    delete s;
}

int dhgp_session_set_profiling(dhgp_session *s, int32_t on) {
    s->profiling = on != 0;
    return DHGP_OK;
}

int dhgp_session_kernel_stats(dhgp_session *s, int32_t max_rows, const char **names, int64_t *launches,
                              double *total_ms, double *bytes, int32_t *rows_out) {
    int32_t n = (int32_t)std::min<size_t>(s->kstats.size(), (size_t)max_rows);
    for (int32_t i = 0; i < n; i++) {
        names[i] = s->kstats[i].name;
        launches[i] = s->kstats[i].launches;
        total_ms[i] = s->kstats[i].ms;
        bytes[i] = s->kstats[i].bytes;
    }
    *rows_out = n;
    return DHGP_OK;
}

void dhgp_free(void *p) { free(p); }

}  // extern "C"
