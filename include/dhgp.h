/*
 * dhgp.h — C-ABI of the B200-native directed-hypergraph partitioner
 * (libdhgp.so, built from paper_2604_14411_b200/csrc/ for sm_100a).
 *
 * Plain pointers and sizes only; no torch types.  Every input is host
 * memory owned by the caller and only read; every output array is caller
 * allocated unless stated otherwise.  Calls are synchronous; the library
 * keeps one CUDA stream per device and serialises calls with a mutex.
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/dhgpart/<file>:<line>).  The reference's Python
 * binding that a maintainer would add is shown in INTEGRATION.md; this
 * repo's own binding is paper_2604_14411_b200/_lib.py (ctypes).
 */
#ifndef DHGP_H
#define DHGP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (map 1:1 onto dhgpart.errors, errors.py:4-27) ------- */
#define DHGP_OK 0
#define DHGP_ERR_INFEASIBLE 1     /* InfeasibleError   (hgraph.py:376-401)  */
#define DHGP_ERR_MAX_LEVELS 2     /* DhgError "max_levels" (driver.py:98)   */
#define DHGP_ERR_MATCHING 3       /* MatchingInvariantError (_kernels.pyx:139) */
#define DHGP_ERR_INVALID_RESULT 4 /* DhgError "internal error" (driver.py:146) */
#define DHGP_ERR_CUDA 5           /* CUDA runtime / launch failure          */
#define DHGP_ERR_ARG 6            /* ValueError: malformed arguments        */
#define DHGP_ERR_UNSUPPORTED 7    /* input outside the bit-exact contract   */

/* ---- input hypergraph (the primary fields of hgraph.Hypergraph,
 *      hgraph.py:172-181; derived families are rebuilt on device) ------- */
typedef struct {
    int32_t num_nodes;
    int32_t num_edges;
    const double *edge_weight; /* [E] finite, >= 0                        */
    const int64_t *src_off;    /* [E+1] edge_src.offsets                  */
    const int32_t *src_dat;    /* [src_off[E]]                            */
    const int64_t *dst_off;    /* [E+1] edge_dst.offsets                  */
    const int32_t *dst_dat;    /* [dst_off[E]]                            */
    const int32_t *node_size;  /* [N] or NULL (= all ones)                */
} dhgp_graph;

/* ---- driver.Config + hgraph.Constraints (driver.py:31-52, hgraph.py:302) */
typedef struct {
    int64_t max_size;    /* Omega                                       */
    int64_t max_inbound; /* Delta                                       */
    int32_t max_rounds;
    int32_t batch_size;  /* validated >= 1; result-invariant (coarsen.py:106) */
    int32_t max_levels;
    int32_t device;      /* CUDA ordinal                                */
} dhgp_config;

/* ---- driver.RunStats (driver.py:55-73); library-owned buffers ------- */
typedef struct {
    int64_t num_levels;    /* len(levels), finest first                 */
    int64_t *level_nodes;  /* [num_levels]                              */
    int64_t *level_edges;  /* [num_levels]                              */
    int64_t *level_pins;   /* [num_levels] |src data| + |dst data|       */
    int64_t *trace_off;    /* [num_levels+1]; stage s = coarsest-first   */
    double *trace_val;     /* [trace_off[num_levels]]                    */
    int32_t num_partitions;
    double phase_ms[3];    /* coarsen, refine, total (wall, ms)          */
    int64_t gpu_launches;  /* kernels launched by this call              */
    double device_ms;      /* CUDA-event time of the call on its stream  */
} dhgp_stats;

/* ---- observer payloads (driver.py:106-116, refine.py:295-307) --------- */
#define DHGP_EVENT_LEVEL 1
#define DHGP_EVENT_ROUND 2
typedef struct {
    int32_t kind;
    int32_t level;      /* level: index = len(maps); round: level id     */
    int32_t round;
    int32_t num_nodes;  /* fine N (level) / graph N (round)              */
    int32_t num_edges;
    int32_t num_coarse; /* level only                                    */
    int32_t num_parts;  /* round only                                    */
    /* level payload: forest + cmap + coarse graph primary fields        */
    const int32_t *pair;
    const double *score;
    const int32_t *match;
    const int32_t *gamma;
    const int64_t *c_src_off;
    const int32_t *c_src_dat;
    const int64_t *c_dst_off;
    const int32_t *c_dst_dat;
    const int32_t *c_node_size;
    /* round payload: assignment before the round, MoveSet, PrefixSelection */
    const int32_t *assign;
    int32_t num_moves;
    const int32_t *mv_node;
    const int32_t *mv_from;
    const int32_t *mv_to;
    const double *mv_gain_iso;
    const double *mv_gain_seq;
    int32_t k;
    double total_gain;
    const int64_t *active; /* [num_moves+1] */
} dhgp_event;
typedef void (*dhgp_observer_fn)(const dhgp_event *ev, void *user);

/* ======================================================================= */
/* libdhgp.so — the product (CUDA, sm_100a)                                */
/* ======================================================================= */

const char *dhgp_last_error(void);     /* thread-local message text      */
const char *dhgp_build_info(void);     /* arch / nvcc version string     */
int dhgp_device_count(int32_t *count);

/* dhgpart.partition(g, cfg, observer, timings)  — driver.py:76-163.
 * assign_out [N] caller-owned; stats library-owned (dhgp_stats_free). */
int dhgp_partition(const dhgp_graph *g, const dhgp_config *cfg, int32_t *assign_out, int32_t *num_parts_out,
                   dhgp_stats *stats_out, dhgp_observer_fn obs, void *user);
void dhgp_stats_free(dhgp_stats *s);

/* Device-resident session: the graph is uploaded once and partitioned
 * many times (bench.py's HBM-resident `value`).  Same semantics as
 * dhgp_partition. */
typedef struct dhgp_session dhgp_session;
int dhgp_session_create(const dhgp_graph *g, int32_t device, dhgp_session **out);
int dhgp_session_partition(dhgp_session *s, const dhgp_config *cfg, int32_t *assign_out, int32_t *num_parts_out,
                           dhgp_stats *stats_out);
void dhgp_session_destroy(dhgp_session *s);
/* Per-kernel device timings of the last session_partition call:
 * name[i] (static strings), launches[i], total_ms[i], algorithmic bytes[i]. */
int dhgp_session_kernel_stats(dhgp_session *s, int32_t max_rows, const char **names, int64_t *launches,
                              double *total_ms, double *bytes, int32_t *rows_out);
int dhgp_session_set_profiling(dhgp_session *s, int32_t on);

/* ---- multi-GPU: node-range sharding ----------------
 * No reference interface: the reference is single-threaded.  These extend
 * dhgp_partition (driver.py:76-163) to one process per GPU; the result is
 * bit-identical to the single-GPU call at every world size.  Scoring
 * (coarsen.py:93-132) and proposals (refine.py:82-116) are computed per node
 * range and completed by an in-place allgather; everything else runs
 * replicated. */
#define DHGP_COMM_NCCL 1 /* ncclAllGather on the library stream (libnccl.so.2, loaded at run time) */
#define DHGP_COMM_HOST 2 /* the caller's allgather over host memory (gloo, MPI, tests) */
typedef struct dhgp_comm dhgp_comm;
/* in place: buf holds world * bytes_per_rank bytes; rank r's part is at
 * r * bytes_per_rank.  Return 0 on success. */
typedef int (*dhgp_allgather_fn)(void *user, void *buf, int64_t bytes_per_rank);
int dhgp_comm_nccl_unique_id(uint8_t *id_out /* [128] */);
int dhgp_comm_init_nccl(int32_t world, int32_t rank, const uint8_t *id /* [128] */, int32_t device,
                        dhgp_comm **out);
int dhgp_comm_init_host(int32_t world, int32_t rank, dhgp_allgather_fn fn, void *user, dhgp_comm **out);
/* phases over fewer than min_units nodes (or moves) run replicated (default 65536) */
int dhgp_comm_set_min_units(dhgp_comm *cm, int64_t min_units);
int dhgp_comm_stats(const dhgp_comm *cm, int64_t *allgathers, double *bytes);
void dhgp_comm_destroy(dhgp_comm *cm);
int dhgp_partition_sharded(const dhgp_graph *g, const dhgp_config *cfg, dhgp_comm *cm, int32_t *assign_out,
                           int32_t *num_parts_out, dhgp_stats *stats_out);
int dhgp_session_set_comm(dhgp_session *s, dhgp_comm *cm); /* NULL = single GPU */
/* the range rule of every sharded phase: returns 1 (and [lo, hi), chunk) when
 * n units are split over `world` ranks, 0 when the phase runs replicated */
int dhgp_shard_range(int32_t world, int32_t rank, int64_t min_units, int64_t n, int64_t *lo, int64_t *hi,
                     int64_t *chunk);

/* ---- input path on the GPU: hgraph.parse_dhg (hgraph.py:409-467) ------
 * text = the edge lines (everything after the header line, trailing blank
 * lines removed).  begin: finds the lines and parses every line whose tokens
 * are unsigned decimal integers; returns the line count (the caller raises
 * the reference's count error when it differs from num_edges; nothing else is
 * done then) and the number of "slow" lines the host must parse itself.
 * finish: takes the host's results for those lines (pin counts, weight,
 * error flag, ids), builds the CSR and flags every bad line; *first_bad_line
 * is the first one (-1 if none) — the caller re-derives its message. */
typedef struct dhgp_parse dhgp_parse;
int dhgp_parse_dhg_begin(const char *text, int64_t len, int64_t num_edges, int64_t num_nodes, int32_t device,
                         dhgp_parse **out, int64_t *lines_found, int64_t *num_slow);
int dhgp_parse_dhg_slow_lines(dhgp_parse *ps, int64_t *line_idx, int64_t *byte_lo, int64_t *byte_hi);
int dhgp_parse_dhg_finish(dhgp_parse *ps, const int64_t *slow_ks, const int64_t *slow_kd, const double *slow_w,
                          const uint8_t *slow_err, const int64_t *slow_ids_off, const int32_t *slow_ids,
                          int64_t *first_bad_line, int64_t *nsrc, int64_t *ndst);
int dhgp_parse_dhg_fetch(dhgp_parse *ps, double *w, int64_t *src_off, int32_t *src_dat, int64_t *dst_off,
                         int32_t *dst_dat);
int dhgp_parse_dhg_line_range(dhgp_parse *ps, int64_t line, int64_t *byte_lo, int64_t *byte_hi);
void dhgp_parse_free(dhgp_parse *ps);

/* ---- data model (hgraph.py) ------------------------------------------ */
/* Hypergraph._from_csr derived families — hgraph.py:212-238.  Output
 * sizes: in = dst_off[E], out = src_off[E], pins/inc = *num_pins_out
 * (<= src_off[E]+dst_off[E]; call with pin_dat/inc_dat = NULL first to
 * query, or pass buffers of the upper-bound size). */
int dhgp_incidence(const dhgp_graph *g, int32_t device, int64_t *in_off, int32_t *in_dat, int64_t *out_off,
                   int32_t *out_dat, int64_t *pin_off, int32_t *pin_dat, int64_t *inc_off, int32_t *inc_dat,
                   int64_t *num_pins_out);
/* coarsen.materialize_neighbors — coarsen.py:78-85.  nb_dat is
 * library-owned (free with dhgp_free). */
int dhgp_neighbors(const dhgp_graph *g, int32_t device, int64_t *nb_off, int32_t **nb_dat, int64_t *nnz_out);
void dhgp_free(void *p);
/* hgraph.check_feasibility — hgraph.py:376-401 (message in last_error) */
int dhgp_check_feasibility(const dhgp_graph *g, int64_t max_size, int64_t max_inbound, int32_t device);
/* baselines.one_pass (method 0, baselines.py:16-40) and
 * baselines.overlap_greedy (method 1, baselines.py:43-91): the reference's
 * comparison partitioners, bit-identical; check_feasibility first.
 * assign_out: [num_nodes], caller-owned. */
int dhgp_baseline(const dhgp_graph *g, int64_t max_size, int64_t max_inbound, int32_t method, int32_t device,
                  int32_t *assign_out, int32_t *num_parts_out);
/* hgraph.partition_sizes / distinct_inbound_sizes / connectivity —
 * hgraph.py:317-356 */
int dhgp_evaluate(const dhgp_graph *g, const int32_t *assign, int32_t num_parts, int32_t device, int64_t *sizes_out,
                  int64_t *inbound_out, double *connectivity_out);

/* ---- kernel-level seams: dhgpart.kernels (kernels.py:58-103) -------- */
/* All CSR arguments are (offsets int64[S+1], data int32[...]). */
int dhgp_union_size_sorted(const int32_t *a, int64_t na, const int32_t *b, int64_t nb, int32_t device,
                           int64_t *out); /* _kernels.pyx:35-44 */
int dhgp_fill_histograms(int32_t N, const int64_t *inc_off, const int32_t *inc_dat, int32_t E,
                         const int64_t *pin_off, const int32_t *pin_dat, const double *w, const int64_t *nbr_off,
                         const int32_t *nbr_dat, int64_t batch, int32_t device,
                         double *hist); /* _kernels.pyx:47-72 */
int dhgp_select_first_valid(int32_t N, const int64_t *order, const int64_t *nbr_off, const int32_t *nbr_dat,
                            const double *hist, const int32_t *node_size, const int64_t *in_off,
                            const int32_t *in_dat, int64_t max_size, int64_t max_inbound, int32_t device,
                            int32_t *pair, double *score); /* _kernels.pyx:75-103 */
int dhgp_resolve_matching(int32_t N, const int32_t *pair, const double *score, int32_t device,
                          int32_t *match); /* _kernels.pyx:106-181 */
int dhgp_connectivity_value(int32_t E, const int64_t *pin_off, const int32_t *pin_dat, const double *w,
                            int32_t N, const int32_t *assign, int32_t device,
                            double *out); /* _kernels.pyx:184-213 */
int dhgp_compute_pins(int32_t E, const int64_t *pin_off, const int32_t *pin_dat, const int64_t *dst_off,
                      const int32_t *dst_dat, int32_t N, const int32_t *assign, int32_t K, int32_t device,
                      int32_t *pins, int32_t *pins_in); /* _kernels.pyx:216-231 (dense, parity only) */
int dhgp_propose_moves(int32_t N, const int64_t *inc_off, const int32_t *inc_dat, int32_t E,
                       const int64_t *pin_off, const int32_t *pin_dat, const double *w, const int32_t *pins,
                       int32_t K, const int32_t *assign, const int64_t *part_sizes, const int32_t *node_size,
                       int64_t max_size, int32_t device, int32_t *target,
                       double *gain); /* _kernels.pyx:234-311 */
int dhgp_sequence_gains(int32_t N, const int64_t *inc_off, const int32_t *inc_dat, int32_t E,
                        const int64_t *pin_off, const int32_t *pin_dat, const double *w, const int32_t *pins,
                        int32_t K, int32_t M, const int32_t *node, const int32_t *from_part, const int32_t *to_part,
                        const double *gain_iso, const int64_t *pos, int32_t device,
                        double *gain_seq); /* _kernels.pyx:314-364 */
/* refine.build_events_and_select — refine.py:178-247 (pins_in dense) */
int dhgp_build_events_and_select(int32_t N, const int64_t *in_off, const int32_t *in_dat,
                                 const int32_t *node_size, int32_t E, int32_t K, int32_t M, const int32_t *node,
                                 const int32_t *from_part, const int32_t *to_part, const double *gain_seq,
                                 const int32_t *pins_in, const int64_t *part_sizes, const int64_t *part_inbound,
                                 int64_t max_size, int64_t max_inbound, int32_t device, int64_t *k_out,
                                 double *total_gain_out, int64_t *active);

#ifdef __cplusplus
}
#endif
#endif /* DHGP_H */
