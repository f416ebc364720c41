/* pprg.h — C ABI of the B200-native single-source PPR engine.
 *
 * The drop-in boundary for the reference's C++ core API
 * (the ppr/ headers under /root/reference/proj/core/include). Plain pointers and sizes, no
 * C++ or torch types. Each entry point names the reference interface it
 * replaces (file:line under /root/reference/proj). The C++ shim in
 * paper_2101_03652_b200/cpp (namespace ppr::) re-exposes these with the
 * reference's own signatures and exception types; INTEGRATION.md shows the
 * binding.
 *
 * Conventions
 *   - Graphs are immutable device-resident handles; each handle owns its CUDA
 *     stream and is safe to share between host threads (calls serialize).
 *   - Output vectors are CALLER-allocated, query-major: out[q * n + v] for
 *     query q (k queries per call). Host memory unless the *_device variant or
 *     PPRG_OUT_DEVICE flag says the pointers are device pointers. NULL skips.
 *   - Status codes: PPRG_OK, PPRG_EINVAL (std::invalid_argument in the
 *     reference), PPRG_EDATA (std::runtime_error), PPRG_EINTERNAL
 *     (std::logic_error), PPRG_ECUDA / PPRG_ENCCL (device / collective).
 *     pprg_last_error() returns the calling thread's last message.
 */
#ifndef PPRG_H
#define PPRG_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PPRG_OK 0
#define PPRG_EINVAL 1
#define PPRG_EDATA 2
#define PPRG_EINTERNAL 3
#define PPRG_ECUDA 4
#define PPRG_ENCCL 5

#define PPRG_OUT_DEVICE 1u /* output pointers are device pointers on the graph's GPU */
#define PPRG_ASYNC_HOST 2u /* host outputs: return once computed; the last block's copies
                              may still be landing -- pprg_graph_sync(g) waits for them.
                              Lets consecutive calls overlap copies with compute. */
#define PPRG_DETERMINISTIC 4u /* bitwise-reproducible results: identical inputs give identical
                                 bits on every run (the reference's rerun guarantee, SPEC.md
                                 "two runs with identical argv produce identical result files").
                                 Deterministic sweeps run in waves with double-buffered y
                                 (more sweeps), local phases pop before they scatter, and
                                 every cross-thread sum is exact fixed point. Slower. */

#define PPRG_RNG_PHILOX4X32_10 2u /* PPRW rng-id byte for our walk index (reference uses 1 = mt19937_64, rng.hpp:10) */

typedef struct pprg_graph pprg_graph;
typedef struct pprg_index pprg_index;
typedef struct pprg_part pprg_part;

/* Per-query statistics (PPRVector fields, types.hpp:57-65, plus device counters). */
typedef struct {
  double achieved_r_sum;   /* PPRVector::achieved_r_sum */
  uint64_t pushes;         /* PPRVector::pushes: edge pushes, deg_eff per node push */
  uint64_t walks;          /* PPRVector::walks */
  uint32_t sweeps;         /* global-phase sweeps (PowerPush) or iterations (PowItr) */
  uint32_t local_levels;   /* frontier levels of the queue phase */
  int32_t used_scan_phase; /* PowerPushTrace::used_scan_phase (push.hpp:97-100) */
  int32_t reserved;
} pprg_query_stats;

/* Per-call device counters (for the roofline). */
typedef struct {
  double device_ms;        /* CUDA-event time of the device section */
  double sweep_ms;         /* CUDA-event time of the global-sweep kernels */
  double local_ms;         /* CUDA-event time of the local (queue) phase */
  double final_ms;         /* CUDA-event time of the final residue pass */
  uint64_t alg_bytes;      /* SURVEY 8(d) algorithmic bytes of the global sweeps */
  uint64_t sweep_launches; /* persistent sweep-kernel launches */
  uint32_t max_sweeps;
  uint32_t kernel_launches;/* kernels this library launched for the call */
} pprg_call_stats;

const char* pprg_last_error(void);
int pprg_version(void);
/* Process-wide default for PPRG_DETERMINISTIC (0 = off at load). Calls without
 * a flags argument (pprg_run_traced, pprg_run_observed) follow it; calls with
 * flags are deterministic when either the flag or the default is set. */
int pprg_set_deterministic(int on);
int pprg_device_count(int* count);

/* ---- graphs (graph.hpp) -------------------------------------------------- */
/* Graph(std::vector<uint64_t> out_offsets, std::vector<NodeId> out_neighbors)
 * graph.hpp:18, graph.cpp:13-34 (same validation and messages). */
int pprg_graph_create(const uint64_t* offsets, const uint32_t* neighbors, uint64_t n, int device,
                      pprg_graph** out);
/* build_graph_from_edges(edges) graph.hpp:92, graph.cpp:36-63; pairs = 2*count
 * u64 (src, dst), bit-exact CSR (relabel, input-order neighbours). */
int pprg_graph_build_from_edges(const uint64_t* pairs, uint64_t count, int device,
                                pprg_graph** out);
/* Synthetic inputs (no reference counterpart). Cleaned (self-loops
 * and duplicates removed), sorted, then built with build_graph_from_edges
 * semantics. edges_out (optional, capacity draws) receives the canonical
 * cleaned list as (src << 32 | dst) before relabelling; *edge_count_out its length. */
int pprg_graph_generate_rmat(int scale, uint64_t edge_factor, double a, double b, double c,
                             uint64_t seed, int device, uint64_t* edges_out,
                             uint64_t* edge_count_out, pprg_graph** out);
int pprg_graph_generate_chung_lu(uint64_t n, uint64_t draws, double beta, uint64_t seed, int device,
                                 uint64_t* edges_out, uint64_t* edge_count_out, pprg_graph** out);
/* load_graph_cache / save_graph_cache graph.hpp:102-106, graph.cpp:115-143:
 * the PPRG file streams through pinned staging straight into / out of device
 * memory (same format, checks and messages as the reference). */
int pprg_graph_load_cache(const char* path, int device, pprg_graph** out);
int pprg_graph_save_cache(pprg_graph* g, const char* path);
/* n(), m(), dead_ends().size() — graph.hpp:20-21,33 */
int pprg_graph_info(const pprg_graph* g, uint64_t* n, uint64_t* m, uint64_t* dead_ends);
/* out_offsets()/out_neighbors()/dead_ends() — graph.hpp:31-33 (device -> host) */
int pprg_graph_export(const pprg_graph* g, uint64_t* offsets, uint32_t* neighbors,
                      uint32_t* dead_ends);
/* In-CSR used by the pull sweeps (internal layout, exported for tests). */
int pprg_graph_export_transpose(pprg_graph* g, uint64_t* in_offsets, uint32_t* in_neighbors);
void pprg_graph_destroy(pprg_graph* g);

/* ---- high-precision engines (push.hpp) ----------------------------------- */
/* power_iteration(g, s, alpha, lambda) push.hpp:80-81, push.cpp:81-108, for k sources. */
int pprg_power_iteration(pprg_graph* g, const uint32_t* sources, uint32_t k, double alpha,
                         double lambda, double* reserve_out, double* residue_out, uint32_t flags,
                         pprg_query_stats* qstats, pprg_call_stats* cstats);
/* sim_forward_push push.hpp:86-87, push.cpp:110-138 */
int pprg_sim_forward_push(pprg_graph* g, const uint32_t* sources, uint32_t k, double alpha,
                          double lambda, double* reserve_out, double* residue_out, uint32_t flags,
                          pprg_query_stats* qstats, pprg_call_stats* cstats);
/* fifo_forward_push(g, s, alpha, r_max, lambda_stop) push.hpp:92-94, push.cpp:140-149;
 * lambda_stop <= 0 means none. */
int pprg_fifo_forward_push(pprg_graph* g, const uint32_t* sources, uint32_t k, double alpha,
                           double r_max, double lambda_stop, double* reserve_out,
                           double* residue_out, uint32_t flags, pprg_query_stats* qstats,
                           pprg_call_stats* cstats);
/* power_push(g, s, alpha, lambda, cfg) push.hpp:105-107, push.cpp:151-206;
 * scan_threshold < 0 means the default n/4 (types.hpp:25). epoch_r_max_out
 * (optional, epoch_num doubles) = PowerPushTrace::epoch_r_max. */
int pprg_power_push(pprg_graph* g, const uint32_t* sources, uint32_t k, double alpha,
                    double lambda, uint32_t epoch_num, int64_t scan_threshold,
                    double* reserve_out, double* residue_out, uint32_t flags,
                    pprg_query_stats* qstats, pprg_call_stats* cstats, double* epoch_r_max_out);

/* ---- vertex-partitioned power_push (BASELINE configs[4]) ------
 * One session per (part, source block) on a graph resident on this part's
 * GPU. Part p of nparts owns the pull-sweep rows [node_lo, node_hi), cut at
 * row-aligned tiles so every part holds ~m/nparts in-edges (every part
 * computes the same cut). The caller moves data between parts:
 *   begin -> (nparts > 1) broadcast part 0's x, resum -> all-reduce(partial_sums,
 *   2*64 doubles) -> start
 *   while need_sweeps: all-gather y row slices [lo*C, hi*C) (C = columns)
 *                      -> sweep -> all-reduce(counters, 5*C doubles, device)
 *                      -> advance(summed counters, host) until done
 *   finish -> all-reduce(residue_sums) = exact r_sum per source.
 * The epoch rule is power_push's (push.cpp:168-197): r_sum = 1 - alpha*sum(x)
 * and the push counters come from every part, so all parts take identical
 * decisions. finish writes this part's rows [node_lo, node_hi) of the
 * query-major outputs (k x n) and leaves other rows untouched. */
/* Per-column global-phase state and the host epoch rule the sessions use
 * (push.cpp:168-197 restated over summed counters; host-only, no GPU). */
typedef struct {
  double r_sum;
  double D;        /* (1 - alpha) * sum of x over dead ends */
  int32_t epoch;
  int32_t done;
  uint32_t sweeps;
  uint64_t pushes;
} pprg_column_state;
int pprg_epoch_init(pprg_column_state* cols, uint32_t columns, const double* sum_x,
                    const double* sum_dead_x, const double* epoch_lambda, uint32_t epoch_num,
                    double alpha, int* need_sweeps);
/* summed = [pushed mass | edge pushes | node pushes | dead-end mass | pushed out-degree] x columns */
int pprg_epoch_advance(pprg_column_state* cols, uint32_t columns, const double* summed,
                       const double* epoch_lambda, uint32_t epoch_num, double alpha, int* done);

int pprg_part_begin(pprg_graph* g, uint32_t nparts, uint32_t part, const uint32_t* sources,
                    uint32_t k, double alpha, double lambda, uint32_t epoch_num,
                    int64_t scan_threshold, double* partial_sums, uint64_t* node_lo,
                    uint64_t* node_hi, pprg_part** out);
int pprg_part_start(pprg_part* p, const double* summed, int* need_sweeps);
/* device pointers: y [n * columns] (interleaved u*columns + c) and counters [5 * columns] */
int pprg_part_buffers(pprg_part* p, double** y, uint32_t* columns, double** counters);
/* The local queue phase (push.cpp:163-166) is level-synchronous with fp64
 * atomics, so two parts running it need not stop in the same state. A
 * multi-part query therefore adopts ONE part's result: the caller copies
 * part 0's x [n * columns] (device pointer from pprg_part_local_x) into every
 * other part's x, then calls pprg_part_resum to recompute that part's
 * partial_sums before the all-reduce that feeds pprg_part_start. */
int pprg_part_local_x(pprg_part* p, double** x);
int pprg_part_resum(pprg_part* p, double* partial_sums);
/* one global sweep over this part's rows; local_counters (host, optional) gets a copy */
int pprg_part_sweep(pprg_part* p, double* local_counters);
int pprg_part_advance(pprg_part* p, const double* summed, int* done);
int pprg_part_finish(pprg_part* p, double* reserve_out, double* residue_out, uint32_t flags,
                     double* residue_sums);
int pprg_part_stats(const pprg_part* p, pprg_query_stats* qstats, pprg_call_stats* cstats);
void pprg_part_destroy(pprg_part* p);
/* Fused exchange (instead of the y all-gather): the sweep kernel stores every
 * pushed y row of this part straight into the peers' y buffers (other GPUs'
 * buffers over NVLink via the IPC calls below, or other parts' buffers on the
 * same device). Set before pprg_part_start; up to 15 peers. With peers set
 * the per-sweep y exchange is skipped (counters are still all-reduced, which
 * also orders every part's sweep before the next). */
int pprg_part_set_peers(pprg_part* p, double* const* peer_y, uint32_t npeers);
int pprg_part_ipc_handle(pprg_part* p, void* handle /* 64 bytes, cudaIpcMemHandle_t */);
int pprg_ipc_open(int device, const void* handle, void** ptr);
int pprg_ipc_close(int device, void* ptr);

/* Columns (sources) per device block for a k-source call: the batch width the
 * engines use (a power of two, padding columns inert). Not in the reference. */
int pprg_block_columns(const pprg_graph* g, uint32_t k, uint32_t* out);
/* Which kernel runs the global phase (push.cpp:168-197) of an unobserved
 * k-source power_push call on this graph: *out = 1 for the delta sweeps
 * (k_dsweeps: explicit residues, 16-bit per-sweep shares; wide blocks whose
 * gather operand is far beyond L2, or PPRG_DELTA=1), 0 for k_sweeps (cumulative
 * y rows). Results obey the same bounds either way. Not in the reference. */
int pprg_uses_delta_sweeps(const pprg_graph* g, uint32_t k, int* out);

/* One high-precision query with its progress series: the reference's
 * run_high_precision + CheckpointRecorder (sweep.cpp:25-61), recorded at
 * global-sweep / iteration / frontier-level granularity (pushes = cumulative
 * edge pushes, r_sum after that step, time_ns since the call started). FIFO
 * uses r_max = lambda / m_eff and power_push the default config, as
 * sweep.cpp:55-60. *count = points written (<= capacity). */
#define PPRG_ALGO_POWITR 0
#define PPRG_ALGO_SIMFWDPUSH 1
#define PPRG_ALGO_FIFO 2
#define PPRG_ALGO_POWERPUSH 3
typedef struct {
  uint64_t pushes;
  double r_sum;
  uint64_t time_ns;
} pprg_checkpoint;
int pprg_run_traced(pprg_graph* g, int algo, uint32_t source, double alpha, double lambda,
                    double* estimates_out, pprg_query_stats* qstats, pprg_checkpoint* points,
                    uint32_t capacity, uint32_t* count);

/* One single-source query with a step observer (PushObserver, push.hpp:62-70,
 * at step granularity): after every frontier level, global sweep or
 * iteration, cb receives the full reserve / residue (host, n doubles each,
 * valid during the call), r_sum and the cumulative edge pushes. param is
 * lambda, or r_max for PPRG_ALGO_FIFO (with lambda_stop, <= 0 = none);
 * epoch_num / scan_threshold as pprg_power_push (0 / -1 = defaults). */
typedef void (*pprg_step_callback)(void* user, const double* reserve, const double* residue,
                                   double r_sum, uint64_t pushes, uint32_t step);
int pprg_run_observed(pprg_graph* g, int algo, uint32_t source, double alpha, double param,
                      double lambda_stop, uint32_t epoch_num, int64_t scan_threshold,
                      double* reserve_out, double* residue_out, pprg_query_stats* qstats,
                      pprg_step_callback cb, void* user);

/* ground_truth(g, s, alpha) metrics.hpp:41, metrics.cpp:44-55: the answer at
 * lambda = 1e-17 (r_sum <= 1e-17 on exit), for k sources; graphs with
 * n <= 2000 are cross-checked against an independent engine (l1 <= 1e-12,
 * PPRG_EINTERNAL otherwise). estimates_out is required. */
int pprg_ground_truth(pprg_graph* g, const uint32_t* sources, uint32_t k, double alpha,
                      double* estimates_out, uint32_t flags, pprg_query_stats* qstats,
                      pprg_call_stats* cstats);

/* refine(g, s, alpha, r_max, state) push.hpp:118-119, push.cpp:208-222, on k
 * caller states (reserve / residue, k x n query-major, updated in place):
 * every active node in id order, drained until no residue exceeds
 * deg_eff * r_max; qstats pushes = the refine's pushes, r_sum = exact. */
int pprg_refine(pprg_graph* g, const uint32_t* sources, uint32_t k, double alpha, double r_max,
                double* reserve_inout, double* residue_inout, uint32_t flags,
                pprg_query_stats* qstats, pprg_call_stats* cstats);

/* ---- SpeedPPR (speedppr.hpp, walk_index.hpp) ------------------------------- */
/* compute_walk_budget(n, eps, mu) speedppr.hpp:16-17 */
int pprg_walk_budget(uint64_t n, double epsilon, double mu, uint64_t* out);
/* build_index(g, alpha, seed) walk_index.hpp:50, walk_index.cpp:44-54; Philox
 * walks keyed (seed, slot) — rng-id PPRG_RNG_PHILOX4X32_10. */
int pprg_index_build(pprg_graph* g, double alpha, uint64_t seed, pprg_index** out);
/* WalkIndex(alpha, seed, rng_id, offsets, endpoints) walk_index.hpp:23-24 (offsets
 * must equal the graph's out-offsets). */
int pprg_index_from_host(pprg_graph* g, double alpha, uint64_t seed, const uint32_t* endpoints,
                         pprg_index** out);
int pprg_index_export(const pprg_index* idx, uint32_t* endpoints);
/* load_index / save_index walk_index.hpp:52-56, walk_index.cpp:57-104, device-
 * direct; load also runs check_compatible(g) (walk_index.cpp:36-42). Files
 * carry rng-id PPRG_RNG_PHILOX4X32_10; other ids are "unknown generator id". */
int pprg_index_load(pprg_graph* g, const char* path, pprg_index** out);
int pprg_index_save(const pprg_index* idx, const char* path);
void pprg_index_destroy(pprg_index* idx);
/* speedppr_query(g, s, cfg, index) speedppr.hpp:37-38, speedppr.cpp:74-111;
 * mu <= 0 means 1/n; idx may be NULL. */
int pprg_speedppr(pprg_graph* g, const pprg_index* idx, const uint32_t* sources, uint32_t k,
                  double alpha, double epsilon, double mu, uint64_t seed, double* estimates_out,
                  uint32_t flags, pprg_query_stats* qstats, pprg_call_stats* cstats);
/* monte_carlo_phase(g, s, alpha, state, W, [index,] rng) speedppr.hpp:24-30,
 * speedppr.cpp:23-72, on a caller push state of one source (host reserve /
 * residue, n doubles each): every v with residue r > 0 runs ceil(r*W) walks
 * (clamped to deg_eff within the reference's slack, PPRG_EINTERNAL beyond it),
 * each adding r/ceil(r*W) at its terminal; index prefixes are used where v has
 * out-edges. Walks are Philox streams keyed by seed (the reference's Rng
 * stream cannot be reproduced in parallel). */
int pprg_monte_carlo(pprg_graph* g, const pprg_index* idx, uint32_t source, double alpha,
                     uint64_t walk_budget, uint64_t seed, const double* reserve,
                     const double* residue, double* estimates_out, uint64_t* walks_out);
/* random_walk(g, start, source, alpha, rng) walk_index.hpp:12 for a batch of
 * (start_i, k_i, v_i) walk ids under one tag (test hook for the walk stream). */
int pprg_walk_terminals(pprg_graph* g, const uint32_t* starts, const uint32_t* ks,
                        const uint32_t* vs, uint64_t count, uint32_t source, uint32_t tag,
                        double alpha, uint64_t seed, uint32_t* out);

/* Wait until every host-output copy issued by earlier calls on g has landed. */
int pprg_graph_sync(pprg_graph* g);

/* ---- device buffers for device-resident outputs (bench / zero-copy) ------- */
int pprg_device_alloc(int device, uint64_t bytes, void** out);
int pprg_device_free(int device, void* p);
/* Page-locked host buffers for result vectors: device-to-host copies into
 * them run at full link speed and overlap the next block's compute. */
int pprg_host_alloc(uint64_t bytes, void** out);
int pprg_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
