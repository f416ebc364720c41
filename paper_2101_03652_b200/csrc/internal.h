// Internal C++ interfaces of the engine (not exported; the C ABI in
// include/pprg.h is the boundary).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace pprg {

// Row-aligned tile of the transpose for the pull sweeps: rows [r0, r0+nr)
// with their contiguous in-edges [e0, e0+ne); or, for a row with more in-edges
// than a tile holds ("hub"), piece `piece` of `npieces` of that row.
struct TileDesc {
  uint64_t e0;
  uint32_t ne, r0, nr, hub, piece, npieces;
};

// Device-resident immutable graph. The out-CSR is the canonical, reference-
// identical layout (graph.hpp:44-46: u64 offsets, u32 neighbours, dead-end
// list); the transpose and the tile map are derived internal layouts for the
// pull sweeps.
struct Graph {
  int device = 0;
  int sm_count = 148;
  uint64_t n = 0, m = 0, n_dead = 0;
  DevBuf<uint64_t> off;       // out offsets [n+1]
  DevBuf<uint32_t> nbr;       // out neighbours [m]
  DevBuf<uint32_t> deg;       // out-degree [n] (0 = dead end)
  DevBuf<double> inv_deg;     // 1 / effective degree [n]
  DevBuf<uint32_t> dead;      // dead-end ids ascending [n_dead]
  DevBuf<uint64_t> in_off;    // transpose offsets [n+1] (lazy)
  DevBuf<uint32_t> in_nbr;    // transpose neighbours [m], ascending per row
  // rows of the transpose with in-degree > 0 (the others never receive mass)
  uint64_t n_rows = 0;
  DevBuf<uint64_t> cin_off;   // [n_rows+1] offsets of the compacted rows into in_nbr
  DevBuf<uint32_t> cin_row;   // [n_rows] node id of compacted row
  DevBuf<uint32_t> cin_deg;   // [n_rows] out-degree of the compacted row's node
  DevBuf<double> cin_inv;     // [n_rows] 1 / effective out-degree
  std::map<uint32_t, DevBuf<uint2>> tile_d;      // per tile size: (first row, rows) of tile j
  std::map<uint32_t, DevBuf<uint32_t>> tile_split;  // per tile size: compact rows spanning tiles
  std::mutex mu;
  cudaStream_t stream = nullptr;
  // ---- execution lanes (concurrent queries from many host
  // threads, each on its own stream and scratch). A query takes one lane:
  // its stream, its workspaces, and a 1/nlanes share of every persistent
  // kernel's resident blocks, so the lanes' cooperative kernels always fit on
  // the device together. Column blocks of >= 4 columns take every lane (the
  // whole device); graphs of >= PPRG_LANE_MAX_M in-edges have one lane.
  struct Lane {
    cudaStream_t stream = nullptr;  // lanes[0] uses `stream`
    cudaEvent_t done = nullptr;     // recorded when the lane is released
    bool busy = false;
  };
  std::vector<Lane> lanes;
  std::mutex lane_mu;
  std::condition_variable lane_cv;
  int exclusive_waiters = 0;
  std::recursive_mutex build_mu;  // lazily derived structures (transpose, tile plans)

  ~Graph();
  void finish_build();  // deg / inv_deg / dead-ends from off; validates
  void ensure_transpose();
  const uint2* tile_desc(uint32_t edges_per_tile, uint64_t* ntiles);
  const uint32_t* split_rows(uint32_t edges_per_tile, uint64_t* count);
  struct Plan {
    DevBuf<TileDesc> tiles;
    std::vector<TileDesc> host;  // same list (partition cuts)
    uint64_t ntiles = 0, nhubs = 0;
  };
  std::map<uint64_t, Plan> plans;  // key: (T << 32) | RMAX
  // rows packed while a tile holds <= max_edges in-edges and <= max_rows rows; a
  // row longer than max_edges is a tile of its own, and a row longer than
  // hub_edges (default max_edges) is cut into pieces of hub_edges edges
  const Plan& tile_plan(uint32_t max_edges, uint32_t max_rows, uint32_t hub_edges = 0);
  uint64_t m_eff() const { return m + n_dead; }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) PPRG_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

std::unique_ptr<Graph> graph_from_csr(const uint64_t* h_off, const uint32_t* h_nbr, uint64_t n,
                                      int device);
std::unique_ptr<Graph> graph_from_edges(const uint64_t* h_pairs, uint64_t count, int device);
std::unique_ptr<Graph> graph_rmat(int scale, uint64_t edge_factor, double a, double b, double c,
                                  uint64_t seed, int device, std::vector<uint64_t>* h_edges_out);
std::unique_ptr<Graph> graph_chung_lu(uint64_t n_raw, uint64_t draws, double beta, uint64_t seed,
                                      int device, std::vector<uint64_t>* h_edges_out);

// ---- queries --------------------------------------------------------------
struct ColumnStats {
  double r_sum = 0;
  uint64_t pushes = 0;
  uint64_t walks = 0;
  uint32_t sweeps = 0;        // global-phase sweeps (powerpush) / iterations (powitr)
  uint32_t local_levels = 0;  // frontier levels of the local (queue) phase
  int used_scan_phase = 0;
};

struct CallStats {
  double device_ms = 0;       // events around the whole device section
  double sweep_ms = 0;        // events around the persistent global-sweep kernel(s)
  double local_ms = 0;        // local (queue) phase incl. its exact r_sum
  double final_ms = 0;        // final explicit-residue pass
  uint64_t alg_bytes = 0;     // SURVEY 8(d) algorithmic bytes of the global sweeps
  uint64_t sweep_launches = 0;
  uint32_t max_sweeps = 0;
  uint32_t kernel_launches = 0;
};

struct Outputs {  // host or device pointers (k x n, query-major); any may be null
  double* reserve = nullptr;
  double* residue = nullptr;
  bool on_device = false;
  bool async_host = false;  // return before the last host copies land (graph_sync waits)
};
void graph_sync(Graph& g);  // wait for every pending host-output copy of g
// Small device->host read-back through mapped pinned memory (no copy engine),
// synchronous on st; counted in t_readback_kernels.
void d2h_small(void* dst, const void* src, size_t bytes, cudaStream_t st);
extern thread_local uint64_t t_readback_kernels;

enum class Engine { PowerPush, PowItr, SimFwdPush, Fifo };

void run_push_engine(Graph& g, Engine eng, const uint32_t* sources, uint32_t k, double alpha,
                     double lambda, uint32_t epoch_num, int64_t scan_threshold, double r_max_fifo,
                     double lambda_stop_fifo, const Outputs& out, ColumnStats* cols,
                     CallStats* call);

// Interleaved [u*K + c] state left in the graph workspace by the SpeedPPR push
// stage (x = pushed mass, res = explicit residues after refine).
struct PushView {
  int K = 0;
  uint32_t k = 0;
  double* x = nullptr;
  double* res = nullptr;
  const uint32_t* d_src = nullptr;
  std::vector<uint32_t> src;
};
uint32_t block_width(uint64_t n, uint32_t k);
bool delta_block(Graph& g, uint32_t k);  // the global phase of a k-source block runs as delta sweeps
void refine_state(Graph& g, const uint32_t* sources, uint32_t k, double alpha, double r_max,
                  double* reserve, double* residue, bool on_device, ColumnStats* cols,
                  CallStats* call);  // padded columns per block for k queries
void speedppr_push_stage(Graph& g, const uint32_t* sources, uint32_t k, double alpha,
                         double lambda, double r_max, ColumnStats* cols, CallStats* call,
                         PushView* view);

// The lane the calling thread's query runs on (set by LaneGuard).
struct LaneCtx {
  int lane;
  cudaStream_t stream;
  double frac;  // share of a persistent kernel's resident blocks
};
extern thread_local const LaneCtx* t_lane;
inline cudaStream_t qstream(const Graph& g) { return t_lane ? t_lane->stream : g.stream; }
inline int qlane() { return t_lane ? t_lane->lane : 0; }
// Acquire a lane (exclusive: all of them) for the scope of one query call.
class LaneGuard {
 public:
  LaneGuard(Graph& g, bool exclusive);
  ~LaneGuard();
  LaneGuard(const LaneGuard&) = delete;
  LaneGuard& operator=(const LaneGuard&) = delete;

 private:
  Graph& g_;
  bool all_;
  LaneCtx ctx_;
  const LaneCtx* prev_;
};

// Progress trace of a traced single-source call (the reference's
// CheckpointRecorder, sweep.hpp:30-45, at sweep / level granularity). A
// thread-local sink, set by pprg_run_traced for the duration of one call.
struct TracePoint {
  uint64_t pushes;
  double r_sum;
  uint64_t time_ns;
};
struct TraceSink {
  std::vector<TracePoint> pts;
  uint64_t host_t0 = 0;    // steady-clock ns at the call start
  uint64_t dev_t0 = 0;     // %globaltimer at the call start
};
extern thread_local TraceSink* g_trace;

// Step observer of an observed single-source call (the reference's
// PushObserver, push.hpp:62-70, at step granularity: after every frontier
// level, global sweep or iteration the full reserve / residue are copied to
// the host and handed to `cb`).
typedef void (*StepCallback)(void* user, const double* reserve, const double* residue,
                             double r_sum, uint64_t pushes, uint32_t step);
struct StepSink {
  StepCallback cb = nullptr;
  void* user = nullptr;
  uint32_t step = 0;
  std::vector<double> hr, hq;
};
extern thread_local StepSink* g_obs;
// Deterministic mode of the current call (PPRG_DETERMINISTIC): bitwise-
// reproducible results, set by the C ABI for the duration of one call.
extern thread_local bool t_det;
struct DetScope {
  bool prev;
  explicit DetScope(bool on) : prev(t_det) { t_det = on; }
  ~DetScope() { t_det = prev; }
};
uint64_t host_now_ns();
uint64_t device_now_ns(Graph& g);

// Per-column global-phase state (layout = pprg_column_state).
struct ColInit {
  double r_sum;
  double D;
  int epoch;
  int done;
  uint32_t sweeps;
  uint64_t pushes;
};
bool epoch_init(ColInit* st, int K, const double* sum_x, const double* sum_dead_x,
                const double* lam, uint32_t E, double alpha);
bool epoch_advance(ColInit* st, int K, const double* summed, const double* lam, uint32_t E,
                   double alpha);

// Vertex-partitioned PowerPush session (push.cu; BASELINE configs[4]).
struct PartSession;
PartSession* part_begin(Graph& g, uint32_t nparts, uint32_t part, const uint32_t* sources,
                        uint32_t k, double alpha, double lambda, uint32_t E, int64_t scan_threshold,
                        double* partial_host, uint64_t* lo_out, uint64_t* hi_out);
bool part_start(PartSession* s, const double* summed);
void part_sweep(PartSession* s, double* local_host);
bool part_advance(PartSession* s, const double* summed);
void part_finish(PartSession* s, double* reserve, double* residue, bool on_device, double* rpart);
void part_stats(const PartSession* s, ColumnStats* cols, CallStats* call);
double* part_y(PartSession* s, uint32_t* K);
double* part_counters(PartSession* s);
double* part_x(PartSession* s);
void part_resum(PartSession* s, double* partial_host);
int part_device(const PartSession* s);
void part_set_peers(PartSession* s, double* const* peer_y, uint32_t npeers);
void part_destroy(PartSession* s);

struct WalkIndex {
  int device = 0;
  double alpha = 0;
  uint64_t seed = 0;
  uint64_t m = 0;
  DevBuf<uint32_t> endpoints;  // [m], slice v = [off[v], off[v+1])
};

std::unique_ptr<Graph> graph_load_cache(const std::string& path, int device);
void graph_save_cache(Graph& g, const std::string& path);
std::unique_ptr<WalkIndex> index_build(Graph& g, double alpha, uint64_t seed);
std::unique_ptr<WalkIndex> index_load(Graph& g, const std::string& path);
void monte_carlo(Graph& g, const WalkIndex* idx, uint32_t s, double alpha, uint64_t W, uint64_t seed,
                 const double* h_reserve, const double* h_residue, double* h_est, uint64_t* walks);
void index_save(Graph& g, const WalkIndex& w, const std::string& path);
std::unique_ptr<WalkIndex> index_from_host(Graph& g, double alpha, uint64_t seed,
                                           const uint32_t* h_endpoints);
void speedppr(Graph& g, const WalkIndex* idx, const uint32_t* sources, uint32_t k, double alpha,
              double epsilon, double mu, uint64_t seed, double* est_out, bool out_on_device,
              ColumnStats* cols, CallStats* call);
// Walk terminals of walks (k_i, v_i) from start_i under tag (test hook).
void walk_terminals(Graph& g, const uint32_t* h_start, const uint32_t* h_k, const uint32_t* h_v,
                    uint64_t count, uint32_t source, uint32_t tag, double alpha, uint64_t seed,
                    uint32_t* h_out);

}  // namespace pprg
