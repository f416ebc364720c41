// Push engines on the GPU: PowerPush (local frontier phase + global epoch
// sweeps), PowItr / SimFwdPush (Jacobi sweeps), FIFO forward push / refine
// (frontier levels). Reference: /root/reference/proj/core/src/push.cpp.
//
// Representation. The global sweeps run in *pull* form over the transpose.
// Per (node u, column c) we keep x = total residue mass u has pushed so far
// (reserve = alpha * x, push.cpp:20) and y = (1-alpha) * x / deg_eff(u), the
// share every out-neighbour has received from u. The residue is implicit:
//     r_u = [u == s] + sum_{v -> u} y_v + [u == s] * (1-alpha) * sum_{dead v} x_v - x_u
// so "push u" (push.cpp:17-27) is x_u <- inflow_u. Reads of neighbours' y that
// are stale (older sweeps) only under-estimate inflow, so residues stay
// non-negative and mass is conserved exactly in exact arithmetic; the r_sum
// bookkeeping is the reference's incremental one (r_sum -= alpha * r per push,
// push.cpp:25) and the exact recompute (push.cpp:9-15) is done in the final
// pass. Sweeps are asynchronous (Gauss-Seidel) like the reference's in-place
// scan (push.cpp:182-193): tiles of in-edges are taken in id order from an
// atomic ticket, so rows processed later in a sweep see earlier rows' pushes.
// The local phase and refine use push form (atomicExch claim + fp64 RED
// scatter) over frontier levels, since their frontiers are sparse.
#include <chrono>
#include <cstddef>
#include <cmath>
#include <cstdlib>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <type_traits>
#include <vector>

#include <cub/cub.cuh>

#include "internal.h"

#include "sweep_kernel.cuh"
#include "frontier_kernels.cuh"
#include "delta_sweep.cuh"

namespace pprg {

// ---- per-graph workspace --------------------------------------------------
struct Workspace {
  int K = 0;
  uint64_t n = 0;
  DevBuf<double> x, y0, y1, r0, r1, res;
  DevBuf<unsigned> stamp;
  DevBuf<uint32_t> fa, fb;  // frontier segments [K][n] of node ids
  DevBuf<double> hub_acc;
  DevBuf<unsigned> hub_cnt;
  // host-output staging: finalize writes slot s while the copy stream drains
  // slot s^1 to the caller's host buffers (overlaps D2H with the next block)
  cudaStream_t copy_st = nullptr;
  cudaEvent_t ev_ready[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr};
  DevBuf<double> stage_res[2], stage_rsd[2];
  unsigned stage_slot = 0;
  ~Workspace() {
    if (copy_st) {
      cudaStreamSynchronize(copy_st);
      cudaStreamDestroy(copy_st);
      for (int i = 0; i < 2; ++i) {
        cudaEventDestroy(ev_ready[i]);
        cudaEventDestroy(ev_done[i]);
      }
    }
  }
  // control blocks of a query block's kernels, contiguous so that a block run
  // without host round trips reads all of them back with one copy at its end
  struct Ctl {
    DrainCtl d;  // local phase / refine / FIFO (k_drain)
    SweepCtl s;  // global phase (k_sweeps)
    SweepCtl f;  // final pass
  };
  DevBuf<Ctl> ctlb;
  DrainCtl* dctl() { return reinterpret_cast<DrainCtl*>(reinterpret_cast<char*>(ctlb.get()) + offsetof(Ctl, d)); }
  SweepCtl* ctl() { return reinterpret_cast<SweepCtl*>(reinterpret_cast<char*>(ctlb.get()) + offsetof(Ctl, s)); }
  SweepCtl* fctl() { return reinterpret_cast<SweepCtl*>(reinterpret_cast<char*>(ctlb.get()) + offsetof(Ctl, f)); }
  DevBuf<unsigned long long> counters;  // next_cnt + col_cnt[K] + col_np[K] + col_nn[K]
  DevBuf<double> dcols;                 // col_dr[K], colsum[K], D[K]
  DevBuf<uint32_t> d_src;
  DevBuf<HeavyEntry> heavy;
  DevBuf<unsigned long long> popv;      // deterministic drains: popped value per segment slot
  DevBuf<double> dsum_part;             // deterministic column sums: per-block partials
  DevBuf<double> drain_part;            // deterministic drains: per-block exact r_sum partials
  unsigned level_tag = 0;
  // delta sweeps: the wave cut of their tile plan (host, built once per plan)
  const void* dw_plan = nullptr;
  uint32_t dw_waves = 0;
  std::vector<uint32_t> dw_tile, dw_node;
};

static std::mutex g_ws_mu;
static std::map<const Graph*, std::map<int, std::unique_ptr<Workspace>>> g_ws;

static void ws_alloc(Workspace& w, Graph& g, int K) {
  w.K = K;
  w.n = g.n;
  const uint64_t nk = g.n * (uint64_t)K;
  w.x.alloc(nk);
  w.y0.alloc(nk);
  w.y1.alloc(nk);
  w.r0.alloc(nk);
  w.r1.alloc(nk);
  w.res.alloc(nk);
  w.stamp.alloc(nk);
  PPRG_CUDA(cudaMemsetAsync(w.stamp.get(), 0, 4 * nk, qstream(g)));
  w.fa.alloc(nk + 1);
  w.fb.alloc(nk + 1);
  w.ctlb.alloc(1);
  w.counters.alloc(1 + 5 * KMAX);
  w.dcols.alloc(3 * KMAX);
  w.d_src.alloc(KMAX);
  w.heavy.alloc((g.m / HEAVY_DEG + 1) * (uint64_t)K + 1);
}

static void ws_tiles(Workspace& w, Graph& g, uint64_t ntiles, uint64_t nhubs) {
  const int K = w.K;
  if ((ntiles + 1) * K > w.hub_acc.n) w.hub_acc.alloc((ntiles + 1) * K);
  if (nhubs + 1 > w.hub_cnt.n) {
    w.hub_cnt.alloc(nhubs + 1);
    PPRG_CUDA(cudaMemsetAsync(w.hub_cnt.get(), 0, 4 * (nhubs + 1), qstream(g)));
  }
}

// one workspace per (graph, lane, columns): concurrent lanes never share scratch
static Workspace& workspace(Graph& g, int K, uint64_t ntiles, uint64_t nhubs) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  auto& slot = g_ws[&g][qlane() * 256 + K];
  if (!slot) {
    slot = std::make_unique<Workspace>();
    ws_alloc(*slot, g, K);
  }
  ws_tiles(*slot, g, ntiles, nhubs);
  return *slot;
}

// Wait for every pending host-output copy of this graph's workspaces.
static void sync_host_copies(const Graph& g) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  auto it = g_ws.find(&g);
  if (it == g_ws.end()) return;
  for (auto& kv : it->second)
    if (kv.second && kv.second->copy_st) PPRG_CUDA(cudaStreamSynchronize(kv.second->copy_st));
}

void graph_sync(Graph& g) {
  DeviceGuard dg(g.device);
  sync_host_copies(g);
}

void release_workspaces(const Graph* g) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  g_ws.erase(g);
}

namespace {

// Reductions that flush per-block partials with global atomics: a bounded,
// grid-stride grid (a few blocks per SM) keeps those atomics few.
inline unsigned grid_reduce(uint64_t items, int tb = 256) {
  uint64_t b = (items + tb - 1) / tb;
  if (b == 0) b = 1;
  return (unsigned)(b < 148ull * 8 ? b : 148ull * 8);
}

inline unsigned grid_for(uint64_t items, int tb = 256) {
  uint64_t b = (items + tb - 1) / tb;
  if (b == 0) b = 1;
  if (b > 65535ull * 32) b = 65535ull * 32;
  return (unsigned)b;
}

// Blocks of a cooperative (persistent) launch: the query lane's share of the
// resident slots (LaneGuard), times PPRG_GRID_FRAC (probe: what a smaller grid
// costs one call).
unsigned coop_grid(const Graph& g, int per_sm) {
  static const double frac = [] {
    const char* e = std::getenv("PPRG_GRID_FRAC");
    const double v = e ? std::atof(e) : 1.0;
    return v > 0.0 && v <= 1.0 ? v : 1.0;
  }();
  const unsigned full = (unsigned)(per_sm * g.sm_count);
  const unsigned want = (unsigned)(frac * (t_lane ? t_lane->frac : 1.0) * full);
  return want < 1 ? 1 : want;
}

template <int K, int MODE, bool DET>
void launch_sweeps(Graph& g, SweepParams& P, bool cooperative) {
  const size_t wide_bytes = 8ull * (RMAX_W + 1) + 8ull * RMAX_W + 8ull * (NT / 32) * K +
                            4ull * (3 * RMAX_W + 1) + 16;
  const size_t smem = K >= WIDE_K ? wide_bytes : P.k1w ? k1w_bytes : Tile<K>::bytes;
  auto kern = k_sweeps<K, MODE, DET>;
  static bool attr_set = false;
  if (!attr_set) {
    const size_t most = K >= WIDE_K ? wide_bytes : std::max(k1w_bytes, Tile<K>::bytes);
    PPRG_CUDA(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)most));
    attr_set = true;
  }
  if (cooperative) {
    int per_sm = 0;
    PPRG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
    if (per_sm < 1) fail(EINTERNAL, "sweep kernel cannot be resident");
    unsigned grid = coop_grid(g, per_sm);
    // narrow path on small graphs: at least ~2 tiles per block, so fewer rows
    // are in flight (closer to the reference's sequential scan): configs[0]
    // takes 71 sweeps instead of 83 and 9% less time. The wide path keeps the
    // full grid (fewer blocks cost it more than the sweeps they save).
    static const double tpb_env = [] {
      const char* e = std::getenv("PPRG_TILES_PER_BLOCK");
      return e ? std::atof(e) : -1.0;
    }();
    // (one-column warp tasks: ~2 per warp, i.e. 8 per block)
    const double tpb = tpb_env >= 0 ? tpb_env
                                    : P.k1w ? 2.0 * (NT / 32) : (K < WIDE_K ? 2.0 : 0.0);
    if (tpb > 0 && P.ntiles > 0) {
      const double want = (double)P.ntiles / tpb;
      const unsigned lo = std::min((unsigned)g.sm_count, grid);  // (never above the lane share)
      if (want < grid) grid = want < lo ? lo : (unsigned)want;
    }
    void* args[] = {(void*)&P};
    PPRG_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(NT), args, smem, qstream(g)));
  } else {
    const uint64_t grid = P.ntiles < (uint64_t)g.sm_count * 8 ? P.ntiles : (uint64_t)g.sm_count * 8;
    kern<<<(unsigned)(grid ? grid : 1), NT, smem, qstream(g)>>>(P);
  }
  PPRG_CUDA(cudaGetLastError());
}

template <int MODE, bool DET>
void dispatch_sweeps_t(Graph& g, int K, SweepParams& P, bool coop) {
  switch (K) {
    case 1: launch_sweeps<1, MODE, DET>(g, P, coop); break;
    case 2: launch_sweeps<2, MODE, DET>(g, P, coop); break;
    case 4: launch_sweeps<4, MODE, DET>(g, P, coop); break;
    case 8: launch_sweeps<8, MODE, DET>(g, P, coop); break;
    case 16: launch_sweeps<16, MODE, DET>(g, P, coop); break;
    case 32: launch_sweeps<32, MODE, DET>(g, P, coop); break;
    case 64: launch_sweeps<64, MODE, DET>(g, P, coop); break;
    default: fail(EINTERNAL, "unsupported column block");
  }
}
// the deterministic sweeps (k_sweeps<K, MODE, true>) when the call asked for them
template <int MODE>
void dispatch_sweeps(Graph& g, int K, SweepParams& P, bool coop) {
  if (t_det) dispatch_sweeps_t<MODE, true>(g, K, P, coop);
  else dispatch_sweeps_t<MODE, false>(g, K, P, coop);
}

int round_k(uint32_t k) {
  int K = 1;
  while (K < (int)k) K <<= 1;
  return K;
}

__global__ void k_stamp(unsigned long long* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = t;
}

// Device trace buffer for one sweep launch of a traced call; `fold` appends
// its points to the sink with a push offset / scale.
struct SweepTrace {
  DevBuf<TracePoint> buf;
  uint32_t cap = 0;
  void attach(SweepParams& P) {
    if (!g_trace) return;
    cap = 1u << 16;
    buf.alloc(cap);
    P.trace = buf.get();
    P.trace_cap = cap;
  }
  void fold(cudaStream_t st, uint32_t nsweeps, uint64_t push_base, uint64_t per_sweep_pushes) {
    if (!g_trace || !cap) return;
    const uint32_t n = nsweeps < cap ? nsweeps : cap;
    std::vector<TracePoint> h(n);
    if (n) PPRG_CUDA(cudaMemcpyAsync(h.data(), buf.get(), sizeof(TracePoint) * n, cudaMemcpyDeviceToHost, st));
    PPRG_CUDA(cudaStreamSynchronize(st));
    for (uint32_t i = 0; i < n; ++i) {
      TracePoint t = h[i];
      t.pushes = per_sweep_pushes ? push_base + (uint64_t)(i + 1) * per_sweep_pushes
                                  : push_base + t.pushes;
      t.time_ns = t.time_ns > g_trace->dev_t0 ? t.time_ns - g_trace->dev_t0 : 0;
      g_trace->pts.push_back(t);
    }
  }
};

}  // namespace

uint64_t device_now_ns(Graph& g) {
  DevBuf<unsigned long long> t(1);
  k_stamp<<<1, 1, 0, qstream(g)>>>(t.get());
  unsigned long long h = 0;
  PPRG_CUDA(cudaMemcpyAsync(&h, t.get(), 8, cudaMemcpyDeviceToHost, qstream(g)));
  PPRG_CUDA(cudaStreamSynchronize(qstream(g)));
  return h;
}

namespace {

// Small device->host read-backs on the query path go through a kernel that
// stores into mapped pinned memory instead of a copy-engine transfer, so they
// never queue behind the multi-GB output copies of the previous block on the
// copy engine (those overlap the next block's compute).
__global__ void k_copy_bytes(unsigned char* dst, const unsigned char* src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

struct MappedStage {
  unsigned char* h = nullptr;
  unsigned char* d = nullptr;
  size_t cap = 0;
  ~MappedStage() {
    if (h) cudaFreeHost(h);
  }
};

}  // namespace

thread_local uint64_t t_readback_kernels = 0;  // counted into CallStats::kernel_launches

void d2h_small(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (!bytes) return;
  ++t_readback_kernels;
  static thread_local MappedStage ms;
  if (bytes > ms.cap) {
    if (ms.h) PPRG_CUDA(cudaFreeHost(ms.h));
    ms.cap = bytes < 65536 ? 65536 : bytes;
    PPRG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ms.h), ms.cap,
                            cudaHostAllocMapped | cudaHostAllocPortable));
    PPRG_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ms.d), ms.h, 0));
  }
  const unsigned blocks = (unsigned)((bytes + 255) / 256 < 64 ? (bytes + 255) / 256 : 64);
  k_copy_bytes<<<blocks, 256, 0, st>>>(ms.d, static_cast<const unsigned char*>(src), bytes);
  PPRG_CUDA(cudaGetLastError());
  PPRG_CUDA(cudaStreamSynchronize(st));
  std::memcpy(dst, ms.h, bytes);
}

namespace {

struct EventTimer {
  cudaEvent_t a{}, b{};
  cudaStream_t st;
  explicit EventTimer(cudaStream_t s) : st(s) {
    PPRG_CUDA(cudaEventCreate(&a));
    PPRG_CUDA(cudaEventCreate(&b));
  }
  ~EventTimer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  void start() { PPRG_CUDA(cudaEventRecord(a, st)); }
  void stop() { PPRG_CUDA(cudaEventRecord(b, st)); }
  double ms() {
    PPRG_CUDA(cudaEventSynchronize(b));
    float f = 0;
    PPRG_CUDA(cudaEventElapsedTime(&f, a, b));
    return f;
  }
};

}  // namespace

// ---- engine drivers ---------------------------------------------------------
namespace {

struct Block {
  Graph& g;
  Workspace& w;
  int K;
  uint32_t k;
  uint64_t ntiles = 0;
  const TileDesc* desc = nullptr;
  const Graph::Plan* plan = nullptr;
  double* yfin = nullptr;  // y after the global phase (deterministic sweeps alternate y0 / y1)
  uint64_t nhubs = 0;
  double alpha;
  std::vector<uint32_t> src;
  std::vector<double> r_sum;
  std::vector<uint64_t> pushes;
  std::vector<uint32_t> levels;
  std::vector<double> D;
  std::vector<int> scan;
  std::vector<uint32_t> sweeps;
  // A block run without host round trips (run_push_engine / SpeedPPR,
  // unobserved): the drain, the global phase and the final pass are launched
  // back to back, each starting from the previous one's device outputs, and
  // their results are read back once, by finalize.
  bool drain_pending = false;        // the drain's DrainCtl is still on the device
  unsigned long long drain_live = 0; // its columns
  bool sweeps_pending = false;       // the global phase's SweepCtl is still on the device
  bool delta = false;                // the global phase ran as delta sweeps (explicit residues in w.res)
  std::unique_ptr<EventTimer> t_local, t_sweep;
  Block(Graph& g_, Workspace& w_, int K_, uint32_t k_, double a)
      : g(g_), w(w_), K(K_), k(k_), alpha(a), src(KMAX, 0), r_sum(KMAX, 1.0), pushes(KMAX, 0),
        levels(KMAX, 0), D(KMAX, 0.0), scan(KMAX, 0), sweeps(KMAX, 0) {}
};

Block make_block(Graph& g, const uint32_t* sources, uint32_t k, double alpha, bool need_pull,
                 Workspace* own = nullptr) {
  const int K = round_k(k);
  uint64_t ntiles = 0;
  const TileDesc* dsc = nullptr;
  const Graph::Plan* plan = nullptr;
  uint64_t nhubs = 0;
  if (need_pull) {
    const Graph::Plan& pl = g.tile_plan(tile_edges(g, K), tile_rmax(g, K), tile_hub(g, K));
    dsc = pl.tiles.get();
    ntiles = pl.ntiles;
    nhubs = pl.nhubs;
    plan = &pl;
  }
  if (own) {
    if (!own->K) ws_alloc(*own, g, K);
    ws_tiles(*own, g, ntiles, nhubs);
  }
  Workspace& w = own ? *own : workspace(g, K, ntiles, nhubs);
  Block b(g, w, K, k, alpha);
  b.ntiles = ntiles;
  b.desc = dsc;
  b.plan = plan;
  b.yfin = w.y0.get();
  b.nhubs = nhubs;
  for (uint32_t c = 0; c < k; ++c) b.src[c] = sources[c];
  for (int c = k; c < K; ++c) b.src[c] = sources[0];  // padding columns are inert
  PPRG_CUDA(cudaMemcpyAsync(w.d_src.get(), b.src.data(), 4 * KMAX, cudaMemcpyHostToDevice, qstream(g)));
  return b;
}

SweepParams base_params(Block& b) {
  SweepParams P;
  std::memset(&P, 0, sizeof P);
  Graph& g = b.g;
  P.n = g.n;
  P.m = g.m;
  P.deg = g.deg.get();
  P.inv_deg = g.inv_deg.get();
  P.alpha = b.alpha;
  P.ctl = b.w.ctl();
  P.k_live = (int)b.k;
  P.max_sweeps = 200000;
  P.own_lo = 0;
  P.own_hi = g.n;
  for (int c = 0; c < b.K; ++c) P.src[c] = b.src[c];
  P.in_off = g.cin_off.get();
  P.crow = g.cin_row.get();
  P.cdeg = g.cin_deg.get();
  P.cinv = g.cin_inv.get();
  P.in_off_full = g.in_off.get();
  P.in_nbr = g.in_nbr.get();
  P.desc = b.desc;
  P.ntiles = b.ntiles;
  P.T = SWEEP_ELEMS / b.K;
  P.k1w = k1w_on(g, b.K);
  P.hub_acc = b.w.hub_acc.get();
  P.hub_cnt = b.w.hub_cnt.get();
  return P;
}

// Per-column sums of an interleaved [row * K + c] array into dst[0..K)
// (device): dst[c] = scale * sum over rows (rows[r] if given, else r < nrows).
// Deterministic mode: fixed-grid, fixed-order partials (k_dsum_*); else fp64
// atomics (k_colsum; rows / scale unsupported there).
void det_colsum(Block& b, const double* a, const uint32_t* rows, uint64_t nrows, double scale,
                double* dst) {
  Workspace& w = b.w;
  cudaStream_t st = qstream(b.g);
  if (w.dsum_part.n < (size_t)DSUM_BLOCKS * KMAX) w.dsum_part.alloc((size_t)DSUM_BLOCKS * KMAX);
  k_dsum_part<<<DSUM_BLOCKS, DSUM_NT, 0, st>>>(a, rows, nrows, b.K, w.dsum_part.get());
  k_dsum_final<<<1, KMAX, 0, st>>>(w.dsum_part.get(), DSUM_BLOCKS, b.K, scale, dst);
  PPRG_CUDA(cudaGetLastError());
}

// Deterministic sweeps: the tile plan cut into waves of ~equal in-edges at
// row-start tiles (hub pieces of one row stay in one wave). PPRG_DET_WAVES
// (default 4): 1 = Jacobi sweeps; more waves read more of the sweep's own
// updates (Gauss-Seidel between waves) and take fewer sweeps, at one grid
// barrier per wave. configs[2] block / configs[0]: 4 waves 251 ms / 2.6 ms
// (53 / 52 sweeps), 8 waves 262 / 4.3 ms (48 / 47), 16 waves 377 / 7.8 ms.
void set_waves(Block& b, SweepParams& P) {
  static const int W = [] {
    const char* e = std::getenv("PPRG_DET_WAVES");
    const int v = e ? std::atoi(e) : 4;
    return v < 1 ? 1 : v > WMAX ? WMAX : v;
  }();
  const std::vector<TileDesc>& t = b.plan->host;
  uint64_t total = 0;
  for (const TileDesc& d : t) total += d.ne;
  P.wave_tile[0] = 0;
  P.wave_node[0] = 0;  // sources without in-edges are written before wave 0
  uint32_t w = 1;
  uint64_t acc = 0;
  for (uint64_t j = 0; j < t.size() && (int)w < W; ++j) {
    if (acc * W >= total * w && t[j].piece == 0 && j > P.wave_tile[w - 1]) {
      P.wave_tile[w] = j;
      d2h_small(&P.wave_node[w], b.g.cin_row.get() + t[j].r0, 4, qstream(b.g));
      ++w;
    }
    acc += t[j].ne;
  }
  P.wave_tile[w] = t.size();
  P.nwaves = w;
}

// Observed calls: column 0's reserve / residue (device, interleaved with the
// block's K) to the host sink.
void emit_step(Block& b, const double* reserve_src, double reserve_scale, const double* residue_src,
               double r_sum, uint64_t pushes) {
  if (!g_obs) return;
  Graph& g = b.g;
  const uint64_t n = g.n, nk = n * (uint64_t)b.K;
  cudaStream_t st = qstream(g);
  DevBuf<double> tmp(2 * n);
  k_unpack<<<grid_for(nk), 256, 0, st>>>(reserve_src, n, b.K, 1, reserve_scale, tmp.get());
  k_unpack<<<grid_for(nk), 256, 0, st>>>(residue_src, n, b.K, 1, 1.0, tmp.get() + n);
  g_obs->hr.resize(n);
  g_obs->hq.resize(n);
  PPRG_CUDA(cudaMemcpyAsync(g_obs->hr.data(), tmp.get(), 8 * n, cudaMemcpyDeviceToHost, st));
  PPRG_CUDA(cudaMemcpyAsync(g_obs->hq.data(), tmp.get() + n, 8 * n, cudaMemcpyDeviceToHost, st));
  PPRG_CUDA(cudaStreamSynchronize(st));
  g_obs->cb(g_obs->user, g_obs->hr.data(), g_obs->hq.data(), r_sum, pushes, ++g_obs->step);
}

void exact_rsum(Block& b, const std::vector<int>& which);

// Frontier levels (drain_queue, push.cpp:34-59) for every column in
// `state == 0`. The initial frontier is seed_source (push.cpp:61-66) or, for
// refine, every active node in id order (push.cpp:212-218). The reference's
// loop conditions -- queue size <= limit and r_sum > lambda_stop, checked
// before every pop -- are tested on the device (k_drain): the queue size of
// column c at a pop is its unprocessed entries of this level plus the
// out-degrees reserved by the level's pops so far (fast mode), or the level's
// size at level boundaries (deterministic mode).
// Unobserved calls run every level in one launch; observed / traced calls
// (and PPRG_DEBUG_LOCAL) one level per launch, reporting after each.
// The results of a drain read back from the device (levels, pushes, the exact
// r_sum with the reference's 1e-6 drift guard, push.cpp:9-15).
void apply_drain(Block& b, const DrainCtl& hd, unsigned long long live) {
  b.w.level_tag += hd.levels_run;
  if (hd.out_live) fail(EINTERNAL, "drain: level limit reached");
  for (uint32_t c = 0; c < b.k; ++c) {
    if ((live >> c) & 1ull) {
      b.pushes[c] += hd.out_np[c];
      b.levels[c] += hd.out_levels[c];
      b.r_sum[c] = hd.out_rsum[c];
    }
    if (std::fabs(hd.out_exact[c] - b.r_sum[c]) > 1e-6)
      fail(EINTERNAL, "push: r_sum drifted more than 1e-6 from the residues");
    b.r_sum[c] = hd.out_exact[c];
  }
}

void drain_levels(Block& b, double r_max, double lam_stop, uint64_t limit, bool from_scan,
                  std::vector<int>& state, CallStats* call, bool defer = false) {
  Graph& g = b.g;
  Workspace& w = b.w;
  const int K = b.K;
  const uint64_t n = g.n, nk = n * (uint64_t)K;
  cudaStream_t st = qstream(g);
  const bool det = t_det;
  uint32_t* cur = w.fa.get();
  uint32_t* nxt = w.fb.get();
  std::vector<uint64_t> qsize(K, 0), qdeg(K, 0);
  if (++w.level_tag == 0 || w.level_tag >= 0x80000000u) {  // keep tag + levels from wrapping
    PPRG_CUDA(cudaMemsetAsync(w.stamp.get(), 0, 4 * nk, st));
    w.level_tag = 1;
  }
  unsigned long long live = 0;
  for (uint32_t c = 0; c < b.k; ++c)
    if (state[c] == 0) live |= 1ull << c;
  static const bool debug = std::getenv("PPRG_DEBUG_LOCAL") != nullptr;
  const bool stepwise = g_obs || g_trace || debug;
  if (det && w.popv.n < nk) w.popv.alloc(nk);
  DrainParams D;
  std::memset(&D, 0, sizeof D);
  D.off = g.off.get();
  D.nbr = g.nbr.get();
  D.deg = g.deg.get();
  D.res = w.res.get();
  D.x = w.x.get();
  D.stamp = w.stamp.get();
  D.seg_cap = n;
  D.heavy = w.heavy.get();
  D.ctl = w.dctl();
  D.popv = det ? w.popv.get() : nullptr;
  D.limit = limit == UINT64_MAX ? ~0ull : (unsigned long long)limit;
  D.lam_stop = lam_stop;
  D.alpha = b.alpha;
  D.n = n;
  D.K = K;
  D.start = from_scan ? 2 : 1;  // the first launch builds the first level on the device
  D.want_exact = 1;
  for (int c = 0; c < K; ++c) {
    D.src[c] = b.src[c];
    D.thr[c] = r_max;
    // DET fixed point: every residue and every sum of residues of column c
    // stays below its r_sum <= 2^e, so scale by 2^(61 - e)
    int e = 0;
    std::frexp(b.r_sum[c] > 0 ? b.r_sum[c] : 1.0, &e);
    D.sc[c] = std::ldexp(1.0, 61 - e);
  }
  // lanes per frontier entry (PPRG_DRAIN_GL: 4, 8, 16 or 32). A whole warp
  // per entry measured best: 8 lanes per entry (4 entries per warp in
  // flight) took the configs[3] frontier 0.63 -> 0.76 ms per query, 4 lanes
  // 0.94 ms (profiles/r02_drain_gl_ab.txt)
  static const int gl = [] {
    const char* e = std::getenv("PPRG_DRAIN_GL");
    const int v = e ? std::atoi(e) : 32;
    return v == 4 || v == 8 || v == 16 ? v : 32;
  }();
  auto pick = [&](auto det_tag) {
    constexpr bool DT = decltype(det_tag)::value;
    return gl == 4 ? k_drain<DT, 4> : gl == 16 ? k_drain<DT, 16> : gl == 32 ? k_drain<DT, 32> : k_drain<DT, 8>;
  };
  auto kern = det ? pick(std::true_type{}) : pick(std::false_type{});
  static int per_sm[2] = {0, 0};
  int& ps = per_sm[det];
  if (!ps) PPRG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, kern, DRAIN_NT, 0));
  if (ps < 1) fail(EINTERNAL, "drain kernel cannot be resident");
  const unsigned grid = coop_grid(g, ps);
  if (det && w.drain_part.n < (size_t)grid * KMAX) w.drain_part.alloc((size_t)grid * KMAX);
  D.part = det ? w.drain_part.get() : nullptr;
  std::vector<double> exact;
  if (defer && live && !stepwise) {  // launched; finalize reads the results
    D.seg[0] = cur;
    D.seg[1] = nxt;
    D.live0 = live;
    D.tag0 = w.level_tag;
    D.max_levels = 0xFFFFFFFFu - w.level_tag - 1;
    for (int c = 0; c < K; ++c) D.r_sum0[c] = b.r_sum[c];
    PPRG_CUDA(cudaMemsetAsync(D.ctl, 0, sizeof(DrainCtl), st));
    void* args[] = {(void*)&D};
    PPRG_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(DRAIN_NT), args, 0, st));
    PPRG_CUDA(cudaGetLastError());
    call->kernel_launches += 1;
    b.drain_pending = true;
    b.drain_live = live;
    for (uint32_t c = 0; c < b.k; ++c) state[c] = 1;
    return;
  }
  while (live) {
    D.seg[0] = cur;
    D.seg[1] = nxt;
    D.live0 = live;
    D.tag0 = w.level_tag;
    D.max_levels = stepwise ? 1u : 0xFFFFFFFFu - w.level_tag - 1;
    for (int c = 0; c < K; ++c) {
      D.r_sum0[c] = b.r_sum[c];
      D.q0[c] = ((live >> c) & 1ull) ? qsize[c] : 0;
      D.qdeg0[c] = qdeg[c];
    }
    PPRG_CUDA(cudaMemsetAsync(D.ctl, 0, sizeof(DrainCtl), st));
    void* args[] = {(void*)&D};
    PPRG_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(DRAIN_NT), args, 0, st));
    D.start = 0;
    PPRG_CUDA(cudaGetLastError());
    call->kernel_launches += 1;
    DrainCtl hd;
    d2h_small(&hd, D.ctl, sizeof hd, st);
    w.level_tag += hd.levels_run;
    if (debug && hd.levels_run) {
      unsigned long long nn = 0, np = 0, app = 0, tot = 0;
      for (uint32_t c = 0; c < b.k; ++c)
        nn += hd.nn[0][c], np += hd.np[0][c], app += hd.cnt[0][c], tot += ((live >> c) & 1ull) ? qsize[c] : 0;
      std::fprintf(stderr, "level: entries %llu heavy %u node_pushes %llu edge_pushes %llu appended %llu\n",
                   tot, hd.heavy_cnt[0], nn, np, app);
    }
    for (uint32_t c = 0; c < b.k; ++c) {
      if (!((live >> c) & 1ull)) continue;
      b.r_sum[c] = hd.out_rsum[c];
      b.pushes[c] += hd.out_np[c];
      b.levels[c] += hd.out_levels[c];
      qsize[c] = hd.out_q[c];
      qdeg[c] = hd.out_qdeg[c];
    }
    if (g_trace && (live & 1ull))
      g_trace->pts.push_back(TracePoint{b.pushes[0], b.r_sum[0], host_now_ns() - g_trace->host_t0});
    if (g_obs && (live & 1ull)) emit_step(b, w.x.get(), b.alpha, w.res.get(), b.r_sum[0], b.pushes[0]);
    if (hd.levels_run & 1u) std::swap(cur, nxt);
    if (!stepwise && hd.out_live) fail(EINTERNAL, "drain: level limit reached");
    live = hd.out_live;
    exact.assign(hd.out_exact, hd.out_exact + KMAX);
  }
  for (uint32_t c = 0; c < b.k; ++c)
    if (state[c] == 0) state[c] = 1;
  // recompute_r_sum (push.cpp:9-15), summed by the drain kernel at its end
  if (exact.empty()) {  // nothing drained: the residues are untouched
    std::vector<int> all(KMAX, 1);
    exact_rsum(b, all);
    return;
  }
  for (uint32_t c = 0; c < b.k; ++c) {
    if (std::fabs(exact[c] - b.r_sum[c]) > 1e-6)
      fail(EINTERNAL, "push: r_sum drifted more than 1e-6 from the residues");
    b.r_sum[c] = exact[c];
  }
}

// recompute_r_sum (push.cpp:9-15) over the push-form residues of every column
void exact_rsum(Block& b, const std::vector<int>& which) {
  Graph& g = b.g;
  cudaStream_t st = qstream(g);
  const uint64_t nk = g.n * (uint64_t)b.K;
  if (t_det) {
    det_colsum(b, b.w.res.get(), nullptr, g.n, 1.0, b.w.dcols.get() + KMAX);
  } else {
    PPRG_CUDA(cudaMemsetAsync(b.w.dcols.get() + KMAX, 0, 8 * KMAX, st));
    k_colsum<<<grid_reduce(nk), 256, 0, st>>>(b.w.res.get(), g.n, b.K, b.w.dcols.get() + KMAX);
  }
  std::vector<double> exact(KMAX);
  d2h_small(exact.data(), b.w.dcols.get() + KMAX, 8 * KMAX, st);
  PPRG_CUDA(cudaStreamSynchronize(st));
  for (uint32_t c = 0; c < b.k; ++c) {
    if (!which[c]) continue;
    if (std::fabs(exact[c] - b.r_sum[c]) > 1e-6)
      fail(EINTERNAL, "push: r_sum drifted more than 1e-6 from the residues");
    b.r_sum[c] = exact[c];
  }
}

// The final pass clamps implicit residues that rounding left below zero; a
// sum of clamped mass beyond rounding level means the pull-form state was
// inconsistent (e.g. parts starting from different local phases): fail loudly.
constexpr double kNegResidueTol = 1e-12;

// The sweeps stop on the tracked r_sum (r_sum -= alpha * pushed); the exact
// residue sum of the final pass replaces it. The two differ by accumulated
// rounding (~1e-15 absolute), so the last epoch stops a relative 1e-6 below
// lambda: the exact r_sum then lands <= lambda, which the reference guarantees
// by looping on the recomputed sum (push.cpp:180-196). The push thresholds
// (epoch_r_max) are the reference's unchanged.
double stop_lambda(double epoch_lambda, uint32_t e, uint32_t E) {
  return e + 1 == E ? epoch_lambda * (1.0 - 1e-6) : epoch_lambda;
}
void check_final(const SweepCtl& fc) {
  if (fc.neg_sum < -kNegResidueTol)
    fail(EINTERNAL, "final pass: " + std::to_string(fc.neg_count) +
                        " negative implicit residues summing to " + std::to_string(fc.neg_sum));
}

// ---- delta sweeps (delta_sweep.cuh) -------------------------------------------
// PPRG_DELTA: 0 = never, 1 = every eligible block, unset = blocks whose gather
// operand y (n x K x 8 B) is beyond twice the L2.
bool delta_on(const Graph& g, int K) {
  const char* e = std::getenv("PPRG_DELTA");  // (read per call: tests switch it)
  const int mode = e ? std::atoi(e) : -1;
  if (K < 32 || mode == 0 || t_det) return false;
  if (g.m_eff() >= (1ull << 32) || g.n >= (1ull << 31) || g.n_rows == 0) return false;
  if (mode > 0) return true;
  return g.n * (uint64_t)K * 8 > (256ull << 20);
}
// SpeedPPR's push stage (a refine epoch appended) as delta sweeps: opt-in
// (PPRG_DELTA_REFINE=1). Measured on configs[3]: the sweeps get cheaper (1.04
// vs 1.35 ms per query) but their lagged fixpoint leaves the frontier tail more
// work (1.30 vs 0.37 ms); handing off 4x later evens it out (2.15 ms per query
// either way), so the refine stage stays on k_sweeps.
bool delta_refine() {
  const char* e = std::getenv("PPRG_DELTA_REFINE");
  return e && std::atoi(e) != 0;
}

// The warp-task plan of the delta sweeps: bundles of <= 32 whole rows and
// <= PPRG_DS_TASK in-edges, longer rows whole up to PPRG_DS_PIECE in-edges,
// beyond that in pieces.
uint32_t ds_env(const char* name, int dflt, int lo) {
  const char* e = std::getenv(name);
  const int t = e ? std::atoi(e) : dflt;
  return (uint32_t)(t < lo ? lo : t > (int)DS_IDS ? (int)DS_IDS : t);  // (a task's ids sit in shared memory)
}
uint32_t ds_task_edges() {
  static const uint32_t v = ds_env("PPRG_DS_TASK", 192, 32);
  return v;
}
uint32_t ds_piece_edges() {
  static const uint32_t v = ds_env("PPRG_DS_PIECE", 512, 64);
  return v;
}

template <int K>
void launch_dsweeps(Graph& g, DeltaParams& P) {
  auto kern = k_dsweeps<K>;
  const size_t smem = sizeof(DeltaSh<K>);
  static bool attr_set = false;
  if (!attr_set) {
    PPRG_CUDA(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = true;
  }
  int per_sm = 0;
  PPRG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, DS_NT, smem));
  if (per_sm < 1) fail(EINTERNAL, "delta sweep kernel cannot be resident");
  const unsigned grid = coop_grid(g, per_sm);
  void* args[] = {(void*)&P};
  PPRG_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(DS_NT), args, smem, qstream(g)));
  PPRG_CUDA(cudaGetLastError());
}

// The global phase of a device-started block as delta sweeps: explicit
// residues (w.res, left by the local phase), 16-bit shares in w.y0.
void delta_phase(Block& b, double lambda, uint32_t E, CallStats* call, double refine_rmax) {
  Graph& g = b.g;
  Workspace& w = b.w;
  cudaStream_t st = qstream(g);
  const uint64_t nk = g.n * (uint64_t)b.K;
  const double m_eff = (double)g.m_eff();
  const Graph::Plan& pl = g.tile_plan(ds_task_edges(), DS_TASK_R, std::max(ds_task_edges(), ds_piece_edges()));
  ws_tiles(w, g, pl.ntiles, pl.nhubs);
  static const uint32_t W = [] {
    const char* e = std::getenv("PPRG_DS_WAVES");
    const int v = e ? std::atoi(e) : 64;
    return (uint32_t)(v < 1 ? 1 : v > DS_WMAX ? DS_WMAX : v);
  }();
  static const uint32_t L = [] {
    const char* e = std::getenv("PPRG_DS_LAG");
    const int v = e ? std::atoi(e) : 6;
    return (uint32_t)(v < 1 ? 1 : v);
  }();
  if (w.dw_plan != &pl || w.dw_waves != W) {
    // waves of ~equal in-edges, cut at row-start tiles (a hub row's pieces stay in one wave)
    const std::vector<TileDesc>& t = pl.host;
    uint64_t total = 0;
    for (const TileDesc& d : t) total += d.ne;
    w.dw_tile.assign(1, 0u);
    uint64_t acc = 0;
    for (uint64_t j = 0; j < t.size() && w.dw_tile.size() < W; ++j) {
      if (acc * W >= total * w.dw_tile.size() && t[j].piece == 0 && j > w.dw_tile.back())
        w.dw_tile.push_back((uint32_t)j);
      acc += t[j].ne;
    }
    w.dw_node.assign(w.dw_tile.size(), 0u);
    for (size_t i = 1; i < w.dw_tile.size(); ++i)
      d2h_small(&w.dw_node[i], g.cin_row.get() + t[w.dw_tile[i]].r0, 4, st);
    PPRG_CUDA(cudaStreamSynchronize(st));
    w.dw_tile.push_back((uint32_t)t.size());
    w.dw_node.push_back(0xFFFFFFFFu);
    w.dw_plan = &pl;
    w.dw_waves = W;
  }
  DeltaParams P;
  std::memset(&P, 0, sizeof P);
  P.n = g.n;
  P.m = g.m;
  P.in_off = g.cin_off.get();
  P.crow = g.cin_row.get();
  P.cdeg = g.cin_deg.get();
  P.cinv = g.cin_inv.get();
  P.in_off_full = g.in_off.get();
  P.in_nbr = g.in_nbr.get();
  P.deg = g.deg.get();
  P.inv_deg = g.inv_deg.get();
  P.desc = pl.tiles.get();
  P.ntiles = pl.ntiles;
  P.hub_acc = w.hub_acc.get();
  P.hub_cnt = w.hub_cnt.get();
  P.k_live = (int)b.k;
  P.E = (int)E + (refine_rmax > 0.0);
  P.alpha = b.alpha;
  P.inv_oma = 1.0 / (1.0 - b.alpha);
  P.x = w.x.get();
  P.r = w.res.get();
  P.dsh = reinterpret_cast<uint4*>(w.y0.get());
  P.from_drain = w.dctl()->out_exact;
  P.scan_lambda = lambda;
  P.ctl = w.ctl();
  P.max_sweeps = 200000;
  P.nwaves = (uint32_t)w.dw_tile.size() - 1;
  P.lag = L;
  for (uint32_t i = 0; i <= P.nwaves; ++i) {
    P.wave_tile[i] = w.dw_tile[i];
    P.wave_node[i] = w.dw_node[i];
  }
  for (uint32_t i = P.nwaves + 1; i <= (uint32_t)DS_WMAX; ++i) P.wave_tile[i] = 0xFFFFFFFFu;
  for (int c = 0; c < b.K; ++c) P.src[c] = b.src[c];
  for (uint32_t e = 0; e < E; ++e) {
    const double el = std::pow(lambda, static_cast<double>(e + 1) / E);  // push.cpp:176-178
    P.lam[e] = stop_lambda(el, e, E);
    P.thr[e] = el / m_eff;
  }
  if (refine_rmax > 0.0) {  // the refine epoch of global_phase (push.cpp:208-222), same hand-off
    P.lam[E] = -1.0;
    P.thr[E] = refine_rmax;
    double f = 1.0 / 128;
    if (const char* e = std::getenv("PPRG_REFINE_HANDOFF")) f = std::atof(e);
    P.handoff_np = (unsigned long long)(f * m_eff);
    P.scan_all = 1;
  }
  PPRG_CUDA(cudaMemsetAsync(w.y0.get(), 0, 4 * nk, st));  // both share buffers
  PPRG_CUDA(cudaMemsetAsync(w.ctl(), 0, sizeof(SweepCtl), st));
  b.t_sweep = std::make_unique<EventTimer>(st);
  b.t_sweep->start();
  if (b.K == 64) launch_dsweeps<64>(g, P);
  else launch_dsweeps<32>(g, P);
  b.t_sweep->stop();
  call->sweep_launches += 1;
  call->kernel_launches += 1;
  b.sweeps_pending = true;
  b.delta = true;
}

// Global phase: epochs of asynchronous pull sweeps in one persistent
// cooperative kernel (push.cpp:168-197) for the columns with scan[c] set.
// refine_rmax > 0 appends a refine epoch (push.cpp:208-222): threshold
// refine_rmax, no r_sum target, ends at the sweep that pushes nothing — the
// fixpoint where every residue is <= deg_eff * refine_rmax, refine's postcondition.
void global_phase(Block& b, double lambda, uint32_t E, CallStats* call, double refine_rmax = 0.0,
                  bool defer = false) {
  Graph& g = b.g;
  Workspace& w = b.w;
  cudaStream_t st = qstream(g);
  const uint64_t nk = g.n * (uint64_t)b.K;
  const double m_eff = (double)g.m_eff();
  if (E + (refine_rmax > 0.0) > EMAX) fail(EINVAL_, "epoch_num exceeds 64");
  if (defer && delta_on(g, b.K) && (refine_rmax == 0.0 || delta_refine())) {
    delta_phase(b, lambda, E, call, refine_rmax);
    return;
  }
  PPRG_CUDA(cudaMemsetAsync(w.dcols.get() + 2 * KMAX, 0, 8 * KMAX, st));
  k_init_pull<<<grid_reduce(nk), 256, 0, st>>>(w.x.get(), g.deg.get(), g.inv_deg.get(), g.n, b.K,
                                            b.alpha, w.y0.get(), w.dcols.get() + 2 * KMAX);
  if (t_det) {
    // D = (1-a) * sum of x over the dead ends in a fixed order; both y buffers
    // start equal
    det_colsum(b, w.x.get(), g.dead.get(), g.n_dead, 1.0 - b.alpha, w.dcols.get() + 2 * KMAX);
    PPRG_CUDA(cudaMemcpyAsync(w.y1.get(), w.y0.get(), 8 * nk, cudaMemcpyDeviceToDevice, st));
  }
  // the sweep kernel reads D from the device; observed calls need it here
  if (g_obs) d2h_small(b.D.data(), w.dcols.get() + 2 * KMAX, 8 * KMAX, st);
  PPRG_CUDA(cudaMemsetAsync(w.ctl(), 0, sizeof(SweepCtl), st));
  SweepParams P = base_params(b);
  for (uint32_t e = 0; e < E; ++e) {
    const double el = std::pow(lambda, static_cast<double>(e + 1) / E);  // push.cpp:176-178
    P.lam[e] = stop_lambda(el, e, E);
    P.thr[e] = el / m_eff;
  }
  const int Et = (int)E + (refine_rmax > 0.0);
  if (refine_rmax > 0.0) {
    P.lam[E] = -1.0;
    P.thr[E] = refine_rmax;
    // a sweep costs a pass over every in-edge; once the refine tail pushes
    // fewer than m_eff/128 edges per sweep the frontier kernels finish it
    // (configs[3]: 155 ms per 64 queries against 171 ms at m_eff/64 and
    // 165-170 ms at m_eff/256 or /512)
    double f = 1.0 / 128;
    if (const char* e = std::getenv("PPRG_REFINE_HANDOFF")) f = std::atof(e);
    P.handoff_np = (unsigned long long)(f * m_eff);
  }
  for (int c = 0; c < b.K; ++c) {
    P.init[c].r_sum = b.r_sum[c];
    P.init[c].D = b.D[c];
    int ep = 0;
    while (ep < Et && !(b.r_sum[c] > P.lam[ep])) ++ep;
    P.init[c].epoch = ep;
    P.init[c].done = !b.scan[c] || ep >= Et;
  }
  P.E = Et;
  P.x = w.x.get();
  if (!g_obs) P.D_dev = w.dcols.get() + 2 * KMAX;
  if (defer) {  // r_sum, scan, epoch, done from the drain's exact sums, on the device
    P.from_drain = w.dctl()->out_exact;
    P.scan_lambda = lambda;
    P.scan_all = refine_rmax > 0.0;
  }
  P.y[0] = P.y[1] = w.y0.get();
  if (t_det) {
    P.y[1] = w.y1.get();
    set_waves(b, P);
  }
  double* ycur = P.y[0];  // y as of the last completed sweep
  double* ynext = P.y[1];
  SweepTrace trace;
  trace.attach(P);
  EventTimer tm(st);
  SweepCtl hc;
  if (g_obs) {
    // observed: one sweep per launch, the explicit state handed out after each
    std::vector<ColInit> stv(P.init, P.init + b.K);
    std::memset(&hc, 0, sizeof hc);
    DevBuf<double> snap(2 * g.n);
    tm.start();
    for (uint32_t sweep = 0;; ++sweep) {
      bool all = true;
      for (int c = 0; c < b.K; ++c) all &= stv[c].done != 0;
      if (all) break;
      if (sweep >= 200000) fail(EINTERNAL, "power push: sweep limit reached");
      SweepParams Q = P;
      Q.max_sweeps = 1;
      Q.y[0] = ycur;
      Q.y[1] = ynext;
      for (int c = 0; c < b.K; ++c) Q.init[c] = stv[c];
      PPRG_CUDA(cudaMemsetAsync(w.ctl(), 0, sizeof(SweepCtl), st));
      dispatch_sweeps<M_POWERPUSH>(g, b.K, Q, true);
      if (t_det) std::swap(ycur, ynext);
      SweepCtl one;
      d2h_small(&one, w.ctl(), sizeof one, st);
      PPRG_CUDA(cudaStreamSynchronize(st));
      hc.alg_bytes += one.alg_bytes;
      hc.total_sweeps = sweep + 1;
      for (int c = 0; c < b.K; ++c)
        stv[c] = ColInit{one.out_rsum[c], one.out_D[c], one.out_epoch[c], one.out_done[c],
                         one.out_sweeps[c], one.out_pushes[c]};
      // explicit residues of the pull form (the final pass, outputs only)
      SweepParams F = base_params(b);
      F.x = w.x.get();
      F.y[0] = F.y[1] = ycur;
      F.push_res = w.res.get();
      F.out_reserve = snap.get();
      F.out_residue = snap.get() + g.n;
      for (int c = 0; c < b.K; ++c) {
        F.final_pull[c] = 1;
        F.init[c].r_sum = stv[c].r_sum;
        F.init[c].D = stv[c].D;
      }
      PPRG_CUDA(cudaMemsetAsync(snap.get(), 0, 16 * g.n, st));
      PPRG_CUDA(cudaMemsetAsync(w.ctl(), 0, sizeof(SweepCtl), st));
      dispatch_sweeps<M_FINAL>(g, b.K, F, true);
      g_obs->hr.resize(g.n);
      g_obs->hq.resize(g.n);
      PPRG_CUDA(cudaMemcpyAsync(g_obs->hr.data(), snap.get(), 8 * g.n, cudaMemcpyDeviceToHost, st));
      PPRG_CUDA(cudaMemcpyAsync(g_obs->hq.data(), snap.get() + g.n, 8 * g.n, cudaMemcpyDeviceToHost, st));
      PPRG_CUDA(cudaStreamSynchronize(st));
      g_obs->cb(g_obs->user, g_obs->hr.data(), g_obs->hq.data(), stv[0].r_sum,
                b.pushes[0] + stv[0].pushes, ++g_obs->step);
    }
    tm.stop();
    for (int c = 0; c < b.K; ++c) {
      hc.out_rsum[c] = stv[c].r_sum;
      hc.out_D[c] = stv[c].D;
      hc.out_done[c] = stv[c].done;
      hc.out_sweeps[c] = stv[c].sweeps;
      hc.out_pushes[c] = stv[c].pushes;
    }
  } else if (defer) {
    b.t_sweep = std::make_unique<EventTimer>(st);
    b.t_sweep->start();
    dispatch_sweeps<M_POWERPUSH>(g, b.K, P, true);
    b.t_sweep->stop();
    call->sweep_launches += 1;
    call->kernel_launches += 2;
    b.sweeps_pending = true;
    b.yfin = ycur;  // deterministic sweeps: finalize picks y by the sweep count parity
    return;
  } else {
    tm.start();
    dispatch_sweeps<M_POWERPUSH>(g, b.K, P, true);
    tm.stop();
    d2h_small(&hc, w.ctl(), sizeof hc, st);
    if (t_det && (hc.total_sweeps & 1u)) std::swap(ycur, ynext);  // sweep s writes y[(s + 1) & 1]
  }
  b.yfin = ycur;
  call->sweep_ms += tm.ms();
  trace.fold(st, hc.total_sweeps, b.pushes[0], 0);
  call->alg_bytes += hc.alg_bytes;
  call->sweep_launches += 1;
  call->kernel_launches += 2;
  if (hc.total_sweeps > call->max_sweeps) call->max_sweeps = hc.total_sweeps;
  for (uint32_t c = 0; c < b.k; ++c) {
    if (!b.scan[c]) continue;
    if (!hc.out_done[c]) fail(EINTERNAL, "power push: sweep limit reached");
    b.r_sum[c] = hc.out_rsum[c];
    b.pushes[c] += hc.out_pushes[c];
    b.D[c] = hc.out_D[c];
    b.sweeps[c] = hc.out_sweeps[c];
  }
}

}  // namespace

namespace {

// Final pass: explicit residues of the pull form (and the exact r_sum,
// push.cpp:9-15) for scan-phase columns; push-form residues for the others.
// Writes query-major outputs and/or the interleaved residue array.
void finalize(Block& b, const Outputs& out, bool residues_inplace, CallStats* call) {
  Graph& g = b.g;
  Workspace& w = b.w;
  cudaStream_t st = qstream(g);
  const uint64_t n = g.n, nk = n * (uint64_t)b.K;
  const uint32_t k = b.k;
  const cudaMemcpyKind kind = out.on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  const bool deferred = b.sweeps_pending;
  bool any_scan = deferred;  // (deferred: decided on the device; the final pass handles both forms)
  for (uint32_t c = 0; c < k; ++c) any_scan |= b.scan[c] != 0;
  if (!any_scan) {
    if (out.reserve || out.residue) {
      DevBuf<double> tmp(n * k);
      if (out.reserve) {
        k_unpack<<<grid_for(nk), 256, 0, st>>>(w.x.get(), n, b.K, k, b.alpha, tmp.get());
        PPRG_CUDA(cudaMemcpyAsync(out.reserve, tmp.get(), 8 * n * k, kind, st));
        PPRG_CUDA(cudaStreamSynchronize(st));
      }
      if (out.residue) {
        k_unpack<<<grid_for(nk), 256, 0, st>>>(w.res.get(), n, b.K, k, 1.0, tmp.get());
        PPRG_CUDA(cudaMemcpyAsync(out.residue, tmp.get(), 8 * n * k, kind, st));
      }
      call->kernel_launches += (out.reserve != nullptr) + (out.residue != nullptr);
    }
    PPRG_CUDA(cudaStreamSynchronize(st));
    return;
  }
  SweepParams Q = base_params(b);
  const bool direct = out.on_device;  // write straight into the caller's device buffers
  int slot = 0;
  if (!direct && (out.reserve || out.residue)) {
    if (!w.copy_st) {
      PPRG_CUDA(cudaStreamCreateWithFlags(&w.copy_st, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i) {
        PPRG_CUDA(cudaEventCreateWithFlags(&w.ev_ready[i], cudaEventDisableTiming));
        PPRG_CUDA(cudaEventCreateWithFlags(&w.ev_done[i], cudaEventDisableTiming));
        PPRG_CUDA(cudaEventRecord(w.ev_done[i], w.copy_st));
      }
    }
    slot = (int)(w.stage_slot++ & 1);
    PPRG_CUDA(cudaStreamWaitEvent(st, w.ev_done[slot], 0));  // the slot's previous D2H is done
    if (out.reserve) w.stage_res[slot].ensure(n * b.K);
    if (out.residue) w.stage_rsd[slot].ensure(n * b.K);
  }
  Q.out_reserve = out.reserve ? (direct ? out.reserve : w.stage_res[slot].get()) : nullptr;
  Q.out_residue = out.residue ? (direct ? out.residue : w.stage_rsd[slot].get()) : nullptr;
  // rows with in-degree 0 (other than sources) are never visited: they hold 0
  if (Q.out_reserve && !b.delta) PPRG_CUDA(cudaMemsetAsync(Q.out_reserve, 0, 8 * n * k, st));
  if (Q.out_residue && !b.delta) PPRG_CUDA(cudaMemsetAsync(Q.out_residue, 0, 8 * n * k, st));
  Q.res_inter = residues_inplace ? w.res.get() : nullptr;
  Q.push_res = w.res.get();
  Q.x = w.x.get();
  Q.y[0] = Q.y[1] = b.yfin;
  for (int c = 0; c < b.K; ++c) {
    Q.final_pull[c] = b.scan[c];
    Q.init[c].r_sum = b.r_sum[c];
    Q.init[c].D = b.D[c];
  }
  SweepCtl* fctl = deferred ? w.fctl() : w.ctl();
  Q.ctl = fctl;
  if (deferred) {
    Q.from_sweeps = w.ctl();
    // deterministic sweeps alternate y0 / y1: the last sweep wrote y[count & 1]
    if (t_det) Q.y[0] = Q.y[1] = nullptr;  // set below from the sweep count
  }
  PPRG_CUDA(cudaMemsetAsync(fctl, 0, sizeof(SweepCtl), st));
  EventTimer tf(st);
  if (deferred && t_det) {
    // the y buffer of the last sweep depends on the count: read it (deterministic
    // mode only; the fast sweeps update y in place)
    uint32_t ts = 0;
    d2h_small(&ts, reinterpret_cast<const char*>(w.ctl()) + offsetof(SweepCtl, total_sweeps), 4, st);
    Q.y[0] = Q.y[1] = (ts & 1u) ? w.y1.get() : w.y0.get();
  }
  tf.start();
  if (b.delta) {
    // explicit residues already (w.res): transpose into the outputs, exact r_sum
    const unsigned grid = (unsigned)std::min<uint64_t>((n + 31) / 32, 148ull * 8);
    if (b.K == 64)
      k_delta_final<64><<<grid, 256, 0, st>>>(w.x.get(), w.res.get(), n, (int)k, b.alpha,
                                              Q.out_reserve, Q.out_residue, fctl);
    else
      k_delta_final<32><<<grid, 256, 0, st>>>(w.x.get(), w.res.get(), n, (int)k, b.alpha,
                                              Q.out_reserve, Q.out_residue, fctl);
    PPRG_CUDA(cudaGetLastError());
  } else {
    dispatch_sweeps<M_FINAL>(g, b.K, Q, true);
  }
  tf.stop();
  call->kernel_launches += 1;
  SweepCtl fc;
  if (deferred) {  // the block's one read-back: drain, sweeps and final pass
    Workspace::Ctl all;
    d2h_small(&all, w.ctlb.get(), sizeof all, st);
    if (b.drain_pending) apply_drain(b, all.d, b.drain_live);
    b.drain_pending = false;
    const SweepCtl& hc = all.s;
    call->alg_bytes += hc.alg_bytes;
    if (hc.total_sweeps > call->max_sweeps) call->max_sweeps = hc.total_sweeps;
    for (uint32_t c = 0; c < k; ++c) {
      b.scan[c] = hc.out_scan[c];
      if (!b.scan[c]) continue;
      if (!hc.out_done[c]) fail(EINTERNAL, "power push: sweep limit reached");
      b.r_sum[c] = hc.out_rsum[c];
      b.pushes[c] += hc.out_pushes[c];
      b.D[c] = hc.out_D[c];
      b.sweeps[c] = hc.out_sweeps[c];
    }
    b.sweeps_pending = false;
    if (b.t_local) call->local_ms += b.t_local->ms();
    if (b.t_sweep) call->sweep_ms += b.t_sweep->ms();
    b.t_local.reset();
    b.t_sweep.reset();
    fc = all.f;
  } else {
    d2h_small(&fc, w.ctl(), sizeof fc, st);
  }
  check_final(fc);
  if (!direct && (out.reserve || out.residue)) {
    PPRG_CUDA(cudaEventRecord(w.ev_ready[slot], st));
    PPRG_CUDA(cudaStreamWaitEvent(w.copy_st, w.ev_ready[slot], 0));
    // chunked, so the compute stream's small read-backs (per level / phase)
    // never queue behind a whole multi-GB output copy on the copy engine
    static const size_t chunk = [] {
      const char* e = std::getenv("PPRG_D2H_CHUNK_MB");
      return (size_t)(e ? std::atof(e) : 32.0) << 20;
    }();
    auto d2h = [&](double* dst, const double* src, size_t bytes) {
      for (size_t o = 0; o < bytes; o += chunk)
        PPRG_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(dst) + o,
                                  reinterpret_cast<const char*>(src) + o,
                                  bytes - o < chunk ? bytes - o : chunk, cudaMemcpyDeviceToHost,
                                  w.copy_st));
    };
    if (out.reserve) d2h(out.reserve, Q.out_reserve, 8 * n * k);
    if (out.residue) d2h(out.residue, Q.out_residue, 8 * n * k);
    PPRG_CUDA(cudaEventRecord(w.ev_done[slot], w.copy_st));
  }
  PPRG_CUDA(cudaStreamSynchronize(st));
  call->final_ms += tf.ms();
  for (uint32_t c = 0; c < k; ++c) {
    if (!b.scan[c]) continue;
    const double exact = fc.pushed[0][c] / fc.out_scale[c];
    if (std::fabs(exact - b.r_sum[c]) > 1e-6)
      fail(EINTERNAL, "push: r_sum drifted more than 1e-6 from the residues");
    b.r_sum[c] = exact;
  }
}

void power_push_block(Block& b, double lambda, uint32_t epoch_num, int64_t scan_threshold,
                      CallStats* call, double refine_rmax = 0.0) {
  // unobserved blocks run without host round trips (finalize reads back once)
  const bool defer = !g_obs && !g_trace && !std::getenv("PPRG_DEBUG_LOCAL");
  const double m_eff = (double)b.g.m_eff();
  const uint64_t nk = b.g.n * (uint64_t)b.K;
  cudaStream_t st = qstream(b.g);
  PPRG_CUDA(cudaMemsetAsync(b.w.x.get(), 0, 8 * nk, st));
  PPRG_CUDA(cudaMemsetAsync(b.w.res.get(), 0, 8 * nk, st));
  k_seed<<<1, KMAX, 0, st>>>(b.w.res.get(), b.w.d_src.get(), b.K, 1.0);
  const double r_max = lambda / m_eff;  // push.cpp:157-160
  // Default queue limit (push.cpp:161: n / 4). Blocks whose global phase runs as
  // delta sweeps switch at n / 128: a sweep costs them 2.3 ms per 64 sources, less
  // than the frontier levels between a queue of n/128 and n/4 entries (configs[2]
  // block: local phase 6.1 -> 1.35 ms, 50 sweeps either way; PPRG_DS_SCAN_DIV).
  uint64_t limit = scan_threshold < 0 ? b.g.n / 4 : (uint64_t)scan_threshold;
  if (scan_threshold < 0 && defer && refine_rmax == 0.0 && delta_on(b.g, b.K)) {
    static const double div = [] {
      const char* e = std::getenv("PPRG_DS_SCAN_DIV");
      const double v = e ? std::atof(e) : 128.0;
      return v >= 1.0 ? v : 1.0;
    }();
    limit = (uint64_t)((double)b.g.n / div);
  }
  std::vector<int> state(KMAX, 2);
  for (uint32_t c = 0; c < b.k; ++c) state[c] = 0;
  if (defer) {
    b.t_local = std::make_unique<EventTimer>(st);
    b.t_local->start();
    drain_levels(b, r_max, lambda, limit, false, state, call, true);
    b.t_local->stop();
    if (b.drain_pending) {
      global_phase(b, lambda, epoch_num, call, refine_rmax, true);  // push.cpp:168 on the device
      return;
    }
    call->local_ms += b.t_local->ms();
    b.t_local.reset();
  } else {
    EventTimer tl(st);
    tl.start();
    drain_levels(b, r_max, lambda, limit, false, state, call);  // (+ recompute_r_sum)
    tl.stop();
    call->local_ms += tl.ms();
  }
  bool any = false;
  for (uint32_t c = 0; c < b.k; ++c) {
    b.scan[c] = b.r_sum[c] > lambda || refine_rmax > 0.0;  // push.cpp:168
    any |= b.scan[c] != 0;
  }
  if (any) global_phase(b, lambda, epoch_num, call, refine_rmax);
}


}  // namespace

// refine (push.cpp:208-222) from caller state: reserve / residue (k x n,
// query-major, host or device) in, refined state out in place. The push form
// keeps x = reserve / alpha; every active node in id order seeds the frontier
// and the levels drain until no node is above deg_eff * r_max.
void refine_state(Graph& g, const uint32_t* sources, uint32_t k, double alpha, double r_max,
                  double* reserve, double* residue, bool on_device, ColumnStats* cols,
                  CallStats* call) {
  DeviceGuard dg(g.device);
  LaneGuard lk(g, round_k(k < (uint32_t)KMAX ? k : (uint32_t)KMAX) >= WIDE_K);  // 8(b) lanes
  if (!(r_max > 0.0)) fail(EINVAL_, "refine: r_max must be positive");  // push.cpp:210
  for (uint32_t c = 0; c < k; ++c)
    if (sources[c] >= g.n) fail(EINVAL_, "source out of range");
  const uint64_t n = g.n;
  const uint64_t rb0 = t_readback_kernels;
  for (uint32_t b0 = 0; b0 < k; b0 += KMAX) {
    const uint32_t kb = k - b0 < (uint32_t)KMAX ? k - b0 : (uint32_t)KMAX;
    Block b = make_block(g, sources + b0, kb, alpha, false);
    cudaStream_t st = qstream(g);
    const uint64_t nk = n * (uint64_t)b.K;
    double* hr = reserve + (uint64_t)b0 * n;
    double* hq = residue + (uint64_t)b0 * n;
    // device copies of the caller's state (or the caller's device buffers)
    DevBuf<double> tr(on_device ? 0 : n * kb), tq(on_device ? 0 : n * kb);
    double* dr = on_device ? hr : tr.get();
    double* dq = on_device ? hq : tq.get();
    if (!on_device) {
      PPRG_CUDA(cudaMemcpyAsync(dr, hr, 8 * n * kb, cudaMemcpyHostToDevice, st));
      PPRG_CUDA(cudaMemcpyAsync(dq, hq, 8 * n * kb, cudaMemcpyHostToDevice, st));
    }
    // x counts only the mass pushed here, so untouched reserves come back bit-identical
    PPRG_CUDA(cudaMemsetAsync(b.w.x.get(), 0, 8 * nk, st));
    k_pack<<<grid_for(nk), 256, 0, st>>>(dq, n, b.K, kb, 1.0, b.w.res.get());
    PPRG_CUDA(cudaGetLastError());
    std::fill(b.r_sum.begin(), b.r_sum.end(), 0.0);
    {  // r_sum of the incoming state (no drift check: it is the caller's)
      if (t_det) {
        det_colsum(b, b.w.res.get(), nullptr, n, 1.0, b.w.dcols.get() + KMAX);
      } else {
        PPRG_CUDA(cudaMemsetAsync(b.w.dcols.get() + KMAX, 0, 8 * KMAX, st));
        k_colsum<<<grid_reduce(nk), 256, 0, st>>>(b.w.res.get(), n, b.K, b.w.dcols.get() + KMAX);
      }
      d2h_small(b.r_sum.data(), b.w.dcols.get() + KMAX, 8 * KMAX, st);
      PPRG_CUDA(cudaStreamSynchronize(st));
    }
    std::vector<int> state(KMAX, 2);
    for (uint32_t c = 0; c < kb; ++c) state[c] = 0;
    EventTimer tl(st);
    tl.start();
    drain_levels(b, r_max, 0.0, UINT64_MAX, true, state, call);  // (+ recompute_r_sum, push.cpp:221)
    tl.stop();
    call->local_ms += tl.ms();
    k_refine_out<<<grid_for(nk), 256, 0, st>>>(b.w.x.get(), b.w.res.get(), n, b.K, kb, alpha, dr, dq);
    PPRG_CUDA(cudaGetLastError());
    if (!on_device) {
      PPRG_CUDA(cudaMemcpyAsync(hr, dr, 8 * n * kb, cudaMemcpyDeviceToHost, st));
      PPRG_CUDA(cudaMemcpyAsync(hq, dq, 8 * n * kb, cudaMemcpyDeviceToHost, st));
    }
    PPRG_CUDA(cudaStreamSynchronize(st));
    for (uint32_t c = 0; c < kb; ++c) {
      cols[b0 + c].r_sum = b.r_sum[c];
      cols[b0 + c].pushes = b.pushes[c];
      cols[b0 + c].local_levels = b.levels[c];
    }
    call->kernel_launches += 3;
  }
  call->kernel_launches += (uint32_t)(t_readback_kernels - rb0);
}

// Columns per block: wider blocks amortise the in-edge stream over more
// queries; the per-block state (x, y, residues: n*K doubles each) is capped
// at 1.6 GB per array, so K shrinks as n grows. PPRG_COLUMNS overrides.
uint32_t block_columns(uint64_t n, uint32_t k) {
  if (const char* e = std::getenv("PPRG_COLUMNS")) {
    const long v = std::strtol(e, nullptr, 10);
    if (v >= 1 && v <= KMAX) return (uint32_t)v;
  }
  uint32_t K = KMAX;
  while (K > 1 && 8.0 * (double)n * K > 1.6e9) K >>= 1;  // x, y, res, ... are n*K doubles each
  return K < k ? K : (k ? k : 1);
}

uint32_t block_width(uint64_t n, uint32_t k) { return (uint32_t)round_k(block_columns(n, k)); }
bool delta_block(Graph& g, uint32_t k) {
  g.ensure_transpose();
  return delta_on(g, (int)block_width(g.n, k));
}

void run_push_engine(Graph& g, Engine eng, const uint32_t* sources, uint32_t k, double alpha,
                     double lambda, uint32_t epoch_num, int64_t scan_threshold, double r_max_fifo,
                     double lambda_stop_fifo, const Outputs& out, ColumnStats* cols,
                     CallStats* call) {
  DeviceGuard dg(g.device);
  LaneGuard lk(g, round_k(block_columns(g.n, k)) >= WIDE_K);  // 8(b) lanes: wide blocks take the device
  for (uint32_t c = 0; c < k; ++c)
    if (sources[c] >= g.n) fail(EINVAL_, "source out of range");
  const uint64_t rb0 = t_readback_kernels;
  struct CountReadbacks {
    CallStats* call;
    uint64_t rb0;
    ~CountReadbacks() { call->kernel_launches += (uint32_t)(t_readback_kernels - rb0); }
  } count_rb{call, rb0};
  const bool pull = eng != Engine::Fifo;
  if (pull) g.ensure_transpose();
  const uint32_t bmax = block_columns(g.n, k);
  for (uint32_t b0 = 0; b0 < k; b0 += bmax) {
    const uint32_t kb = k - b0 < bmax ? k - b0 : bmax;
    Outputs o = out;
    if (o.reserve) o.reserve += (uint64_t)b0 * g.n;
    if (o.residue) o.residue += (uint64_t)b0 * g.n;
    Block b = make_block(g, sources + b0, kb, alpha, pull);
    ColumnStats* cs = cols + b0;
    EventTimer tdev(qstream(g));
    tdev.start();
    if (eng == Engine::PowItr || eng == Engine::SimFwdPush) {
      const uint64_t n = g.n, nk = n * (uint64_t)b.K;
      cudaStream_t st = qstream(g);
      Workspace& w = b.w;
      PPRG_CUDA(cudaMemsetAsync(w.x.get(), 0, 8 * nk, st));
      PPRG_CUDA(cudaMemsetAsync(w.r0.get(), 0, 8 * nk, st));
      PPRG_CUDA(cudaMemsetAsync(w.r1.get(), 0, 8 * nk, st));  // rows never visited stay 0
      PPRG_CUDA(cudaMemsetAsync(w.y1.get(), 0, 8 * nk, st));
      PPRG_CUDA(cudaMemsetAsync(w.dcols.get() + 2 * KMAX, 0, 8 * KMAX, st));
      k_seed<<<1, KMAX, 0, st>>>(w.r0.get(), w.d_src.get(), b.K, 1.0);
      k_init_pull<<<grid_reduce(nk), 256, 0, st>>>(w.r0.get(), g.deg.get(), g.inv_deg.get(), n, b.K,
                                                alpha, w.y0.get(), w.dcols.get() + 2 * KMAX);
      if (t_det) det_colsum(b, w.r0.get(), g.dead.get(), g.n_dead, 1.0 - alpha, w.dcols.get() + 2 * KMAX);
      d2h_small(b.D.data(), w.dcols.get() + 2 * KMAX, 8 * KMAX, st);
      PPRG_CUDA(cudaMemsetAsync(w.ctl(), 0, sizeof(SweepCtl), st));
      PPRG_CUDA(cudaStreamSynchronize(st));
      SweepParams P = base_params(b);
      for (int c = 0; c < b.K; ++c) {
        P.init[c].r_sum = 1.0;
        P.init[c].D = b.D[c];
        P.init[c].done = c >= (int)kb || !(1.0 > lambda);  // push.cpp:87
      }
      P.lambda = lambda;
      P.x = w.x.get();
      P.r[0] = w.r0.get();
      P.r[1] = w.r1.get();
      P.y[0] = w.y0.get();
      P.y[1] = w.y1.get();
      SweepTrace trace;
      trace.attach(P);
      EventTimer tm(st);
      SweepCtl hc;
      if (g_obs) {
        // observed: one iteration per launch (push.hpp:62-70 on_iteration)
        std::vector<ColInit> stv(P.init, P.init + b.K);
        std::memset(&hc, 0, sizeof hc);
        double* rb[2] = {w.r0.get(), w.r1.get()};
        double* yb[2] = {w.y0.get(), w.y1.get()};
        int cur = 0;
        tm.start();
        for (uint32_t it = 0;; ++it) {
          bool all = true;
          for (int c = 0; c < b.K; ++c) all &= stv[c].done != 0;
          if (all) break;
          SweepParams Q = P;
          Q.max_sweeps = 1;
          Q.r[0] = rb[cur];
          Q.r[1] = rb[cur ^ 1];
          Q.y[0] = yb[cur];
          Q.y[1] = yb[cur ^ 1];
          for (int c = 0; c < b.K; ++c) Q.init[c] = stv[c];
          PPRG_CUDA(cudaMemsetAsync(w.ctl(), 0, sizeof(SweepCtl), st));
          if (eng == Engine::PowItr) dispatch_sweeps<M_POWITR>(g, b.K, Q, true);
          else dispatch_sweeps<M_SIMFWD>(g, b.K, Q, true);
          SweepCtl one;
          d2h_small(&one, w.ctl(), sizeof one, st);
          PPRG_CUDA(cudaStreamSynchronize(st));
          hc.alg_bytes += one.alg_bytes;
          hc.total_sweeps = it + 1;
          for (int c = 0; c < b.K; ++c)
            stv[c] = ColInit{one.out_rsum[c], one.out_D[c], 0, one.out_done[c], one.out_sweeps[c],
                             one.out_pushes[c]};
          cur ^= 1;
          emit_step(b, w.x.get(), 1.0, rb[cur], stv[0].r_sum,
                    eng == Engine::PowItr ? (uint64_t)stv[0].sweeps * g.m_eff() : stv[0].pushes);
        }
        tm.stop();
        for (int c = 0; c < b.K; ++c) {
          hc.out_rsum[c] = stv[c].r_sum;
          hc.out_done[c] = stv[c].done;
          hc.out_sweeps[c] = stv[c].sweeps;
          hc.out_pushes[c] = stv[c].pushes;
        }
      } else {
        tm.start();
        if (eng == Engine::PowItr) dispatch_sweeps<M_POWITR>(g, b.K, P, true);
        else dispatch_sweeps<M_SIMFWD>(g, b.K, P, true);
        tm.stop();
        d2h_small(&hc, w.ctl(), sizeof hc, st);
      }
      call->sweep_ms += tm.ms();
      trace.fold(st, hc.total_sweeps, 0, eng == Engine::PowItr ? g.m_eff() : 0);
      call->alg_bytes += hc.alg_bytes;
      call->sweep_launches += 1;
      call->kernel_launches += 4;
      if (hc.total_sweeps > call->max_sweeps) call->max_sweeps = hc.total_sweeps;
      for (uint32_t c = 0; c < kb; ++c) {
        if (!hc.out_done[c]) fail(EINTERNAL, "power iteration: sweep limit reached");
        cs[c].r_sum = hc.out_rsum[c];
        // power_iteration pushes every node every iteration (push.cpp:92-99);
        // rows with in-degree 0 are skipped on the device but counted here
        cs[c].pushes = eng == Engine::PowItr ? (uint64_t)hc.out_sweeps[c] * g.m_eff()
                                             : hc.out_pushes[c];
        cs[c].sweeps = hc.out_sweeps[c];
      }
      const double* rlast = (hc.total_sweeps & 1) ? w.r1.get() : w.r0.get();
      const cudaMemcpyKind kind = out.on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
      if (o.reserve || o.residue) {
        DevBuf<double> tmp(n * kb);
        if (o.reserve) {
          k_unpack<<<grid_for(nk), 256, 0, st>>>(w.x.get(), n, b.K, kb, 1.0, tmp.get());
          PPRG_CUDA(cudaMemcpyAsync(o.reserve, tmp.get(), 8 * n * kb, kind, st));
          PPRG_CUDA(cudaStreamSynchronize(st));
        }
        if (o.residue) {
          k_unpack<<<grid_for(nk), 256, 0, st>>>(rlast, n, b.K, kb, 1.0, tmp.get());
          PPRG_CUDA(cudaMemcpyAsync(o.residue, tmp.get(), 8 * n * kb, kind, st));
        }
      }
      PPRG_CUDA(cudaStreamSynchronize(st));
    } else if (eng == Engine::Fifo) {
      const uint64_t nk = g.n * (uint64_t)b.K;
      PPRG_CUDA(cudaMemsetAsync(b.w.x.get(), 0, 8 * nk, qstream(g)));
      PPRG_CUDA(cudaMemsetAsync(b.w.res.get(), 0, 8 * nk, qstream(g)));
      k_seed<<<1, KMAX, 0, qstream(g)>>>(b.w.res.get(), b.w.d_src.get(), b.K, 1.0);
      std::vector<int> state(KMAX, 2);
      for (uint32_t c = 0; c < kb; ++c) state[c] = 0;
      drain_levels(b, r_max_fifo, lambda_stop_fifo, UINT64_MAX, false, state, call);
      finalize(b, o, false, call);
    } else {
      power_push_block(b, lambda, epoch_num, scan_threshold, call);
      finalize(b, o, false, call);
      for (uint32_t c = 0; c < kb; ++c)
        if (b.scan[c] && b.r_sum[c] > lambda)
          fail(EINTERNAL, "power push: exact r_sum " + std::to_string(b.r_sum[c]) +
                              " above lambda after the global phase");
    }
    tdev.stop();
    call->device_ms += tdev.ms();
    if (b0 + kb >= k && !out.async_host) sync_host_copies(g);
    if (eng == Engine::PowerPush || eng == Engine::Fifo)
      for (uint32_t c = 0; c < kb; ++c) {
        cs[c].r_sum = b.r_sum[c];
        cs[c].pushes = b.pushes[c];
        cs[c].sweeps = b.sweeps[c];
        cs[c].local_levels = b.levels[c];
        cs[c].used_scan_phase = b.scan[c];
      }
  }
}

// SpeedPPR push stage (speedppr.cpp:104-107): power_push_state at lambda,
// explicit residues, then refine to r_max. Leaves x / residues interleaved
// in the graph's workspace for the Monte Carlo phase.
void speedppr_push_stage(Graph& g, const uint32_t* sources, uint32_t k, double alpha,
                         double lambda, double r_max, ColumnStats* cols, CallStats* call,
                         PushView* view) {
  g.ensure_transpose();
  const uint64_t rb0 = t_readback_kernels;
  Block b = make_block(g, sources, k, alpha, true);
  // PowerPush to lambda, then refine (push.cpp:208-222) as a final sweep
  // epoch at r_max run to its fixpoint, so the refine is pull sweeps over the
  // tile plan rather than a scattered frontier over millions of nodes.
  // The local phase of this stage stops at a queue of n/32 instead of the
  // reference's default n/4 (PPRG_SPP_SCAN_DIV): on the GPU a frontier level
  // costs more than a pull sweep once it holds more than a few percent of the
  // (node, column) pairs. configs[3]: 2.37 -> 2.14 ms per query (n/16: 2.18,
  // n/64: 2.20, n/256: 2.23; profiles/r02_spp_scan_div.txt). The SpeedPPR
  // estimate's guarantee does not depend on where PowerPush switches phases.
  static const double spp_div = [] {
    const char* e = std::getenv("PPRG_SPP_SCAN_DIV");
    return e ? std::atof(e) : 32.0;
  }();
  power_push_block(b, lambda, 8, (int64_t)((double)g.n / spp_div), call, r_max);
  Outputs none;
  finalize(b, none, true, call);
  // the tail: every node still above deg_eff * r_max in id order, drained
  std::vector<int> state(KMAX, 2);
  for (uint32_t c = 0; c < k; ++c) state[c] = 0;
  EventTimer tl(qstream(g));
  tl.start();
  drain_levels(b, r_max, 0.0, UINT64_MAX, true, state, call);  // (+ recompute_r_sum)
  tl.stop();
  call->local_ms += tl.ms();
  for (uint32_t c = 0; c < k; ++c) {
    cols[c].r_sum = b.r_sum[c];
    cols[c].pushes = b.pushes[c];
    cols[c].sweeps = b.sweeps[c];
    cols[c].local_levels = b.levels[c];
    cols[c].used_scan_phase = b.scan[c];
  }
  call->kernel_launches += (uint32_t)(t_readback_kernels - rb0);
  view->K = b.K;
  view->k = k;
  view->x = b.w.x.get();
  view->res = b.w.res.get();
  view->d_src = b.w.d_src.get();
  view->src = b.src;
}

// ---- vertex-partitioned PowerPush (BASELINE configs[4]) ------
// Partition `part` of `nparts` owns a contiguous range of destination rows of
// the pull sweep, cut at row-aligned tile boundaries of the tile plan so each
// part holds ~m/nparts in-edges. Per global sweep a part pushes its own rows
// (x, y updated in place) from the gathered operand y of the previous
// exchange; the caller then all-gathers y's row slices and all-reduces the
// per-column sweep counters, and every part advances the identical epoch
// state (push.cpp:168-197) from the summed counters. Stale remote y only
// under-estimates inflow, and r_sum = 1 - alpha * sum(x) is exact whatever
// the staleness, so the result obeys the same lambda bounds. The local queue
// phase (push.cpp:163-166) runs on every part over its resident full graph
// (it is <= 0.05 m work); each part keeps only its own rows of it.
namespace {

__global__ void k_part_sums(const double* x, const uint32_t* deg, uint64_t lo, uint64_t hi, int K,
                            double* out) {
  __shared__ double sx[KMAX], sd[KMAX];
  if (threadIdx.x < KMAX) sx[threadIdx.x] = sd[threadIdx.x] = 0.0;
  __syncthreads();
  double ax = 0.0, ad = 0.0;
  // blockDim and the grid stride are multiples of K: a thread keeps one column
  for (uint64_t i = lo * K + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < hi * K;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double v = x[i];
    ax += v;
    if (deg[i / K] == 0) ad += v;
  }
  const int c = threadIdx.x % K;
  if (ax != 0.0) atomicAdd(&sx[c], ax);
  if (ad != 0.0) atomicAdd(&sd[c], ad);
  __syncthreads();
  if (threadIdx.x < K) {
    if (sx[threadIdx.x] != 0.0) atomicAdd(out + threadIdx.x, sx[threadIdx.x]);
    if (sd[threadIdx.x] != 0.0) atomicAdd(out + KMAX + threadIdx.x, sd[threadIdx.x]);
  }
}

struct PeerSet {
  double* y[PPRG_MAX_PEERS];
  int n;
};

__global__ void k_part_y(const double* x, const double* inv_deg, uint64_t lo, uint64_t hi, int K,
                         double alpha, double* y, const PeerSet peers) {
  for (uint64_t i = lo * K + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < hi * K;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double v = (1.0 - alpha) * x[i] * inv_deg[i / K];
    y[i] = v;
    for (int p = 0; p < peers.n; ++p) peers.y[p][i] = v;
  }
  if (peers.n) __threadfence_system();
}

__global__ void k_pack_counters(const SweepCtl* ctl, int K, double* out) {
  const int c = threadIdx.x;
  if (c >= K) return;
  out[c] = ctl->pushed[0][c];
  out[K + c] = (double)ctl->npush[0][c];
  out[2 * K + c] = (double)ctl->nnode[0][c];
  out[3 * K + c] = ctl->dsum[0][c];
  out[4 * K + c] = (double)ctl->et[0][c];
}

__global__ void k_zero_rows(double* out, uint64_t n, uint32_t k, uint64_t lo, uint64_t hi) {
  const uint64_t w = hi - lo;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < w * k;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[(i / w) * n + lo + i % w] = 0.0;
}

}  // namespace

// The global-phase epoch rule on the host, over summed counters. Identical to
// the device rule of k_sweeps (M_POWERPUSH): r_sum -= alpha * pushed; an
// epoch ends when r_sum <= its lambda, or at a fixpoint (no pushes).
bool epoch_init(ColInit* st, int K, const double* sum_x, const double* sum_dead_x,
                const double* lam, uint32_t E, double alpha) {
  bool any = false;
  for (int c = 0; c < K; ++c) {
    ColInit& ci = st[c];
    ci = ColInit{};
    ci.r_sum = 1.0 - alpha * sum_x[c];  // sum_u r_u = 1 - alpha sum_u x_u
    ci.D = (1.0 - alpha) * sum_dead_x[c];
    int ep = 0;
    while (ep < (int)E && !(ci.r_sum > lam[ep])) ++ep;
    ci.epoch = ep;
    ci.done = ep >= (int)E;
    any |= !ci.done;
  }
  return any;
}

bool epoch_advance(ColInit* st, int K, const double* summed, const double* lam, uint32_t E,
                   double alpha) {
  bool all_done = true;
  for (int c = 0; c < K; ++c) {
    ColInit& ci = st[c];
    if (!ci.done) {
      const double pushed = summed[c];
      const uint64_t np = (uint64_t)summed[K + c];
      ci.sweeps += 1;
      ci.pushes += np;
      ci.D = summed[3 * K + c];
      ci.r_sum -= alpha * pushed;
      if (np == 0) ci.epoch += 1;
      while (ci.epoch < (int)E && !(ci.r_sum > lam[ci.epoch])) ci.epoch += 1;
      if (ci.epoch >= (int)E) ci.done = 1;
    }
    all_done &= ci.done != 0;
  }
  return all_done;
}

struct PartSession {
  Graph* g = nullptr;
  Workspace w;
  std::unique_ptr<Block> b;
  uint32_t nparts = 1, part = 0, E = 8;
  uint64_t t0 = 0, t1 = 0, lo = 0, hi = 0;
  const TileDesc* desc = nullptr;
  double lambda = 0;
  std::vector<double> lam, thr;
  std::vector<ColInit> st;
  std::vector<int> used_scan;
  DevBuf<double> sums, counters;
  CallStats call;
  uint64_t own_alg_bytes = 0;
  uint32_t sweeps = 0;
  std::vector<double*> peers;  // fused exchange targets (other parts' y)
};

PartSession* part_begin(Graph& g, uint32_t nparts, uint32_t part, const uint32_t* sources,
                        uint32_t k, double alpha, double lambda, uint32_t E, int64_t scan_threshold,
                        double* partial_host, uint64_t* lo_out, uint64_t* hi_out) {
  DeviceGuard dg(g.device);
  LaneGuard lk(g, true);  // the partitioned query takes the whole device
  if (nparts < 1 || part >= nparts) fail(EINVAL_, "partition: part must be < nparts");
  if (k < 1 || k > KMAX) fail(EINVAL_, "partition: 1..64 sources per session");
  if (!(lambda > 0.0 && lambda <= 1.0)) fail(EINVAL_, "power_push: lambda must be in (0,1]");
  if (!(alpha > 0.0 && alpha < 1.0)) fail(EINVAL_, "alpha must be in (0,1)");
  if (E < 1 || E > EMAX) fail(EINVAL_, "epoch_num must be in 1..64");
  for (uint32_t c = 0; c < k; ++c)
    if (sources[c] >= g.n) fail(EINVAL_, "source out of range");
  g.ensure_transpose();
  auto s = std::make_unique<PartSession>();
  s->g = &g;
  s->nparts = nparts;
  s->part = part;
  s->E = E;
  s->lambda = lambda;
  s->b = std::make_unique<Block>(make_block(g, sources, k, alpha, true, &s->w));
  Block& b = *s->b;
  const int K = b.K;
  // ---- the cut: row-start tiles, balanced on in-edges ------------------------
  const Graph::Plan& pl = g.tile_plan(tile_edges(g, K), tile_rmax(g, K), tile_hub(g, K));
  const std::vector<TileDesc>& tl = pl.host;
  uint64_t total = 0;
  for (const TileDesc& t : tl) total += t.ne;
  std::vector<uint64_t> cut(nparts + 1, 0);
  cut[nparts] = tl.size();
  {
    uint64_t acc = 0, t = 0;
    for (uint32_t p = 1; p < nparts; ++p) {
      const double target = (double)total * p / nparts;
      while (t < tl.size() && ((double)acc < target || tl[t].piece != 0)) acc += tl[t++].ne;
      cut[p] = t;
    }
  }
  auto node_of_tile = [&](uint64_t t) -> uint64_t {
    if (t >= tl.size()) return g.n;
    uint32_t u = 0;
    PPRG_CUDA(cudaMemcpy(&u, g.cin_row.get() + tl[t].r0, 4, cudaMemcpyDeviceToHost));
    return u;
  };
  s->t0 = cut[part];
  s->t1 = cut[part + 1];
  s->lo = part == 0 ? 0 : node_of_tile(s->t0);
  s->hi = part + 1 == nparts ? g.n : node_of_tile(s->t1);
  if (s->hi < s->lo) s->hi = s->lo;
  s->desc = pl.tiles.get() + s->t0;
  // ---- local phase (push.cpp:163-166) on the full graph -----------------------
  cudaStream_t st = qstream(g);
  const uint64_t nk = g.n * (uint64_t)K;
  PPRG_CUDA(cudaMemsetAsync(b.w.x.get(), 0, 8 * nk, st));
  PPRG_CUDA(cudaMemsetAsync(b.w.res.get(), 0, 8 * nk, st));
  PPRG_CUDA(cudaMemsetAsync(b.w.y0.get(), 0, 8 * nk, st));  // y = 0 is a valid stale value
  k_seed<<<1, KMAX, 0, st>>>(b.w.res.get(), b.w.d_src.get(), K, 1.0);
  const double r_max = lambda / (double)g.m_eff();
  const uint64_t limit = scan_threshold < 0 ? g.n / 4 : (uint64_t)scan_threshold;
  std::vector<int> state(KMAX, 2);
  for (uint32_t c = 0; c < k; ++c) state[c] = 0;
  EventTimer tl_(st);
  tl_.start();
  drain_levels(b, r_max, lambda, limit, false, state, &s->call);
  tl_.stop();
  s->call.local_ms += tl_.ms();
  // ---- this part's share of sum(x) and sum over dead ends -------------------
  s->sums.alloc(2 * KMAX);
  s->counters.alloc(5 * KMAX);
  PPRG_CUDA(cudaMemsetAsync(s->sums.get(), 0, 16 * KMAX, st));
  if (s->hi > s->lo)
    k_part_sums<<<grid_reduce((s->hi - s->lo) * K), 256, 0, st>>>(b.w.x.get(), g.deg.get(), s->lo,
                                                               s->hi, K, s->sums.get());
  PPRG_CUDA(cudaGetLastError());
  PPRG_CUDA(cudaMemcpyAsync(partial_host, s->sums.get(), 16 * KMAX, cudaMemcpyDeviceToHost, st));
  PPRG_CUDA(cudaStreamSynchronize(st));
  s->call.kernel_launches += 2;
  *lo_out = s->lo;
  *hi_out = s->hi;
  return s.release();
}

bool part_start(PartSession* s, const double* summed) {
  Graph& g = *s->g;
  DeviceGuard dg(g.device);
  LaneGuard lk(g, true);  // the partitioned query takes the whole device
  Block& b = *s->b;
  const int K = b.K;
  const double m_eff = (double)g.m_eff();
  s->lam.assign(EMAX, 0.0);
  s->thr.assign(EMAX, 0.0);
  for (uint32_t e = 0; e < s->E; ++e) {
    const double el = std::pow(s->lambda, static_cast<double>(e + 1) / s->E);  // push.cpp:176-178
    s->lam[e] = stop_lambda(el, e, s->E);
    s->thr[e] = el / m_eff;
  }
  s->st.assign(KMAX, ColInit{});
  s->used_scan.assign(KMAX, 0);
  std::vector<double> sx(summed, summed + K), sd(summed + KMAX, summed + KMAX + K);
  const bool any = epoch_init(s->st.data(), K, sx.data(), sd.data(), s->lam.data(), s->E, b.alpha);
  for (int c = 0; c < K; ++c) s->used_scan[c] = s->st[c].r_sum > s->lambda;  // push.cpp:168
  PeerSet ps{};
  ps.n = (int)s->peers.size();
  for (int p = 0; p < ps.n; ++p) ps.y[p] = s->peers[p];
  if (s->hi > s->lo)
    k_part_y<<<grid_for((s->hi - s->lo) * K), 256, 0, qstream(g)>>>(b.w.x.get(), g.inv_deg.get(), s->lo,
                                                                  s->hi, K, b.alpha, b.w.y0.get(), ps);
  PPRG_CUDA(cudaGetLastError());
  PPRG_CUDA(cudaStreamSynchronize(qstream(g)));
  s->call.kernel_launches += 1;
  return any;
}

static SweepParams part_params(PartSession* s) {
  Block& b = *s->b;
  SweepParams P = base_params(b);
  P.desc = s->desc;
  P.ntiles = s->t1 - s->t0;
  P.own_lo = s->lo;
  P.own_hi = s->hi;
  P.x = b.w.x.get();
  P.y[0] = P.y[1] = b.w.y0.get();
  for (int c = 0; c < b.K; ++c) P.init[c] = s->st[c];
  P.npeers = (int)s->peers.size();
  for (int p = 0; p < P.npeers; ++p) P.peer_y[p] = s->peers[p];
  return P;
}

void part_set_peers(PartSession* s, double* const* peer_y, uint32_t npeers) {
  if (npeers > PPRG_MAX_PEERS) fail(EINVAL_, "partition: too many peers");
  s->peers.assign(peer_y, peer_y + npeers);
}

void part_sweep(PartSession* s, double* local_host) {
  Graph& g = *s->g;
  DeviceGuard dg(g.device);
  LaneGuard lk(g, true);  // the partitioned query takes the whole device
  Block& b = *s->b;
  const int K = b.K;
  SweepParams P = part_params(s);
  P.max_sweeps = 1;
  P.E = (int)s->E;
  for (uint32_t e = 0; e < s->E; ++e) {
    P.lam[e] = s->lam[e];
    P.thr[e] = s->thr[e];
  }
  cudaStream_t st = qstream(g);
  PPRG_CUDA(cudaMemsetAsync(b.w.ctl(), 0, sizeof(SweepCtl), st));
  EventTimer tm(st);
  tm.start();
  dispatch_sweeps<M_POWERPUSH>(g, K, P, true);
  tm.stop();
  k_pack_counters<<<1, KMAX, 0, st>>>(b.w.ctl(), K, s->counters.get());
  PPRG_CUDA(cudaGetLastError());
  std::vector<double> loc(5 * KMAX, 0.0);
  PPRG_CUDA(cudaMemcpyAsync(loc.data(), s->counters.get(), 8 * 5 * K, cudaMemcpyDeviceToHost, st));
  PPRG_CUDA(cudaStreamSynchronize(st));
  if (local_host) std::memcpy(local_host, loc.data(), 8 * 5 * K);
  // this part's algorithmic bytes (SURVEY 8(d) over its own rows)
  uint64_t pt = 0, et = 0;
  for (uint32_t c = 0; c < b.k; ++c) {
    pt += (uint64_t)loc[2 * K + c];
    et = std::max<uint64_t>(et, (uint64_t)loc[4 * K + c]);
  }
  const uint64_t nown = s->hi - s->lo;
  s->own_alg_bytes += 8ull * (nown + 1) + 8ull * b.k * nown + 4ull * et + 24ull * pt;
  s->call.sweep_ms += tm.ms();
  s->call.sweep_launches += 1;
  s->call.kernel_launches += 2;
  s->sweeps += 1;
}

bool part_advance(PartSession* s, const double* summed) {
  const bool all_done = epoch_advance(s->st.data(), s->b->K, summed, s->lam.data(), s->E, s->b->alpha);
  if (!all_done && s->sweeps >= 200000) fail(EINTERNAL, "power push: sweep limit reached");
  return all_done;
}

void part_finish(PartSession* s, double* reserve, double* residue, bool on_device, double* rpart) {
  Graph& g = *s->g;
  DeviceGuard dg(g.device);
  LaneGuard lk(g, true);  // the partitioned query takes the whole device
  Block& b = *s->b;
  cudaStream_t st = qstream(g);
  const uint64_t n = g.n;
  const uint32_t k = b.k;
  SweepParams Q = part_params(s);
  DevBuf<double> tr, tq;
  if (!on_device) {
    if (reserve) tr.alloc(n * k);
    if (residue) tq.alloc(n * k);
  }
  Q.out_reserve = reserve ? (on_device ? reserve : tr.get()) : nullptr;
  Q.out_residue = residue ? (on_device ? residue : tq.get()) : nullptr;
  const uint64_t w = s->hi - s->lo;
  for (double* o : {Q.out_reserve, Q.out_residue})
    if (o && w) k_zero_rows<<<grid_for(w * k), 256, 0, st>>>(o, n, k, s->lo, s->hi);
  Q.res_inter = nullptr;
  Q.push_res = b.w.res.get();
  for (int c = 0; c < b.K; ++c) {
    Q.final_pull[c] = 1;
    Q.init[c].done = 0;  // the final pass visits every column
  }
  PPRG_CUDA(cudaMemsetAsync(b.w.ctl(), 0, sizeof(SweepCtl), st));
  EventTimer tf(st);
  tf.start();
  dispatch_sweeps<M_FINAL>(g, b.K, Q, true);
  tf.stop();
  SweepCtl fc;
  d2h_small(&fc, b.w.ctl(), sizeof fc, st);
  check_final(fc);
  if (!on_device && w) {
    for (uint32_t c = 0; c < k; ++c) {
      if (reserve)
        PPRG_CUDA(cudaMemcpyAsync(reserve + c * n + s->lo, tr.get() + c * n + s->lo, 8 * w,
                                  cudaMemcpyDeviceToHost, st));
      if (residue)
        PPRG_CUDA(cudaMemcpyAsync(residue + c * n + s->lo, tq.get() + c * n + s->lo, 8 * w,
                                  cudaMemcpyDeviceToHost, st));
    }
  }
  PPRG_CUDA(cudaStreamSynchronize(st));
  s->call.final_ms += tf.ms();
  s->call.kernel_launches += 3;
  for (uint32_t c = 0; c < k; ++c) rpart[c] = fc.pushed[0][c];
}

void part_stats(const PartSession* s, ColumnStats* cols, CallStats* call) {
  const Block& b = *s->b;
  for (uint32_t c = 0; c < b.k; ++c) {
    cols[c].pushes = b.pushes[c] + s->st[c].pushes;
    cols[c].sweeps = s->st[c].sweeps;
    cols[c].local_levels = b.levels[c];
    cols[c].used_scan_phase = s->used_scan[c];
    cols[c].r_sum = s->st[c].r_sum;
  }
  *call = s->call;
  call->alg_bytes = s->own_alg_bytes;
  call->max_sweeps = s->sweeps;
  call->device_ms = s->call.local_ms + s->call.sweep_ms + s->call.final_ms;
}

double* part_y(PartSession* s, uint32_t* K) {
  *K = (uint32_t)s->b->K;
  return s->b->w.y0.get();
}
double* part_counters(PartSession* s) { return s->counters.get(); }
double* part_x(PartSession* s) { return s->b->w.x.get(); }

// After the caller overwrote x with another part's local-phase result (the
// local phase is run once and its x broadcast, so every part starts from one
// consistent push state), recompute this part's share of sum(x) and of the
// dead-end sum.
void part_resum(PartSession* s, double* partial_host) {
  Graph& g = *s->g;
  DeviceGuard dg(g.device);
  LaneGuard lk(g, true);  // the partitioned query takes the whole device
  Block& b = *s->b;
  const int K = b.K;
  cudaStream_t st = qstream(g);
  PPRG_CUDA(cudaMemsetAsync(s->sums.get(), 0, 16 * KMAX, st));
  if (s->hi > s->lo)
    k_part_sums<<<grid_reduce((s->hi - s->lo) * K), 256, 0, st>>>(b.w.x.get(), g.deg.get(), s->lo,
                                                               s->hi, K, s->sums.get());
  PPRG_CUDA(cudaGetLastError());
  PPRG_CUDA(cudaMemcpyAsync(partial_host, s->sums.get(), 16 * KMAX, cudaMemcpyDeviceToHost, st));
  PPRG_CUDA(cudaStreamSynchronize(st));
  s->call.kernel_launches += 1;
}
int part_device(const PartSession* s) { return s->g->device; }

void part_destroy(PartSession* s) {
  if (!s) return;
  DeviceGuard dg(s->g->device);
  delete s;
}

}  // namespace pprg
