// Graph build and device residency (hot-path subsystem (1)).
//
// Reference semantics reproduced bit-exactly (graph.cpp:13-63):
//   * survivors = sorted unique endpoint ids, new id = rank (:40-51)
//   * offsets = exclusive scan of per-source counts (:54-56)
//   * neighbours in input order per source (:58-60) -- a stable radix sort
//     keyed on the relabelled source gives exactly the cursor scatter order
//   * dead_ends = ascending ids with out-degree 0 (:19-20); validate (:24-34)
// Generators (R-MAT, Chung-Lu) are counter-based (Philox keyed by
// (seed, edge index)) so host and device agree, then cleaned (self-loops and
// duplicates removed) and sorted before the reference build semantics apply.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include <cstring>

#include "fileio.h"
#include "internal.h"

namespace pprg {
namespace {

constexpr int TB = 256;
inline unsigned blocks_for(uint64_t n, int tb = TB) {
  uint64_t b = (n + tb - 1) / tb;
  return (unsigned)(b ? (b > 0x7fffffffull ? 0x7fffffffull : b) : 1);
}

#define GRID_STRIDE(i, cnt) \
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (cnt); i += (uint64_t)gridDim.x * blockDim.x)

__global__ void k_validate(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint64_t m,
                           unsigned* bad) {
  GRID_STRIDE(v, n) {
    if (off[v + 1] < off[v]) atomicOr(bad, 1u);
    if (off[v + 1] - off[v] > 0xffffffffull) atomicOr(bad, 4u);
  }
  GRID_STRIDE(e, m) {
    if (nbr[e] >= n) atomicOr(bad, 2u);
  }
}

__global__ void k_degrees(const uint64_t* off, uint64_t n, uint32_t* deg, double* inv_deg,
                          unsigned* dead_flag) {
  GRID_STRIDE(v, n) {
    const uint64_t d = off[v + 1] - off[v];
    deg[v] = (uint32_t)d;
    inv_deg[v] = 1.0 / (double)(d ? d : 1);
    dead_flag[v] = d == 0;
  }
}

__global__ void k_scatter_flagged(const unsigned* flag, const unsigned* pos, uint64_t n,
                                  uint32_t* out) {
  GRID_STRIDE(v, n) {
    if (flag[v]) out[pos[v]] = (uint32_t)v;
  }
}

__global__ void k_expand_rows(const uint64_t* off, uint64_t n, uint32_t* src) {
  // one warp per row writes the row id over its edge slice
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (uint64_t v = warp; v < n; v += nw)
    for (uint64_t e = off[v] + lane; e < off[v + 1]; e += 32) src[e] = (uint32_t)v;
}

__global__ void k_count(const uint32_t* keys, uint64_t m, unsigned long long* cnt) {
  GRID_STRIDE(e, m) atomicAdd(cnt + keys[e], 1ull);
}

__global__ void k_nonempty(const uint64_t* in_off, uint64_t n, unsigned* flag) {
  GRID_STRIDE(u, n) flag[u] = in_off[u + 1] > in_off[u];
}
__global__ void k_compact_rows(const uint64_t* in_off, const unsigned* flag, const unsigned* pos,
                               uint64_t n, uint64_t m, uint64_t* cin_off, uint32_t* cin_row,
                               uint64_t n_rows) {
  GRID_STRIDE(u, n) {
    if (flag[u]) {
      cin_off[pos[u]] = in_off[u];
      cin_row[pos[u]] = (uint32_t)u;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cin_off[n_rows] = m;
}

__global__ void k_row_degs(const uint32_t* cin_row, uint64_t n_rows, const uint32_t* deg,
                           const double* inv_deg, uint32_t* cdeg, double* cinv) {
  GRID_STRIDE(r, n_rows) {
    cdeg[r] = deg[cin_row[r]];
    cinv[r] = inv_deg[cin_row[r]];
  }
}

// Tile descriptor: (first compact row touching tile j, number of rows) where
// the rows are the continuation of a row begun in an earlier tile (if any)
// plus the rows starting in [jT, (j+1)T).
__device__ __forceinline__ uint64_t lb_rows(const uint64_t* off, uint64_t n, uint64_t key) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (off[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__global__ void k_tile_desc(const uint64_t* cin_off, uint64_t n_rows, uint64_t m, uint64_t ntiles,
                            uint32_t T, uint2* desc) {
  GRID_STRIDE(j, ntiles) {
    const uint64_t base = j * (uint64_t)T;
    const uint64_t lo = lb_rows(cin_off, n_rows, base);
    const uint64_t hi = lb_rows(cin_off, n_rows, base + T);
    const bool has_head = lo > 0 && base < m && cin_off[lo] > base;
    const uint64_t first = has_head ? lo - 1 : lo;
    desc[j] = make_uint2((uint32_t)first, (uint32_t)(hi - first));
  }
}

// Rows spanning more than one tile (their partials are combined after the
// sweep's grid barrier).
__global__ void k_split_flags(const uint64_t* cin_off, uint64_t n_rows, uint32_t T, unsigned* flag) {
  GRID_STRIDE(r, n_rows) flag[r] = (cin_off[r] / T) != ((cin_off[r + 1] - 1) / T);
}

// own_lo[j] = first row u with in_off[u] >= j*T (lower_bound over row starts)
// ---- generators ------------------------------------------------------------
// R-MAT: edge i descends `scale` levels; level l uses 32-bit word l of the
// Philox stream ctr = (i_lo, i_hi, 'RMAT', l/4) keyed by seed. Quadrants in
// the order a (0,0), b (0,1), c (1,0), d (1,1). Key = (u << 32) | v.
__global__ void k_rmat(uint64_t seed, int scale, uint64_t count, double a, double ab, double abc,
                       uint64_t* keys) {
  GRID_STRIDE(i, count) {
    uint32_t u = 0, v = 0;
    U4 o{};
    for (int l = 0; l < scale; ++l) {
      if ((l & 3) == 0)
        o = philox4x32_10(U4{(uint32_t)i, (uint32_t)(i >> 32), 0x524D4154u, (uint32_t)(l >> 2)},
                          (uint32_t)seed, (uint32_t)(seed >> 32));
      const uint32_t w = (l & 3) == 0 ? o.x : (l & 3) == 1 ? o.y : (l & 3) == 2 ? o.z : o.w;
      const double p = (double)w * 0x1.0p-32;
      const uint32_t bu = p >= ab, bv = (p >= a && p < ab) || p >= abc;
      u = (u << 1) | bu;
      v = (v << 1) | bv;
    }
    keys[i] = ((uint64_t)u << 32) | v;
  }
}

// Chung-Lu ball dropping: draw i picks u by inverse CDF of the out-weights
// and v by inverse CDF of the (permuted) in-weights, from
// Philox(ctr = (i_lo, i_hi, 'CHLU', 0)) words (x,y) and (z,w) as 53-bit
// uniforms.
__device__ __forceinline__ uint32_t inv_cdf(const double* cdf, uint64_t n, double x) {
  uint64_t lo = 0, hi = n - 1;  // first j with cdf[j] > x
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (cdf[mid] > x) hi = mid; else lo = mid + 1;
  }
  return (uint32_t)lo;
}

__global__ void k_chung_lu(uint64_t seed, uint64_t draws, const double* cdf_out,
                           const double* cdf_in, uint64_t n, uint64_t* keys) {
  GRID_STRIDE(i, draws) {
    const U4 o = philox4x32_10(U4{(uint32_t)i, (uint32_t)(i >> 32), 0x43484C55u, 0u},
                               (uint32_t)seed, (uint32_t)(seed >> 32));
    const double x = (double)((((uint64_t)o.y << 32) | o.x) >> 11) * 0x1.0p-53 * cdf_out[n - 1];
    const double y = (double)((((uint64_t)o.w << 32) | o.z) >> 11) * 0x1.0p-53 * cdf_in[n - 1];
    keys[i] = ((uint64_t)inv_cdf(cdf_out, n, x) << 32) | inv_cdf(cdf_in, n, y);
  }
}

__global__ void k_cl_weights(uint64_t n, double expo, double* w) {
  GRID_STRIDE(i, n) w[i] = pow((double)(i + 1), -expo);
}
__global__ void k_perm_keys(uint64_t seed, uint64_t n, uint64_t* keys, uint32_t* vals) {
  GRID_STRIDE(i, n) {
    const U4 o = philox4x32_10(U4{(uint32_t)i, (uint32_t)(i >> 32), 0x5045524Du, 0u},
                               (uint32_t)seed, (uint32_t)(seed >> 32));
    keys[i] = ((uint64_t)o.x << 32) | o.y;
    vals[i] = (uint32_t)i;
  }
}
__global__ void k_gather_w(const double* w, const uint32_t* perm, uint64_t n, double* out) {
  GRID_STRIDE(i, n) out[i] = w[perm[i]];
}

// keep[i] = first of its run and not a self-loop
__global__ void k_clean_flags(const uint64_t* keys, uint64_t cnt, unsigned char* keep) {
  GRID_STRIDE(i, cnt) {
    const uint64_t k = keys[i];
    keep[i] = (i == 0 || keys[i - 1] != k) && ((k >> 32) != (k & 0xffffffffull));
  }
}
__global__ void k_mark_present(const uint64_t* keys, uint64_t cnt, unsigned* present) {
  GRID_STRIDE(i, cnt) {
    present[keys[i] >> 32] = 1;
    present[keys[i] & 0xffffffffull] = 1;
  }
}
__global__ void k_relabel_sorted(const uint64_t* keys, uint64_t cnt, const unsigned* rank,
                                 uint32_t* src, uint32_t* dst) {
  GRID_STRIDE(i, cnt) {
    src[i] = rank[keys[i] >> 32];
    dst[i] = rank[keys[i] & 0xffffffffull];
  }
}

// generic edge list: endpoint ids (2 per pair) and lower_bound relabel
__global__ void k_split_pairs(const uint64_t* pairs, uint64_t cnt, uint64_t* ids) {
  GRID_STRIDE(i, 2 * cnt) ids[i] = pairs[i];
}
__global__ void k_relabel_search(const uint64_t* pairs, uint64_t cnt, const uint64_t* ids,
                                 uint64_t n, uint32_t* src, uint32_t* dst) {
  GRID_STRIDE(i, 2 * cnt) {
    const uint64_t key = pairs[i];
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (ids[mid] < key) lo = mid + 1; else hi = mid;
    }
    if (i & 1) dst[i >> 1] = (uint32_t)lo; else src[i >> 1] = (uint32_t)lo;
  }
}

template <typename F>
void cub_call(F&& f, cudaStream_t st) {
  size_t bytes = 0;
  PPRG_CUDA(f(nullptr, bytes));
  DevBuf<unsigned char> tmp(bytes ? bytes : 1);
  PPRG_CUDA(f(tmp.get(), bytes));
  (void)st;
}

int bits_for(uint64_t maxval) {
  int b = 1;
  while (b < 64 && (maxval >> b)) ++b;
  return b;
}

// offsets (u64, n+1) from per-row counts of `src` (u32 keys < n)
void offsets_from_src(const uint32_t* src, uint64_t m, uint64_t n, uint64_t* off, cudaStream_t st) {
  DevBuf<unsigned long long> cnt(n + 1);
  PPRG_CUDA(cudaMemsetAsync(cnt.get(), 0, 8 * (n + 1), st));
  if (m) k_count<<<blocks_for(m), TB, 0, st>>>(src, m, cnt.get());
  unsigned long long* c = cnt.get();
  uint64_t* o = off;
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, c, (unsigned long long*)o, (int64_t)(n + 1), st);
  }, st);
}

// From a sorted, cleaned key list (u<<32|v): reference build semantics.
std::unique_ptr<Graph> build_from_sorted_keys(DevBuf<uint64_t>& keys, uint64_t cnt, uint64_t id_space,
                                              int device, cudaStream_t st) {
  DevBuf<unsigned> present(id_space + 1), rank(id_space + 1);
  PPRG_CUDA(cudaMemsetAsync(present.get(), 0, 4 * (id_space + 1), st));
  k_mark_present<<<blocks_for(cnt), TB, 0, st>>>(keys.get(), cnt, present.get());
  unsigned* pp = present.get();
  unsigned* rp = rank.get();
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, pp, rp, (int64_t)(id_space + 1), st);
  }, st);
  unsigned n32 = 0;
  PPRG_CUDA(cudaMemcpyAsync(&n32, rank.get() + id_space, 4, cudaMemcpyDeviceToHost, st));
  PPRG_CUDA(cudaStreamSynchronize(st));
  auto g = std::make_unique<Graph>();
  g->device = device;
  g->stream = st;
  g->n = n32;
  g->m = cnt;
  g->nbr.alloc(cnt);
  g->off.alloc(g->n + 1);
  DevBuf<uint32_t> src(cnt);
  k_relabel_sorted<<<blocks_for(cnt), TB, 0, st>>>(keys.get(), cnt, rank.get(), src.get(),
                                                   g->nbr.get());
  offsets_from_src(src.get(), cnt, g->n, g->off.get(), st);
  g->finish_build();
  return g;
}

// sort keys, drop duplicates and self-loops (compaction in place)
uint64_t sort_clean(DevBuf<uint64_t>& keys, uint64_t cnt, int key_bits, cudaStream_t st) {
  DevBuf<uint64_t> sorted(cnt);
  uint64_t* in = keys.get();
  uint64_t* out = sorted.get();
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, in, out, (int64_t)cnt, 0, key_bits, st);
  }, st);
  DevBuf<unsigned char> keep(cnt);
  k_clean_flags<<<blocks_for(cnt), TB, 0, st>>>(sorted.get(), cnt, keep.get());
  DevBuf<unsigned long long> nsel(1);
  unsigned char* kp = keep.get();
  unsigned long long* ns = nsel.get();
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceSelect::Flagged(t, b, out, kp, in, ns, (int64_t)cnt, st);
  }, st);
  unsigned long long h = 0;
  PPRG_CUDA(cudaMemcpyAsync(&h, ns, 8, cudaMemcpyDeviceToHost, st));
  PPRG_CUDA(cudaStreamSynchronize(st));
  return h;
}

}  // namespace

Graph::~Graph() {
  DeviceGuard dg(device);
  for (size_t i = 0; i < lanes.size(); ++i) {
    if (i > 0 && lanes[i].stream) {
      cudaStreamSynchronize(lanes[i].stream);
      cudaStreamDestroy(lanes[i].stream);
    }
    if (lanes[i].done) cudaEventDestroy(lanes[i].done);
  }
  if (stream) {
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
  }
}

// ---- execution lanes --------------------------------------------------------
thread_local const LaneCtx* t_lane = nullptr;

// Lanes of a graph: PPRG_LANES (default 2) on graphs below PPRG_LANE_MAX_M
// in-edges (default 16M), where one query's persistent kernels are latency-
// bound and a half-device grid costs it little (configs[0]: 1.74 vs 1.71 ms;
// a quarter: 2.25 ms, profiles/r02_grid_frac.txt); one lane above, where a
// query needs the whole device.
static void init_lanes(Graph& g) {
  static const int want = [] {
    const char* e = std::getenv("PPRG_LANES");
    const int v = e ? std::atoi(e) : 2;
    return v < 1 ? 1 : v > 8 ? 8 : v;
  }();
  static const uint64_t max_m = [] {
    const char* e = std::getenv("PPRG_LANE_MAX_M");
    return e ? std::strtoull(e, nullptr, 10) : 16000000ull;
  }();
  const int nl = g.m < max_m ? want : 1;
  g.lanes.resize(nl);
  cudaEvent_t built;
  PPRG_CUDA(cudaEventCreateWithFlags(&built, cudaEventDisableTiming));
  PPRG_CUDA(cudaEventRecord(built, g.stream));  // the graph's build and uploads
  for (int i = 0; i < nl; ++i) {
    Graph::Lane& L = g.lanes[i];
    if (i == 0) {
      L.stream = g.stream;
    } else {
      PPRG_CUDA(cudaStreamCreateWithFlags(&L.stream, cudaStreamNonBlocking));
      PPRG_CUDA(cudaStreamWaitEvent(L.stream, built, 0));
    }
    PPRG_CUDA(cudaEventCreateWithFlags(&L.done, cudaEventDisableTiming));
    PPRG_CUDA(cudaEventRecord(L.done, L.stream));
  }
  PPRG_CUDA(cudaEventDestroy(built));
}

// A query takes one free lane, or -- exclusive -- all of them. Ordering on
// the device: an exclusive query's stream (lane 0) waits for every lane's last
// work, and after it every lane waits for it, so a whole-device persistent
// kernel never runs beside another lane's kernel; lanes' own kernels take
// 1/nlanes (x 0.95) of the resident blocks each and always fit together.
LaneGuard::LaneGuard(Graph& g, bool exclusive) : g_(g), all_(false), prev_(t_lane) {
  std::unique_lock<std::mutex> lk(g.lane_mu);
  if (g.lanes.empty()) init_lanes(g);
  const int nl = (int)g.lanes.size();
  auto all_free = [&] {
    for (const Graph::Lane& L : g.lanes)
      if (L.busy) return false;
    return true;
  };
  if (exclusive || nl == 1) {
    ++g.exclusive_waiters;
    g.lane_cv.wait(lk, all_free);
    --g.exclusive_waiters;
    for (Graph::Lane& L : g.lanes) L.busy = true;
    for (int i = 1; i < nl; ++i) PPRG_CUDA(cudaStreamWaitEvent(g.lanes[0].stream, g.lanes[i].done, 0));
    all_ = true;
    ctx_ = LaneCtx{0, g.lanes[0].stream, 1.0};
  } else {
    int pick = -1;
    g.lane_cv.wait(lk, [&] {
      if (g.exclusive_waiters) return false;
      for (int i = 0; i < nl; ++i)
        if (!g.lanes[i].busy) {
          pick = i;
          return true;
        }
      return false;
    });
    g.lanes[pick].busy = true;
    ctx_ = LaneCtx{pick, g.lanes[pick].stream, 0.95 / nl};
  }
  t_lane = &ctx_;
}

LaneGuard::~LaneGuard() {
  t_lane = prev_;
  std::lock_guard<std::mutex> lk(g_.lane_mu);
  if (all_) {
    PPRG_CUDA_NOTHROW(cudaEventRecord(g_.lanes[0].done, g_.lanes[0].stream));
    for (size_t i = 0; i < g_.lanes.size(); ++i) {
      if (i > 0) {
        PPRG_CUDA_NOTHROW(cudaStreamWaitEvent(g_.lanes[i].stream, g_.lanes[0].done, 0));
        PPRG_CUDA_NOTHROW(cudaEventRecord(g_.lanes[i].done, g_.lanes[i].stream));
      }
      g_.lanes[i].busy = false;
    }
  } else {
    Graph::Lane& L = g_.lanes[ctx_.lane];
    PPRG_CUDA_NOTHROW(cudaEventRecord(L.done, L.stream));
    L.busy = false;
  }
  g_.lane_cv.notify_all();
}

void Graph::finish_build() {
  cudaStream_t st = stream;
  DevBuf<unsigned> bad(1);
  PPRG_CUDA(cudaMemsetAsync(bad.get(), 0, 4, st));
  uint64_t first = 0, last = 0;
  PPRG_CUDA(cudaMemcpyAsync(&first, off.get(), 8, cudaMemcpyDeviceToHost, st));
  PPRG_CUDA(cudaMemcpyAsync(&last, off.get() + n, 8, cudaMemcpyDeviceToHost, st));
  k_validate<<<blocks_for(n > m ? n : m), TB, 0, st>>>(off.get(), nbr.get(), n, m, bad.get());
  unsigned hbad = 0;
  PPRG_CUDA(cudaMemcpyAsync(&hbad, bad.get(), 4, cudaMemcpyDeviceToHost, st));
  PPRG_CUDA(cudaStreamSynchronize(st));
  // same messages as Graph::validate (graph.cpp:24-34)
  if (first != 0) fail(EDATA, "graph: offsets must start at 0");
  if (hbad & 1) fail(EDATA, "graph: offsets must be non-decreasing");
  if (last != m) fail(EDATA, "graph: offsets must end at m");
  if (hbad & 2) fail(EDATA, "graph: neighbor id out of range");
  if (hbad & 4) fail(EDATA, "graph: out-degree exceeds 2^32-1");
  deg.alloc(n);
  inv_deg.alloc(n);
  DevBuf<unsigned> flag(n + 1), pos(n + 1);
  PPRG_CUDA(cudaMemsetAsync(flag.get() + n, 0, 4, st));
  k_degrees<<<blocks_for(n), TB, 0, st>>>(off.get(), n, deg.get(), inv_deg.get(), flag.get());
  unsigned* fp = flag.get();
  unsigned* pp = pos.get();
  const uint64_t nn = n;
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, fp, pp, (int64_t)(nn + 1), st);
  }, st);
  unsigned nd = 0;
  PPRG_CUDA(cudaMemcpyAsync(&nd, pos.get() + n, 4, cudaMemcpyDeviceToHost, st));
  PPRG_CUDA(cudaStreamSynchronize(st));
  n_dead = nd;
  dead.alloc(n_dead ? n_dead : 1);
  k_scatter_flagged<<<blocks_for(n), TB, 0, st>>>(flag.get(), pos.get(), n, dead.get());
  PPRG_CUDA(cudaStreamSynchronize(st));
  PPRG_CUDA(cudaGetLastError());
}

void Graph::ensure_transpose() {
  std::lock_guard<std::recursive_mutex> lk(build_mu);
  if (in_off.get()) return;
  cudaStream_t st = stream;
  in_off.alloc(n + 1);
  in_nbr.alloc(m ? m : 1);
  if (m == 0) {
    PPRG_CUDA(cudaMemsetAsync(in_off.get(), 0, 8 * (n + 1), st));
    n_rows = 0;
    cin_off.alloc(1);
    cin_row.alloc(1);
    cin_deg.alloc(1);
    cin_inv.alloc(1);
    PPRG_CUDA(cudaMemsetAsync(cin_off.get(), 0, 8, st));
    PPRG_CUDA(cudaStreamSynchronize(st));
    return;
  }
  DevBuf<uint32_t> src(m), keys_out(m);
  k_expand_rows<<<blocks_for(n * 32ull), TB, 0, st>>>(off.get(), n, src.get());
  // stable sort of (dst, src) pairs in out-CSR order => in-neighbours ascending
  const uint32_t* kin = nbr.get();
  uint32_t* kout = keys_out.get();
  const uint32_t* vin = src.get();
  uint32_t* vout = in_nbr.get();
  const int bits = bits_for(n);
  const uint64_t mm = m;
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, kin, kout, vin, vout, (int64_t)mm, 0, bits, st);
  }, st);
  offsets_from_src(keys_out.get(), m, n, in_off.get(), st);
  // compacted row list of the transpose (in-degree > 0)
  DevBuf<unsigned> flag(n + 1), pos(n + 1);
  PPRG_CUDA(cudaMemsetAsync(flag.get() + n, 0, 4, st));
  k_nonempty<<<blocks_for(n), TB, 0, st>>>(in_off.get(), n, flag.get());
  unsigned* fp = flag.get();
  unsigned* pp = pos.get();
  const uint64_t nn = n;
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, fp, pp, (int64_t)(nn + 1), st);
  }, st);
  unsigned nr = 0;
  PPRG_CUDA(cudaMemcpyAsync(&nr, pos.get() + n, 4, cudaMemcpyDeviceToHost, st));
  PPRG_CUDA(cudaStreamSynchronize(st));
  n_rows = nr;
  cin_off.alloc(n_rows + 1);
  cin_row.alloc(n_rows ? n_rows : 1);
  k_compact_rows<<<blocks_for(n), TB, 0, st>>>(in_off.get(), flag.get(), pos.get(), n, m,
                                               cin_off.get(), cin_row.get(), n_rows);
  cin_deg.alloc(n_rows ? n_rows : 1);
  cin_inv.alloc(n_rows ? n_rows : 1);
  if (n_rows)
    k_row_degs<<<blocks_for(n_rows), TB, 0, st>>>(cin_row.get(), n_rows, deg.get(), inv_deg.get(),
                                                  cin_deg.get(), cin_inv.get());
  PPRG_CUDA(cudaStreamSynchronize(st));
  PPRG_CUDA(cudaGetLastError());
}

const uint2* Graph::tile_desc(uint32_t T, uint64_t* ntiles) {
  std::lock_guard<std::recursive_mutex> lk(build_mu);
  ensure_transpose();
  *ntiles = m / T + 1;
  auto it = tile_d.find(T);
  if (it != tile_d.end()) return it->second.get();
  DevBuf<uint2> d(*ntiles);
  k_tile_desc<<<blocks_for(*ntiles), TB, 0, stream>>>(cin_off.get(), n_rows, m, *ntiles, T, d.get());
  PPRG_CUDA(cudaStreamSynchronize(stream));
  PPRG_CUDA(cudaGetLastError());
  const uint2* p = d.get();
  tile_d.emplace(T, std::move(d));
  return p;
}

const uint32_t* Graph::split_rows(uint32_t T, uint64_t* count) {
  std::lock_guard<std::recursive_mutex> lk(build_mu);
  ensure_transpose();
  auto it = tile_split.find(T);
  if (it != tile_split.end()) {
    *count = it->second.n;
    return it->second.get();
  }
  cudaStream_t st = stream;
  const uint64_t nr = n_rows;
  DevBuf<unsigned> flag(nr + 1), pos(nr + 1);
  PPRG_CUDA(cudaMemsetAsync(flag.get(), 0, 4 * (nr + 1), st));
  if (nr) k_split_flags<<<blocks_for(nr), TB, 0, st>>>(cin_off.get(), nr, T, flag.get());
  unsigned* fp = flag.get();
  unsigned* pp = pos.get();
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, fp, pp, (int64_t)(nr + 1), st);
  }, st);
  unsigned cnt = 0;
  PPRG_CUDA(cudaMemcpyAsync(&cnt, pos.get() + nr, 4, cudaMemcpyDeviceToHost, st));
  PPRG_CUDA(cudaStreamSynchronize(st));
  DevBuf<uint32_t> list(cnt ? cnt : 1);
  if (nr) k_scatter_flagged<<<blocks_for(nr), TB, 0, st>>>(flag.get(), pos.get(), nr, list.get());
  PPRG_CUDA(cudaStreamSynchronize(st));
  PPRG_CUDA(cudaGetLastError());
  list.n = cnt;
  *count = cnt;
  const uint32_t* p = list.get();
  tile_split.emplace(T, std::move(list));
  return p;
}

// Greedy row-aligned packing in id order (so sweeps stay id-ordered): rows are
// added to the current tile while it keeps <= T in-edges and <= R rows; a row
// with more than T in-edges becomes ceil(deg/T) hub pieces of its own.
const Graph::Plan& Graph::tile_plan(uint32_t T, uint32_t R, uint32_t H) {
  std::lock_guard<std::recursive_mutex> lk(build_mu);
  ensure_transpose();
  if (H < T) H = T;
  const uint64_t key = ((uint64_t)T << 40) | ((uint64_t)H << 16) | R;
  auto it = plans.find(key);
  if (it != plans.end()) return it->second;
  std::vector<uint64_t> h_off(n_rows + 1);
  PPRG_CUDA(cudaMemcpyAsync(h_off.data(), cin_off.get(), 8 * (n_rows + 1), cudaMemcpyDeviceToHost, stream));
  PPRG_CUDA(cudaStreamSynchronize(stream));
  std::vector<TileDesc> tl;
  tl.reserve(m / T + n_rows / R + 16);
  uint32_t nhubs = 0;
  TileDesc cur{0, 0, 0, 0, 0, 0, 1};
  auto close = [&] {
    if (cur.nr) tl.push_back(cur);
    cur = TileDesc{0, 0, 0, 0, 0, 0, 1};
  };
  for (uint64_t r = 0; r < n_rows; ++r) {
    const uint64_t d = h_off[r + 1] - h_off[r];
    if (d > H) {
      close();
      const uint32_t np = (uint32_t)((d + H - 1) / H);
      for (uint32_t p = 0; p < np; ++p) {
        const uint64_t e0 = h_off[r] + (uint64_t)p * H;
        const uint64_t ne = std::min<uint64_t>(H, h_off[r + 1] - e0);
        tl.push_back(TileDesc{e0, (uint32_t)ne, (uint32_t)r, 1, nhubs, p, np});
      }
      ++nhubs;
      continue;
    }
    if (d > T) {  // a long row, whole, in a tile of its own
      close();
      tl.push_back(TileDesc{h_off[r], (uint32_t)d, (uint32_t)r, 1, 0, 0, 1});
      continue;
    }
    if (cur.nr && (cur.ne + d > T || cur.nr >= R)) close();
    if (!cur.nr) {
      cur.e0 = h_off[r];
      cur.r0 = (uint32_t)r;
    }
    cur.ne += (uint32_t)d;
    cur.nr += 1;
  }
  close();
  Plan pl;
  pl.ntiles = tl.size();
  pl.nhubs = nhubs;
  pl.tiles.alloc(tl.size() ? tl.size() : 1);
  if (!tl.empty())
    PPRG_CUDA(cudaMemcpyAsync(pl.tiles.get(), tl.data(), sizeof(TileDesc) * tl.size(),
                              cudaMemcpyHostToDevice, stream));
  PPRG_CUDA(cudaStreamSynchronize(stream));
  pl.host = std::move(tl);
  return plans.emplace(key, std::move(pl)).first->second;
}

static cudaStream_t make_stream(int device, int* sms) {
  PPRG_CUDA(cudaSetDevice(device));
  cudaStream_t st;
  PPRG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  PPRG_CUDA(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, device));
  return st;
}

std::unique_ptr<Graph> graph_from_csr(const uint64_t* h_off, const uint32_t* h_nbr, uint64_t n,
                                      int device) {
  if (n > 0xffffffffull) fail(EINVAL_, "graph: n exceeds the NodeId range");
  DeviceGuard dg(device);
  auto g = std::make_unique<Graph>();
  g->device = device;
  g->stream = make_stream(device, &g->sm_count);
  g->n = n;
  g->off.alloc(n + 1);
  PPRG_CUDA(cudaMemcpyAsync(g->off.get(), h_off, 8 * (n + 1), cudaMemcpyHostToDevice, g->stream));
  g->m = h_off[n];
  g->nbr.alloc(g->m ? g->m : 1);
  if (g->m)
    PPRG_CUDA(cudaMemcpyAsync(g->nbr.get(), h_nbr, 4 * g->m, cudaMemcpyHostToDevice, g->stream));
  g->finish_build();
  return g;
}

// PPRG cache (graph.cpp:115-149) straight into device memory; same checks and
// messages as load_graph_cache, then the usual device-side validation.
std::unique_ptr<Graph> graph_load_cache(const std::string& path, int device) {
  FileCloser fc;
  fc.f = std::fopen(path.c_str(), "rb");
  if (!fc.f) fail(EDATA, "cannot open graph cache: " + path);
  char magic[4];
  if (std::fread(magic, 1, 4, fc.f) != 4 || std::memcmp(magic, "PPRG", 4) != 0)
    fail(EDATA, path + ": not a graph cache (bad magic)");
  unsigned char ver = 0;
  if (std::fread(&ver, 1, 1, fc.f) != 1 || ver != 1)
    fail(EDATA, path + ": unsupported graph cache version");
  uint64_t nm[2];
  if (std::fread(nm, 8, 2, fc.f) != 2) fail(EDATA, path + ": truncated graph cache");
  const uint64_t n = nm[0], m = nm[1];
  const uint64_t body = 21ull + 8ull * (n + 1) + 4ull * m;
  if (n >= (1ull << 40) || m >= (1ull << 40) || file_size(fc.f) < body)
    fail(EDATA, path + ": truncated graph cache");
  if (n > 0xffffffffull) fail(EINVAL_, "graph: n exceeds the NodeId range");
  DeviceGuard dg(device);
  auto g = std::make_unique<Graph>();
  g->device = device;
  g->stream = make_stream(device, &g->sm_count);
  g->n = n;
  g->m = m;
  g->off.alloc(n + 1);
  g->nbr.alloc(m ? m : 1);
  {
    Staging stg(g->stream);
    if (!stg.read(fc.f, g->off.get(), 8 * (n + 1)) || !stg.read(fc.f, g->nbr.get(), 4 * m))
      fail(EDATA, path + ": truncated graph cache");
  }
  g->finish_build();
  return g;
}

void graph_save_cache(Graph& g, const std::string& path) {
  DeviceGuard dg(g.device);
  std::lock_guard<std::mutex> lk(g.mu);
  FileCloser fc;
  fc.f = std::fopen(path.c_str(), "wb");
  if (!fc.f) fail(EDATA, "cannot open for writing: " + path);
  const unsigned char ver = 1;
  const uint64_t nm[2] = {g.n, g.m};
  bool ok = std::fwrite("PPRG", 1, 4, fc.f) == 4 && std::fwrite(&ver, 1, 1, fc.f) == 1 &&
            std::fwrite(nm, 8, 2, fc.f) == 2;
  Staging stg(g.stream);
  ok = ok && stg.write(fc.f, g.off.get(), 8 * (g.n + 1)) && stg.write(fc.f, g.nbr.get(), 4 * g.m);
  if (!ok || std::fflush(fc.f) != 0) fail(EDATA, "write failed: " + path);
}

std::unique_ptr<Graph> graph_from_edges(const uint64_t* h_pairs, uint64_t count, int device) {
  if (count == 0) fail(EDATA, "graph is empty after cleaning");  // graph.cpp:37
  DeviceGuard dg(device);
  int sms = 0;
  cudaStream_t st = make_stream(device, &sms);
  DevBuf<uint64_t> pairs(2 * count), ids(2 * count), ids_sorted(2 * count), uniq(2 * count);
  PPRG_CUDA(cudaMemcpyAsync(pairs.get(), h_pairs, 16 * count, cudaMemcpyHostToDevice, st));
  k_split_pairs<<<blocks_for(2 * count), TB, 0, st>>>(pairs.get(), count, ids.get());
  uint64_t* a = ids.get();
  uint64_t* b2 = ids_sorted.get();
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, a, b2, (int64_t)(2 * count), 0, 64, st);
  }, st);
  DevBuf<unsigned long long> nsel(1);
  uint64_t* u = uniq.get();
  unsigned long long* ns = nsel.get();
  cub_call([&](void* t, size_t& b) {
    return cub::DeviceSelect::Unique(t, b, b2, u, ns, (int64_t)(2 * count), st);
  }, st);
  unsigned long long n = 0;
  PPRG_CUDA(cudaMemcpyAsync(&n, ns, 8, cudaMemcpyDeviceToHost, st));
  PPRG_CUDA(cudaStreamSynchronize(st));
  if (n > 0xffffffffull) fail(EINVAL_, "graph: n exceeds the NodeId range");
  DevBuf<uint32_t> src(count), dst(count), src_sorted(count);
  k_relabel_search<<<blocks_for(2 * count), TB, 0, st>>>(pairs.get(), count, uniq.get(), n,
                                                         src.get(), dst.get());
  auto g = std::make_unique<Graph>();
  g->device = device;
  g->stream = st;
  g->sm_count = sms;
  g->n = n;
  g->m = count;
  g->nbr.alloc(count);
  g->off.alloc(n + 1);
  const uint32_t* kin = src.get();
  uint32_t* kout = src_sorted.get();
  const uint32_t* vin = dst.get();
  uint32_t* vout = g->nbr.get();
  const int bits = bits_for(n);
  cub_call([&](void* t, size_t& b) {  // stable => input order within a row
    return cub::DeviceRadixSort::SortPairs(t, b, kin, kout, vin, vout, (int64_t)count, 0, bits, st);
  }, st);
  offsets_from_src(src_sorted.get(), count, n, g->off.get(), st);
  g->finish_build();
  return g;
}

std::unique_ptr<Graph> graph_rmat(int scale, uint64_t edge_factor, double a, double b, double c,
                                  uint64_t seed, int device, std::vector<uint64_t>* h_edges_out) {
  if (scale < 1 || scale > 31) fail(EINVAL_, "rmat: scale must be in [1,31]");
  if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0)) fail(EINVAL_, "rmat: bad quadrant probabilities");
  DeviceGuard dg(device);
  int sms = 0;
  cudaStream_t st = make_stream(device, &sms);
  const uint64_t draws = edge_factor << scale;
  DevBuf<uint64_t> keys(draws ? draws : 1);
  k_rmat<<<blocks_for(draws), TB, 0, st>>>(seed, scale, draws, a, a + b, a + b + c, keys.get());
  const uint64_t cnt = sort_clean(keys, draws, 32 + scale, st);
  if (cnt == 0) fail(EDATA, "graph is empty after cleaning");
  if (h_edges_out) {
    h_edges_out->resize(cnt);
    PPRG_CUDA(cudaMemcpyAsync(h_edges_out->data(), keys.get(), 8 * cnt, cudaMemcpyDeviceToHost, st));
  }
  auto g = build_from_sorted_keys(keys, cnt, 1ull << scale, device, st);
  g->sm_count = sms;
  return g;
}

std::unique_ptr<Graph> graph_chung_lu(uint64_t n_raw, uint64_t draws, double beta, uint64_t seed,
                                      int device, std::vector<uint64_t>* h_edges_out) {
  if (n_raw < 2 || n_raw > 0xffffffffull) fail(EINVAL_, "chung-lu: bad n");
  if (!(beta > 2.0)) fail(EINVAL_, "chung-lu: beta must exceed 2");
  DeviceGuard dg(device);
  int sms = 0;
  cudaStream_t st = make_stream(device, &sms);
  // w_i ~ (i+1)^(-1/(beta-1)); in-weights are a seeded permutation of them
  DevBuf<double> w(n_raw), w_in(n_raw), cdf_out(n_raw), cdf_in(n_raw);
  k_cl_weights<<<blocks_for(n_raw), TB, 0, st>>>(n_raw, 1.0 / (beta - 1.0), w.get());
  {
    DevBuf<uint64_t> pk(n_raw), pk2(n_raw);
    DevBuf<uint32_t> pv(n_raw), pv2(n_raw);
    k_perm_keys<<<blocks_for(n_raw), TB, 0, st>>>(seed ^ 0x5A5A5A5A5A5A5A5Aull, n_raw, pk.get(), pv.get());
    uint64_t* k1 = pk.get();
    uint64_t* k2 = pk2.get();
    uint32_t* v1 = pv.get();
    uint32_t* v2 = pv2.get();
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, k1, k2, v1, v2, (int64_t)n_raw, 0, 64, st);
    }, st);
    k_gather_w<<<blocks_for(n_raw), TB, 0, st>>>(w.get(), pv2.get(), n_raw, w_in.get());
  }
  double* wp = w.get();
  double* wi = w_in.get();
  double* co = cdf_out.get();
  double* ci = cdf_in.get();
  cub_call([&](void* t, size_t& b) { return cub::DeviceScan::InclusiveSum(t, b, wp, co, (int64_t)n_raw, st); }, st);
  cub_call([&](void* t, size_t& b) { return cub::DeviceScan::InclusiveSum(t, b, wi, ci, (int64_t)n_raw, st); }, st);
  DevBuf<uint64_t> keys(draws ? draws : 1);
  k_chung_lu<<<blocks_for(draws), TB, 0, st>>>(seed, draws, cdf_out.get(), cdf_in.get(), n_raw,
                                               keys.get());
  const uint64_t cnt = sort_clean(keys, draws, 32 + bits_for(n_raw), st);
  if (cnt == 0) fail(EDATA, "graph is empty after cleaning");
  if (h_edges_out) {
    h_edges_out->resize(cnt);
    PPRG_CUDA(cudaMemcpyAsync(h_edges_out->data(), keys.get(), 8 * cnt, cudaMemcpyDeviceToHost, st));
  }
  auto g = build_from_sorted_keys(keys, cnt, n_raw, device, st);
  g->sm_count = sms;
  return g;
}

}  // namespace pprg
