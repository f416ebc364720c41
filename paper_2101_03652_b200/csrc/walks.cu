// SpeedPPR (hot-path subsystem (4)): Philox alpha-random walks, the
// epsilon-independent walk index, and the Monte Carlo phase.
// Reference: speedppr.cpp:8-111, walk_index.cpp:10-54.
//
// RNG: the reference draws every walk from one sequential
// mt19937_64 stream, which cannot be parallelised bit-exactly. Here step t of
// walk k out of node v is Philox4x32-10(key = seed, ctr = (k, v, tag, t)) with
// tag = query source (MC walks) or 0xFFFFFFFF (index walks), so every walk is
// independent and reproducible; terminals are bit-identical to the oracle's
// restatement (oracle.c og_philox_walk) and the index is byte-identical per
// seed. Stored index files carry rng-id 2 (PPRG_RNG_PHILOX4X32_10).
#include <algorithm>
#include <cub/cub.cuh>

#include <cmath>
#include <cstring>
#include <vector>

#include "fileio.h"
#include "internal.h"

namespace pprg {
namespace {

inline unsigned gridn(uint64_t items, int tb = 256) {
  uint64_t b = (items + tb - 1) / tb;
  if (b == 0) b = 1;
  if (b > 65535ull * 64) b = 65535ull * 64;
  return (unsigned)b;
}

__device__ __forceinline__ uint64_t row_of(const uint64_t* off, uint64_t n, uint64_t e) {
  uint64_t lo = 0, hi = n;  // last v with off[v] <= e
  while (lo < hi) {
    const uint64_t mid = (lo + hi + 1) >> 1;
    if (off[mid] <= e) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// build_index (walk_index.cpp:44-54): deg(v) walks from every v with v as
// its own pseudo-source; one thread per slot, slot k of v keyed (k, v).
__global__ void k_index(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint64_t m,
                        double alpha, uint64_t seed, uint32_t* ep) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = row_of(off, n, e);
    ep[e] = philox_walk(off, nbr, (uint32_t)v, (uint32_t)v, alpha, seed, (uint32_t)(e - off[v]),
                        (uint32_t)v, kIndexTag);
  }
}

__global__ void k_check_index(const uint32_t* ep, uint64_t m, uint64_t n, unsigned* bad) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
       e += (uint64_t)gridDim.x * blockDim.x)
    if (ep[e] >= n) atomicOr(bad, 1u);
}

__global__ void k_terminals(const uint64_t* off, const uint32_t* nbr, const uint32_t* starts,
                            const uint32_t* ks, const uint32_t* vs, uint64_t count, uint32_t source,
                            uint32_t tag, double alpha, uint64_t seed, uint32_t* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = philox_walk(off, nbr, starts[i], source, alpha, seed, ks[i], vs[i], tag);
}

// W_v = ceil(r W), clamped to deg_eff within the reference's slack
// (speedppr.cpp:30-40); counts for padding columns are 0. Per-column walk
// totals accumulate in shared memory (K <= 64), flushed once per block.
__global__ void k_mc_counts(const double* res, const uint32_t* deg, uint64_t n, int K, int k,
                            double W, unsigned long long* cnt, unsigned* bad,
                            unsigned long long* colw) {
  __shared__ unsigned long long s_w[64];
  for (int c = threadIdx.x; c < 64; c += blockDim.x) s_w[c] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n * K;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % K);
    const double r = res[i];
    unsigned long long wc = 0;
    if (c < k && r > 0.0) {
      const uint32_t d = deg[i / K];
      const double de = d ? (double)d : 1.0;
      wc = (unsigned long long)ceil(r * W);
      if ((double)wc > de) {
        if (r * W > de * (1.0 + 1e-9) + 1e-9) atomicOr(bad, 1u);
        wc = (unsigned long long)de;
      }
      if (wc) atomicAdd(&s_w[c], wc);
    }
    cnt[i] = wc;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < K; c += blockDim.x)
    if (s_w[c]) atomicAdd(colw + c, s_w[c]);
}

__global__ void k_est_init(const double* x, uint64_t nk, double alpha, double* est) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nk;
       i += (uint64_t)gridDim.x * blockDim.x)
    est[i] = alpha * x[i];
}

struct McParams {
  const uint64_t* off;
  const uint32_t* nbr;
  const uint32_t* deg;
  const double* res;
  const unsigned long long* cnt;
  const uint32_t* index;           // may be null
  uint64_t nk;
  int K;
  double alpha;
  uint64_t seed;
  double* est;
  uint32_t src[64];
  double sc[64];  // deterministic mode: fixed-point scale of column c's sum (qterm)
};

// Deterministic mode: walk contributions are summed as integers (the
// contribution * 2^S rounded; exact fp64 sums while every partial sum stays
// below 2^53) into a zeroed accumulator, so the order of the atomics does not
// matter; k_est_combine then adds the reserve: est = base_scale * base + acc / sc.
template <bool DET>
__device__ __forceinline__ double mc_term(double v, const McParams& P, int c) {
  if constexpr (DET) return rint(v * P.sc[c]);
  else return v;
}
__global__ void k_est_combine(const double* base, double base_scale, uint64_t nk, int K,
                              const double* sc, double* est) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nk;
       i += (uint64_t)gridDim.x * blockDim.x)
    est[i] = (base ? base_scale * base[i] : 0.0) + est[i] / sc[i % K];
}
// fixed-point scale for a column whose contributions sum to at most `bound`
inline double det_scale_host(double bound) {
  int e = 0;
  std::frexp(bound > 1e-280 ? bound : 1e-280, &e);
  return std::ldexp(1.0, 52 - e);
}

// One walk's terminal: a stored index terminal (index prefix,
// speedppr.cpp:66-71) or a fresh Philox walk keyed (seed, source, (k, v)).
__device__ __forceinline__ uint32_t mc_terminal(const McParams& P, uint32_t v, int c, uint32_t kk) {
  if (P.index && P.deg[v]) return P.index[P.off[v] + kk];
  return philox_walk(P.off, P.nbr, v, P.src[c], P.alpha, P.seed, kk, v, P.src[c]);
}

// Entries (v, c) with W_v <= 32 walks: one thread each, its walks in a loop;
// larger entries go to a list for k_mc_big (warp per entry).
template <bool DET>
__global__ void k_mc_entries(const __grid_constant__ McParams P, uint64_t* big,
                             unsigned long long* nbig) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < P.nk;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long wc = P.cnt[i];
    if (!wc) continue;
    if (wc > 32) {
      big[atomicAdd(nbig, 1ull)] = i;
      continue;
    }
    const uint32_t v = (uint32_t)(i / P.K);
    const int c = (int)(i % P.K);
    const double contribution = mc_term<DET>(P.res[i] / (double)wc, P, c);  // speedppr.cpp:41
    // four walks' terminals resolved before their adds (independent loads in
    // flight). A walk stops at v itself with probability alpha: those are
    // counted and added once (one atomic instead of ~alpha * wc).
    uint32_t kk = 0, self = 0;
    for (; kk + 4 <= (uint32_t)wc; kk += 4) {
      uint32_t t[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) t[j] = mc_terminal(P, v, c, kk + j);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (t[j] == v) ++self;
        else atomicAdd(P.est + (uint64_t)t[j] * P.K + c, contribution);
      }
    }
    for (; kk < (uint32_t)wc; ++kk) {
      const uint32_t t = mc_terminal(P, v, c, kk);
      if (t == v) ++self;
      else atomicAdd(P.est + (uint64_t)t * P.K + c, contribution);
    }
    if (self) atomicAdd(P.est + i, (double)self * contribution);
  }
}

template <bool DET>
__global__ void k_mc_big(const __grid_constant__ McParams P, const uint64_t* big,
                         const unsigned long long* nbig_p) {
  const unsigned long long nbig = *nbig_p;
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t w = w0; w < nbig; w += nw) {
    const uint64_t i = big[w];
    const uint32_t v = (uint32_t)(i / P.K);
    const int c = (int)(i % P.K);
    const unsigned long long wc = P.cnt[i];
    const double contribution = mc_term<DET>(P.res[i] / (double)wc, P, c);
    unsigned long long kk = lane;
    unsigned self = 0;  // walks that stop at v itself, added once per warp
    for (; kk + 96 < wc; kk += 128) {  // four walks per lane resolved before their adds
      uint32_t t[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) t[j] = mc_terminal(P, v, c, (uint32_t)(kk + 32 * j));
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (t[j] == v) ++self;
        else atomicAdd(P.est + (uint64_t)t[j] * P.K + c, contribution);
      }
    }
    for (; kk < wc; kk += 32) {
      const uint32_t t = mc_terminal(P, v, c, (uint32_t)kk);
      if (t == v) ++self;
      else atomicAdd(P.est + (uint64_t)t * P.K + c, contribution);
    }
    self = __reduce_add_sync(0xffffffffu, self);
    if (lane == 0 && self) atomicAdd(P.est + i, (double)self * contribution);
  }
}

// pure-sampling branch (speedppr.cpp:90-102): W walks from s, weight 1/W
__global__ void k_mc_pure(const uint64_t* off, const uint32_t* nbr, uint64_t W, int K, int k,
                          const uint32_t* src, double alpha, uint64_t seed, double* est,
                          double det_w) {  // deterministic mode: the integer 1/W * 2^S, else 0
  const uint64_t total = W * (uint64_t)k;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < total;
       w += (uint64_t)gridDim.x * blockDim.x) {
    const int c = (int)(w / W);
    const uint32_t kk = (uint32_t)(w % W);
    const uint32_t s = src[c];
    const uint32_t t = philox_walk(off, nbr, s, s, alpha, seed, kk, s, s);
    atomicAdd(est + (uint64_t)t * K + c, det_w > 0.0 ? det_w : 1.0 / (double)W);
  }
}

__global__ void k_unpack_est(const double* a, uint64_t n, int K, int k, double* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n * K;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % K);
    if (c < k) out[(uint64_t)c * n + i / K] = a[i];
  }
}

template <typename F>
void cub_run(F&& f) {
  size_t bytes = 0;
  PPRG_CUDA(f(nullptr, bytes));
  DevBuf<unsigned char> tmp(bytes ? bytes : 1);
  PPRG_CUDA(f(tmp.get(), bytes));
}

}  // namespace

std::unique_ptr<WalkIndex> index_build(Graph& g, double alpha, uint64_t seed) {
  DeviceGuard dg(g.device);
  LaneGuard lk(g, true);
  auto w = std::make_unique<WalkIndex>();
  w->device = g.device;
  w->alpha = alpha;
  w->seed = seed;
  w->m = g.m;
  w->endpoints.alloc(g.m ? g.m : 1);
  if (g.m)
    k_index<<<gridn(g.m), 256, 0, g.stream>>>(g.off.get(), g.nbr.get(), g.n, g.m, alpha, seed,
                                              w->endpoints.get());
  PPRG_CUDA(cudaGetLastError());
  PPRG_CUDA(cudaStreamSynchronize(g.stream));
  return w;
}

std::unique_ptr<WalkIndex> index_from_host(Graph& g, double alpha, uint64_t seed,
                                           const uint32_t* h_endpoints) {
  DeviceGuard dg(g.device);
  LaneGuard lk(g, true);
  auto w = std::make_unique<WalkIndex>();
  w->device = g.device;
  w->alpha = alpha;
  w->seed = seed;
  w->m = g.m;
  w->endpoints.alloc(g.m ? g.m : 1);
  DevBuf<unsigned> bad(1);
  PPRG_CUDA(cudaMemsetAsync(bad.get(), 0, 4, g.stream));
  if (g.m) {
    PPRG_CUDA(cudaMemcpyAsync(w->endpoints.get(), h_endpoints, 4 * g.m, cudaMemcpyHostToDevice, g.stream));
    k_check_index<<<gridn(g.m), 256, 0, g.stream>>>(w->endpoints.get(), g.m, g.n, bad.get());
  }
  unsigned hb = 0;
  PPRG_CUDA(cudaMemcpyAsync(&hb, bad.get(), 4, cudaMemcpyDeviceToHost, g.stream));
  PPRG_CUDA(cudaStreamSynchronize(g.stream));
  if (hb) fail(EDATA, "walk index: endpoint id out of range");  // walk_index.cpp:32-33
  return w;
}

namespace {
__global__ void k_cmp_u64(const uint64_t* a, const uint64_t* b, uint64_t n, unsigned* diff) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (a[i] != b[i]) atomicOr(diff, 1u);
}
}  // namespace

// PPRW (walk_index.cpp:57-104) straight into device memory, checked against
// the graph like WalkIndex's constructor + check_compatible (walk_index.cpp:19-42).
std::unique_ptr<WalkIndex> index_load(Graph& g, const std::string& path) {
  DeviceGuard dg(g.device);
  LaneGuard lk(g, true);
  FileCloser fc;
  fc.f = std::fopen(path.c_str(), "rb");
  if (!fc.f) fail(EDATA, "cannot open walk index: " + path);
  char magic[4];
  if (std::fread(magic, 1, 4, fc.f) != 4 || std::memcmp(magic, "PPRW", 4) != 0)
    fail(EDATA, path + ": not a walk index (bad magic)");
  unsigned char vr[2] = {0, 0};
  if (std::fread(vr, 1, 2, fc.f) != 2 || vr[0] != 1) fail(EDATA, path + ": unsupported walk index version");
  if (vr[1] != 2) fail(EDATA, path + ": unknown generator id");  // rng-id 2 = Philox4x32-10
  double alpha = 0;
  uint64_t snm[3];
  if (std::fread(&alpha, 8, 1, fc.f) != 1 || std::fread(snm, 8, 3, fc.f) != 3)
    fail(EDATA, path + ": truncated walk index");
  const uint64_t n = snm[1], m = snm[2];
  if (n != g.n || m != g.m) fail(EDATA, "walk index does not match the graph shape");
  if (file_size(fc.f) < 38ull + 8ull * (n + 1) + 4ull * m) fail(EDATA, path + ": truncated walk index");
  auto w = std::make_unique<WalkIndex>();
  w->device = g.device;
  w->alpha = alpha;
  w->seed = snm[0];
  w->m = m;
  w->endpoints.alloc(m ? m : 1);
  DevBuf<uint64_t> off(n + 1);
  DevBuf<unsigned> flags(2);
  PPRG_CUDA(cudaMemsetAsync(flags.get(), 0, 8, g.stream));
  {
    Staging stg(g.stream);
    if (!stg.read(fc.f, off.get(), 8 * (n + 1)) || !stg.read(fc.f, w->endpoints.get(), 4 * m))
      fail(EDATA, path + ": truncated walk index");
  }
  k_cmp_u64<<<gridn(n + 1), 256, 0, g.stream>>>(off.get(), g.off.get(), n + 1, flags.get());
  if (m) k_check_index<<<gridn(m), 256, 0, g.stream>>>(w->endpoints.get(), m, n, flags.get() + 1);
  unsigned hf[2] = {0, 0};
  PPRG_CUDA(cudaMemcpyAsync(hf, flags.get(), 8, cudaMemcpyDeviceToHost, g.stream));
  PPRG_CUDA(cudaStreamSynchronize(g.stream));
  if (hf[0]) fail(EDATA, "walk index slice length differs from out-degree");
  if (hf[1]) fail(EDATA, "walk index: endpoint id out of range");
  return w;
}

void index_save(Graph& g, const WalkIndex& w, const std::string& path) {
  DeviceGuard dg(g.device);
  LaneGuard lk(g, true);
  FileCloser fc;
  fc.f = std::fopen(path.c_str(), "wb");
  if (!fc.f) fail(EDATA, "cannot open for writing: " + path);
  const unsigned char vr[2] = {1, 2};
  const uint64_t snm[3] = {w.seed, g.n, g.m};
  bool ok = std::fwrite("PPRW", 1, 4, fc.f) == 4 && std::fwrite(vr, 1, 2, fc.f) == 2 &&
            std::fwrite(&w.alpha, 8, 1, fc.f) == 1 && std::fwrite(snm, 8, 3, fc.f) == 3;
  Staging stg(g.stream);
  ok = ok && stg.write(fc.f, g.off.get(), 8 * (g.n + 1)) && stg.write(fc.f, w.endpoints.get(), 4 * g.m);
  if (!ok || std::fflush(fc.f) != 0) fail(EDATA, "write failed: " + path);
}

// monte_carlo_phase (speedppr.cpp:23-72) on a caller push state (host
// reserve / residue of one source): W_v walks per node with residue, index
// prefixes where v has out-edges, fresh Philox walks otherwise.
void monte_carlo(Graph& g, const WalkIndex* idx, uint32_t s, double alpha, uint64_t W, uint64_t seed,
                 const double* h_reserve, const double* h_residue, double* h_est, uint64_t* walks) {
  DeviceGuard dg(g.device);
  LaneGuard lk(g, false);  // one source: a lane
  if (s >= g.n) fail(EINVAL_, "monte carlo: source out of range");
  const uint64_t n = g.n;
  cudaStream_t st = qstream(g);
  DevBuf<double> res(n), est(n);
  DevBuf<unsigned long long> cnt(n), colw(65);
  DevBuf<uint64_t> big(n);
  DevBuf<unsigned> bad(1);
  DevBuf<uint32_t> dsrc(1);
  const bool det = t_det;
  DevBuf<double> base(det ? n : 0), dsc(det ? 1 : 0);
  PPRG_CUDA(cudaMemcpyAsync(res.get(), h_residue, 8 * n, cudaMemcpyHostToDevice, st));
  PPRG_CUDA(cudaMemcpyAsync(det ? base.get() : est.get(), h_reserve, 8 * n, cudaMemcpyHostToDevice, st));
  double hsc = 1.0;
  if (det) {
    double rs = 0.0;  // the contributions sum to the residue mass
    for (uint64_t v = 0; v < n; ++v) rs += h_residue[v] > 0 ? h_residue[v] : 0.0;
    hsc = det_scale_host(2.0 * rs);
    PPRG_CUDA(cudaMemsetAsync(est.get(), 0, 8 * n, st));
    PPRG_CUDA(cudaMemcpyAsync(dsc.get(), &hsc, 8, cudaMemcpyHostToDevice, st));
  }
  PPRG_CUDA(cudaMemsetAsync(bad.get(), 0, 4, st));
  PPRG_CUDA(cudaMemsetAsync(colw.get(), 0, 8 * 65, st));
  k_mc_counts<<<std::min<unsigned>(gridn(n), g.sm_count * 8), 256, 0, st>>>(
      res.get(), g.deg.get(), n, 1, 1, (double)W, cnt.get(), bad.get(), colw.get());
  unsigned hb = 0;
  PPRG_CUDA(cudaMemcpyAsync(&hb, bad.get(), 4, cudaMemcpyDeviceToHost, st));
  PPRG_CUDA(cudaStreamSynchronize(st));
  if (hb) fail(EINTERNAL, "monte carlo: residue exceeds degree/W, state not refined");
  McParams P;
  std::memset(&P, 0, sizeof P);
  P.off = g.off.get();
  P.nbr = g.nbr.get();
  P.deg = g.deg.get();
  P.res = res.get();
  P.cnt = cnt.get();
  P.index = idx ? idx->endpoints.get() : nullptr;
  P.nk = n;
  P.K = 1;
  P.alpha = alpha;
  P.seed = seed;
  P.est = est.get();
  P.src[0] = s;
  P.sc[0] = hsc;
  if (det) {
    k_mc_entries<true><<<gridn(n), 256, 0, st>>>(P, big.get(), colw.get() + 64);
    k_mc_big<true><<<g.sm_count * 8, 256, 0, st>>>(P, big.get(), colw.get() + 64);
    k_est_combine<<<gridn(n), 256, 0, st>>>(base.get(), 1.0, n, 1, dsc.get(), est.get());
  } else {
    k_mc_entries<false><<<gridn(n), 256, 0, st>>>(P, big.get(), colw.get() + 64);
    k_mc_big<false><<<g.sm_count * 8, 256, 0, st>>>(P, big.get(), colw.get() + 64);
  }
  PPRG_CUDA(cudaGetLastError());
  unsigned long long hw = 0;
  PPRG_CUDA(cudaMemcpyAsync(h_est, est.get(), 8 * n, cudaMemcpyDeviceToHost, st));
  PPRG_CUDA(cudaMemcpyAsync(&hw, colw.get(), 8, cudaMemcpyDeviceToHost, st));
  PPRG_CUDA(cudaStreamSynchronize(st));
  *walks = hw;
}

void walk_terminals(Graph& g, const uint32_t* h_start, const uint32_t* h_k, const uint32_t* h_v,
                    uint64_t count, uint32_t source, uint32_t tag, double alpha, uint64_t seed,
                    uint32_t* h_out) {
  DeviceGuard dg(g.device);
  LaneGuard lk(g, true);
  if (!count) return;
  DevBuf<uint32_t> s(count), kk(count), v(count), o(count);
  PPRG_CUDA(cudaMemcpyAsync(s.get(), h_start, 4 * count, cudaMemcpyHostToDevice, g.stream));
  PPRG_CUDA(cudaMemcpyAsync(kk.get(), h_k, 4 * count, cudaMemcpyHostToDevice, g.stream));
  PPRG_CUDA(cudaMemcpyAsync(v.get(), h_v, 4 * count, cudaMemcpyHostToDevice, g.stream));
  k_terminals<<<gridn(count), 256, 0, g.stream>>>(g.off.get(), g.nbr.get(), s.get(), kk.get(),
                                                  v.get(), count, source, tag, alpha, seed, o.get());
  PPRG_CUDA(cudaGetLastError());
  PPRG_CUDA(cudaMemcpyAsync(h_out, o.get(), 4 * count, cudaMemcpyDeviceToHost, g.stream));
  PPRG_CUDA(cudaStreamSynchronize(g.stream));
}

namespace {
// Per-call Monte Carlo buffers and the two-slot output staging of speedppr().
struct McState {
  DevBuf<unsigned long long> cnt, colw;
  DevBuf<uint64_t> big;
  DevBuf<double> est, stage[2], sc;
  DevBuf<unsigned> bad;
  uint64_t nk = 0;
  unsigned slot = 0;
  cudaStream_t copy_st = nullptr;
  cudaEvent_t ready[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};
  explicit McState(cudaStream_t st) {
    colw.alloc(65);
    bad.alloc(1);
    PPRG_CUDA(cudaStreamCreateWithFlags(&copy_st, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      PPRG_CUDA(cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming));
      PPRG_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
      PPRG_CUDA(cudaEventRecord(done[i], copy_st));
    }
    (void)st;
  }
  ~McState() {
    cudaStreamSynchronize(copy_st);
    for (int i = 0; i < 2; ++i) {
      cudaEventDestroy(ready[i]);
      cudaEventDestroy(done[i]);
    }
    cudaStreamDestroy(copy_st);
  }
};
}  // namespace

void speedppr(Graph& g, const WalkIndex* idx, const uint32_t* sources, uint32_t k, double alpha,
              double epsilon, double mu, uint64_t seed, double* est_out, bool out_on_device,
              ColumnStats* cols, CallStats* call) {
  DeviceGuard dg(g.device);
  LaneGuard lk(g, k > 2);  // narrow batches share the device by lanes
  for (uint32_t c = 0; c < k; ++c)
    if (sources[c] >= g.n) fail(EINVAL_, "speedppr: source out of range");
  const uint64_t n = g.n;
  if (n < 2) fail(EINVAL_, "walk budget: need n >= 2");
  const double mu_eff = mu > 0.0 ? mu : 1.0 / (double)n;
  const uint64_t W = (uint64_t)std::ceil(2.0 * (2.0 * epsilon / 3.0 + 2.0) * std::log((double)n) /
                                         (epsilon * epsilon * mu_eff));  // speedppr.cpp:8-18
  const uint64_t m_eff = g.m_eff();
  cudaStream_t st = qstream(g);
  const cudaMemcpyKind kind = out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  cudaEvent_t e0, e1;
  PPRG_CUDA(cudaEventCreate(&e0));
  PPRG_CUDA(cudaEventCreate(&e1));
  PPRG_CUDA(cudaEventRecord(e0, st));
  McState mc(st);
  // sources per push-stage block (PPRG_SPP_COLUMNS, a power of two <= 64)
  static const uint32_t spp_cols = [] {
    const char* e = std::getenv("PPRG_SPP_COLUMNS");
    const long v = e ? std::strtol(e, nullptr, 10) : 64;
    return (uint32_t)(v == 1 || v == 2 || v == 4 || v == 8 || v == 16 || v == 32 ? v : 64);
  }();
  for (uint32_t b0 = 0; b0 < k; b0 += spp_cols) {
    const uint32_t kb = k - b0 < spp_cols ? k - b0 : spp_cols;
    ColumnStats* cs = cols + b0;
    if (W <= m_eff) {
      int K = 1;
      while (K < (int)kb) K <<= 1;
      DevBuf<double> est(n * K), outb(out_on_device ? 0 : n * kb);
      DevBuf<uint32_t> dsrc(64);
      PPRG_CUDA(cudaMemcpyAsync(dsrc.get(), sources + b0, 4 * kb, cudaMemcpyHostToDevice, st));
      PPRG_CUDA(cudaMemsetAsync(est.get(), 0, 8 * n * K, st));
      if (W > 0xffffffffull) fail(EINVAL_, "speedppr: walk budget exceeds 2^32 walks per query");
      // deterministic mode: walk counts (exact integers), divided by W after
      k_mc_pure<<<gridn(W * kb), 256, 0, st>>>(g.off.get(), g.nbr.get(), W, K, kb, dsrc.get(), alpha,
                                              seed, est.get(), t_det ? 1.0 : 0.0);
      if (t_det) {
        std::vector<double> hs(K, (double)W);
        DevBuf<double> dsc(K);
        PPRG_CUDA(cudaMemcpyAsync(dsc.get(), hs.data(), 8 * K, cudaMemcpyHostToDevice, st));
        k_est_combine<<<gridn(n * K), 256, 0, st>>>(nullptr, 0.0, n * (uint64_t)K, K, dsc.get(), est.get());
        PPRG_CUDA(cudaStreamSynchronize(st));  // dsc is freed at scope exit
      }
      double* dst = est_out ? (out_on_device ? est_out + (uint64_t)b0 * n : outb.get()) : nullptr;
      if (dst) k_unpack_est<<<gridn(n * K), 256, 0, st>>>(est.get(), n, K, kb, dst);
      if (est_out && !out_on_device)
        PPRG_CUDA(cudaMemcpyAsync(est_out + (uint64_t)b0 * n, outb.get(), 8 * n * kb, kind, st));
      PPRG_CUDA(cudaStreamSynchronize(st));
      PPRG_CUDA(cudaGetLastError());
      call->kernel_launches += 2;
      for (uint32_t c = 0; c < kb; ++c) {
        cs[c].walks = W;
        cs[c].pushes = 0;
        cs[c].r_sum = 0;
      }
      continue;
    }
    const double lambda = (double)m_eff / (double)W;
    const double r_max = 1.0 / (double)W;
    PushView pv;
    speedppr_push_stage(g, sources + b0, kb, alpha, lambda, r_max, cs, call, &pv);
    const int K = pv.K;
    const uint64_t nk = n * (uint64_t)K;
    // buffers live across blocks: a cudaFree per block would synchronise the
    // device and serialise the previous block's output copy with this block
    if (!mc.cnt.get() || mc.nk < nk) {
      mc.nk = nk;
      mc.cnt.alloc(nk);
      mc.big.alloc(nk);
      mc.est.alloc(nk);
    }
    unsigned long long* nbig = mc.colw.get() + 64;
    PPRG_CUDA(cudaMemsetAsync(mc.bad.get(), 0, 4, st));
    PPRG_CUDA(cudaMemsetAsync(mc.colw.get(), 0, 8 * 65, st));
    k_mc_counts<<<std::min<unsigned>(gridn(nk), g.sm_count * 8), 256, 0, st>>>(
        pv.res, g.deg.get(), n, K, kb, (double)W, mc.cnt.get(), mc.bad.get(), mc.colw.get());
    const bool det = t_det;
    if (det) PPRG_CUDA(cudaMemsetAsync(mc.est.get(), 0, 8 * nk, st));
    else k_est_init<<<gridn(nk), 256, 0, st>>>(pv.x, nk, alpha, mc.est.get());
    McParams P;
    std::memset(&P, 0, sizeof P);
    P.off = g.off.get();
    P.nbr = g.nbr.get();
    P.deg = g.deg.get();
    P.res = pv.res;
    P.cnt = mc.cnt.get();
    P.index = idx ? idx->endpoints.get() : nullptr;
    P.nk = nk;
    P.K = K;
    P.alpha = alpha;
    P.seed = seed;
    P.est = mc.est.get();
    for (int c = 0; c < K; ++c) P.src[c] = pv.src[c];
    // Entries run thread-per-(v, c); entries over 32 walks are queued and run
    // warp-per-entry by a fixed-size grid that reads the queue length on device.
    if (det) {
      // column c's contributions sum to its residue mass after refine
      std::vector<double> hs(K, 1.0);
      for (uint32_t c = 0; c < kb; ++c) hs[c] = P.sc[c] = det_scale_host(2.0 * cs[c].r_sum);
      for (int c = kb; c < K; ++c) P.sc[c] = 1.0;
      if (!mc.sc.get()) mc.sc.alloc(64);
      PPRG_CUDA(cudaMemcpyAsync(mc.sc.get(), hs.data(), 8 * K, cudaMemcpyHostToDevice, st));
      k_mc_entries<true><<<gridn(nk), 256, 0, st>>>(P, mc.big.get(), nbig);
      k_mc_big<true><<<g.sm_count * 8, 256, 0, st>>>(P, mc.big.get(), nbig);
      k_est_combine<<<gridn(nk), 256, 0, st>>>(pv.x, alpha, nk, K, mc.sc.get(), mc.est.get());
    } else {
      k_mc_entries<false><<<gridn(nk), 256, 0, st>>>(P, mc.big.get(), nbig);
      k_mc_big<false><<<g.sm_count * 8, 256, 0, st>>>(P, mc.big.get(), nbig);
    }
    PPRG_CUDA(cudaGetLastError());
    if (est_out && out_on_device) {
      k_unpack_est<<<gridn(nk), 256, 0, st>>>(mc.est.get(), n, K, kb, est_out + (uint64_t)b0 * n);
    } else if (est_out) {
      // staged: the copy of this block overlaps the next block's compute
      const int slot = mc.slot++ & 1;
      PPRG_CUDA(cudaStreamWaitEvent(st, mc.done[slot], 0));
      mc.stage[slot].ensure(n * 64);
      k_unpack_est<<<gridn(nk), 256, 0, st>>>(mc.est.get(), n, K, kb, mc.stage[slot].get());
      PPRG_CUDA(cudaEventRecord(mc.ready[slot], st));
      PPRG_CUDA(cudaStreamWaitEvent(mc.copy_st, mc.ready[slot], 0));
      PPRG_CUDA(cudaMemcpyAsync(est_out + (uint64_t)b0 * n, mc.stage[slot].get(), 8 * n * kb,
                                cudaMemcpyDeviceToHost, mc.copy_st));
      PPRG_CUDA(cudaEventRecord(mc.done[slot], mc.copy_st));
    }
    unsigned long long hw[65];
    unsigned hb = 0;
    d2h_small(hw, mc.colw.get(), 8 * 65, st);
    d2h_small(&hb, mc.bad.get(), 4, st);
    if (hb) fail(EINTERNAL, "monte carlo: residue exceeds degree/W, state not refined");
    call->kernel_launches += 7;
    for (uint32_t c = 0; c < kb; ++c) cs[c].walks = hw[c];
    for (uint32_t c = 0; c < kb; ++c) cs[c].r_sum = 0;  // speedppr.cpp:47
  }
  PPRG_CUDA(cudaEventRecord(e1, st));
  PPRG_CUDA(cudaEventSynchronize(e1));
  PPRG_CUDA(cudaStreamSynchronize(mc.copy_st));  // every block's estimates are on the host
  float ms = 0;
  PPRG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  call->device_ms += ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

}  // namespace pprg
