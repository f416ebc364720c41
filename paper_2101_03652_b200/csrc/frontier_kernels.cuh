// Device side of the frontier (push-form) levels: the local phase of PowerPush,
// refine and FIFO forward push, plus the small per-block helper kernels.
// Included by push.cu only (one translation unit).
#pragma once
#include "sweep_kernel.cuh"

namespace pprg {
// ---- local phase / refine / FIFO: frontier levels in push form ------------
// Entry = linear index i = u*K + c. One warp per entry: claim r with
// atomicExch (the FIFO pop, push.cpp:38-41), x += r, scatter (1-a) r / deg_eff
// with fp64 RED, and append newly active (t, c) once per level (stamp).
// Frontier of one level: per column c a FIFO segment
// cur[c*seg_cap, c*seg_cap + q_c) of node ids, so an entry's position in its
// segment is the number of pops of column c before it.
struct FrontierParams {
  const uint64_t* off;
  const uint32_t* nbr;
  const uint32_t* deg;
  double* res;
  double* x;
  unsigned* stamp;
  const uint32_t* cur;
  uint32_t* next;
  uint64_t seg_cap;
  uint64_t total;                 // sum of q_c
  unsigned long long* col_cnt;    // [K] appends per column this level (= next segment length)
  double* col_dr;                 // [K] alpha * sum r pushed
  unsigned long long* col_np;     // [K] edge pushes
  unsigned long long* col_nn;     // [K] node pushes
  unsigned* col_stop;             // [K] set when the queue outgrows `limit` (push.cpp:38)
  unsigned long long* col_resv;   // [K] out-degrees reserved by this level's pops
  unsigned long long limit;
  unsigned long long col_live;    // bit c set: column c still in this phase
  unsigned level_tag;
  int K;
  double alpha;
  uint64_t pre[KMAX + 1];         // segment prefix: column c owns [pre[c], pre[c+1])
  uint32_t src[KMAX];
  double thr[KMAX];
};

struct HeavyEntry {  // a frontier node whose scatter is spread over the grid
  uint64_t begin;    // first out-edge
  uint32_t deg;
  uint32_t c;
  double share;
};
constexpr uint32_t HEAVY_DEG = 2048;

// Append t to column c's next segment once per level when it becomes active
// (drain_queue's enqueue test, push.cpp:49-53); one atomic per ballot group.
__device__ __forceinline__ void maybe_append(const FrontierParams& P, bool app, uint32_t t, int c,
                                             unsigned mask) {
  const unsigned bal = __ballot_sync(mask, app);
  if (app) {
    const int lane = threadIdx.x & 31, leader = __ffs(bal) - 1;
    unsigned long long basepos = 0;
    if (lane == leader) basepos = atomicAdd(P.col_cnt + c, (unsigned long long)__popc(bal));
    basepos = __shfl_sync(bal, basepos, leader);
    P.next[(uint64_t)c * P.seg_cap + basepos + __popc(bal & ((1u << lane) - 1u))] = t;
  }
}

__device__ __forceinline__ void relax_scatter(const FrontierParams& P, uint32_t t, int c,
                                              double share, bool ok, unsigned mask) {
  bool app = false;
  if (ok) {
    const uint64_t ti = (uint64_t)t * P.K + c;
    const double nv = atomicAdd(P.res + ti, share) + share;
    const uint32_t td = __ldg(P.deg + t);
    if (nv > (double)(td ? td : 1) * P.thr[c])
      app = atomicExch(P.stamp + ti, P.level_tag) != P.level_tag;
  }
  maybe_append(P, app, t, c, mask);
}

// One warp per frontier entry (v, c): check drain_queue's loop condition
// (queue size <= limit before the pop, push.cpp:38), claim r (the pop,
// push.cpp:40-43), x += r, then scatter (1-a) r / deg_eff to the effective
// out-neighbours with fp64 atomics, 4 independent atomics per lane in flight.
// Entries with more than HEAVY_DEG out-edges are queued for k_frontier_heavy_chunks,
// so a hub never serialises one warp. Per-column counters accumulate in
// shared memory and are flushed once per block.
__global__ void __launch_bounds__(256) k_frontier(const __grid_constant__ FrontierParams P,
                                                  HeavyEntry* heavy, unsigned* heavy_cnt) {
  __shared__ double sh_dr[KMAX];
  __shared__ unsigned long long sh_np[KMAX], sh_nn[KMAX];
  const int K = P.K;
  for (int i = threadIdx.x; i < K; i += blockDim.x) sh_dr[i] = 0, sh_np[i] = 0, sh_nn[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t w = w0; w < P.total; w += nw) {
    int c = 0;
    while (w >= P.pre[c + 1]) ++c;
    if (!((P.col_live >> c) & 1ull)) continue;
    const uint64_t pos = w - P.pre[c];
    const uint32_t v = P.cur[(uint64_t)c * P.seg_cap + pos];
    const uint64_t i = (uint64_t)v * K + c;
    const uint32_t d = P.deg[v];
    double r = 0.0;
    if (lane == 0) {
      bool stop = *(volatile unsigned*)(P.col_stop + c) != 0;
      if (!stop && P.limit != ~0ull) {
        // appends of the pops before this one are bounded by their out-degrees,
        // reserved at pop time, so concurrent warps see the queue growth at once
        const unsigned long long reserved = atomicAdd(P.col_resv + c, (unsigned long long)(d ? d : 1));
        const unsigned long long q = P.pre[c + 1] - P.pre[c];
        if (q - pos + reserved > P.limit) {
          stop = true;
          P.col_stop[c] = 1;
        }
      }
      if (!stop)
        r = __longlong_as_double((long long)atomicExch((unsigned long long*)(P.res + i), 0ull));
    }
    r = __shfl_sync(0xffffffffu, r, 0);
    if (!(r > 0.0)) continue;
    const uint64_t de = d ? d : 1;
    const double share = (1.0 - P.alpha) * r / (double)de;
    const uint64_t b = P.off[v];
    if (lane == 0) {
      P.x[i] += r;
      atomicAdd(&sh_dr[c], P.alpha * r);
      atomicAdd(&sh_np[c], (unsigned long long)de);
      atomicAdd(&sh_nn[c], 1ull);
      if (de > HEAVY_DEG) heavy[atomicAdd(heavy_cnt, 1u)] = HeavyEntry{b, d, (uint32_t)c, share};
    }
    if (de > HEAVY_DEG) continue;
    for (uint64_t q0 = 0; q0 < de; q0 += 128) {
      uint32_t t[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t q = q0 + lane + 32 * k;
        t[k] = q < de ? (d ? __ldg(P.nbr + b + q) : P.src[c]) : 0xFFFFFFFFu;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) relax_scatter(P, t[k], c, share, t[k] != 0xFFFFFFFFu, 0xffffffffu);
    }
  }
  __syncthreads();
  for (int cc = threadIdx.x; cc < K; cc += blockDim.x) {
    if (sh_dr[cc] != 0.0) atomicAdd(P.col_dr + cc, sh_dr[cc]);
    if (sh_np[cc]) atomicAdd(P.col_np + cc, sh_np[cc]);
    if (sh_nn[cc]) atomicAdd(P.col_nn + cc, sh_nn[cc]);
  }
}

// The scatter of heavy entries by chunks of HEAVY_CHUNK out-edges of one entry
// (host-built list: no per-edge search for the owning entry), a block per
// chunk, four neighbour ids per thread loaded before the first atomic. Every
// lane of a chunk shares the entry's column, so appends group the whole warp.
constexpr uint32_t HEAVY_CHUNK = 1024;
struct HeavyChunk {
  uint32_t h;      // heavy entry
  uint32_t first;  // first out-edge of the chunk, relative to the entry
};

__global__ void __launch_bounds__(256) k_frontier_heavy_chunks(const __grid_constant__ FrontierParams P,
                                                               const HeavyEntry* heavy,
                                                               const HeavyChunk* chunks,
                                                               unsigned nchunks) {
  for (unsigned ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const HeavyChunk k = chunks[ch];
    const HeavyEntry e = heavy[k.h];
    const uint32_t end = e.deg - k.first < HEAVY_CHUNK ? e.deg : k.first + HEAVY_CHUNK;
    const uint32_t q0 = k.first + threadIdx.x;
    uint32_t t[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t q = q0 + 256u * i;
      t[i] = q < end ? __ldg(P.nbr + e.begin + q) : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      relax_scatter(P, t[i], (int)e.c, e.share, t[i] != 0xFFFFFFFFu, 0xffffffffu);
  }
}

// Enqueue every active (u, c) in id order (refine, push.cpp:212-218) into
// column c's segment. Order within a segment follows warp-aggregated appends
// over ascending ids.
__global__ void k_scan_active(const double* res, const uint32_t* deg, uint64_t n, int K,
                              const double* thr, unsigned long long col_live, unsigned* stamp,
                              unsigned tag, uint32_t* out, uint64_t seg_cap,
                              unsigned long long* col_cnt) {
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x; i0 < n * K;
       i0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    const bool in = i < n * K;
    const int c = in ? (int)(i % K) : -1;
    const uint32_t d = in ? deg[i / K] : 0;
    const bool a = in && ((col_live >> c) & 1ull) && res[i] > (double)(d ? d : 1) * thr[c];
    const unsigned grp = __match_any_sync(0xffffffffu, c);
    const unsigned bal = __ballot_sync(0xffffffffu, a) & grp;
    if (a) {
      stamp[i] = tag;
      const int lane = threadIdx.x & 31, leader = __ffs(bal) - 1;
      unsigned long long b = 0;
      if (lane == leader) b = atomicAdd(col_cnt + c, (unsigned long long)__popc(bal));
      b = __shfl_sync(bal, b, leader);
      out[(uint64_t)c * seg_cap + b + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)(i / K);
    }
  }
}

// per-column sums of an [n*K] array (exact r_sum recompute, push.cpp:9-15).
// The grid stride is a multiple of K, so each thread only ever sees column
// tid % K: thread-local sums, then one shared atomic per thread.
__global__ void k_colsum(const double* a, uint64_t n, int K, double* out) {
  __shared__ double sh[KMAX];
  if (threadIdx.x < KMAX) sh[threadIdx.x] = 0;
  __syncthreads();
  double loc = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n * K;
       i += (uint64_t)gridDim.x * blockDim.x)
    loc += a[i];
  if (loc != 0.0) atomicAdd(&sh[threadIdx.x % K], loc);
  __syncthreads();
  if (threadIdx.x < K) atomicAdd(out + threadIdx.x, sh[threadIdx.x]);
}

// y = (1-a) x / deg_eff; D = (1-a) sum_dead x
__global__ void k_init_pull(const double* x, const uint32_t* deg, const double* inv_deg,
                            uint64_t n, int K, double alpha, double* y, double* D) {
  __shared__ double sh[KMAX];
  if (threadIdx.x < KMAX) sh[threadIdx.x] = 0;
  __syncthreads();
  double loc = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n * K;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = i / K;
    const double xv = x[i];
    y[i] = (1.0 - alpha) * xv * inv_deg[u];
    if (deg[u] == 0) loc += (1.0 - alpha) * xv;
  }
  if (loc != 0.0) atomicAdd(&sh[threadIdx.x % K], loc);
  __syncthreads();
  if (threadIdx.x < K && sh[threadIdx.x] != 0.0) atomicAdd(D + threadIdx.x, sh[threadIdx.x]);
}

__global__ void k_seed(double* a, const uint32_t* src, int K, double v) {
  const int c = threadIdx.x;
  if (c < K) a[(uint64_t)src[c] * K + c] = v;
}

// interleaved [u*K + c] -> query-major [c*n + u] for live columns
__global__ void k_unpack(const double* a, uint64_t n, int K, int k_live, double scale, double* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n * K;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % K);
    if (c < k_live) out[(uint64_t)c * n + i / K] = scale * a[i];
  }
}

// query-major [c*n + u] -> interleaved [u*K + c] (padding columns 0)
__global__ void k_pack(const double* in, uint64_t n, int K, int k_live, double scale, double* a) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n * K;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % K);
    a[i] = c < k_live ? scale * in[(uint64_t)c * n + i / K] : 0.0;
  }
}

// refine outputs: reserve += alpha * (mass pushed here), residue = res
__global__ void k_refine_out(const double* x, const double* res, uint64_t n, int K, int k_live,
                             double alpha, double* reserve, double* residue) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n * K;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % K);
    if (c >= k_live) continue;
    const uint64_t o = (uint64_t)c * n + i / K;
    if (x[i] != 0.0) reserve[o] += alpha * x[i];
    residue[o] = res[i];
  }
}

// One-column sweeps run as warp tasks (sweep_k1_warps) on graphs with at least
// PPRG_K1W_MIN_M in-edges (default 4M); smaller graphs, where a sweep is a few
// microseconds of latency chains, keep the block-tile path (tile_rows).
inline bool k1w_on(const Graph& g, int K) {
  if (K != 1 || !PPRG_K1W) return false;
  static const uint64_t min_m = [] {
    const char* e = std::getenv("PPRG_K1W_MIN_M");
    return e ? std::strtoull(e, nullptr, 10) : 4000000ull;
  }();
  return g.m >= min_m;
}
// Wide-path tile size: WIDE_T, or smaller on graphs too small to give every
// resident block about PPRG_WIDE_TILES tiles per sweep (a power of two, at
// least 256 in-edges), so small graphs do not leave most of the grid idle.
inline uint32_t wide_tile_edges(const Graph& g) {
  static const double per_block = [] {
    const char* e = std::getenv("PPRG_WIDE_TILES");
    return e ? std::atof(e) : 2.0;
  }();
  if (per_block <= 0) return WIDE_T;
  const double want = (double)g.m / (per_block * 8.0 * (double)g.sm_count);
  uint32_t t = WIDE_T;
  while (t > 256 && (double)t > want) t >>= 1;
  return t;
}
inline uint32_t tile_edges(const Graph& g, int K) {
  if (k1w_on(g, K)) return K1W_T;
  return K >= WIDE_K ? wide_tile_edges(g) : (uint32_t)(SWEEP_ELEMS / K);
}
inline uint32_t tile_hub(const Graph& g, int K) { return k1w_on(g, K) ? K1W_H : tile_edges(g, K); }
inline uint32_t tile_rmax(const Graph& g, int K) {
  if (k1w_on(g, K)) return K1W_R;
  if (K >= WIDE_K) return RMAX_W;
  const int T = SWEEP_ELEMS / K;
  return T < 256 ? T : 256;
}

}  // namespace pprg
