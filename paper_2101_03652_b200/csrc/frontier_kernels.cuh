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

// Where a level's scatter lands: residues, the enqueue test's thresholds and
// stamps, and column c's next segment with its append counter.
struct ScatterCtx {
  double* res;
  const uint32_t* deg;
  const double* thr;              // [K] enqueue threshold per unit of deg_eff
  unsigned* stamp;
  unsigned tag;
  uint32_t* next;
  uint64_t seg_cap;
  int K;
  unsigned long long* col_cnt;    // [K] appends (= next segment length)
};

// Append t to column c's next segment once per level when it becomes active
// (drain_queue's enqueue test, push.cpp:49-53); one atomic per ballot group.
__device__ __forceinline__ void maybe_append(const ScatterCtx& C, bool app, uint32_t t, int c,
                                             unsigned mask) {
  const unsigned bal = __ballot_sync(mask, app);
  if (app) {
    const int lane = threadIdx.x & 31, leader = __ffs(bal) - 1;
    unsigned long long basepos = 0;
    if (lane == leader) basepos = atomicAdd(C.col_cnt + c, (unsigned long long)__popc(bal));
    basepos = __shfl_sync(bal, basepos, leader);
    C.next[(uint64_t)c * C.seg_cap + basepos + __popc(bal & ((1u << lane) - 1u))] = t;
  }
}

__device__ __forceinline__ void relax_scatter(const ScatterCtx& C, uint32_t t, int c, double share,
                                              bool ok, unsigned mask) {
  bool app = false;
  if (ok) {
    const uint64_t ti = (uint64_t)t * C.K + c;
    const double nv = atomicAdd(C.res + ti, share) + share;
    const uint32_t td = __ldg(C.deg + t);
    if (nv > (double)(td ? td : 1) * C.thr[c])
      app = atomicExch(C.stamp + ti, C.tag) != C.tag;
  }
  maybe_append(C, app, t, c, mask);
}

// Per-block counters of a level (shared), flushed once per block.
struct LevelAcc {
  double* dr;
  unsigned long long* np;
  unsigned long long* nn;
};

// One frontier entry (v, c) at position pos of its column's segment of
// length q, popped by one warp: check drain_queue's loop condition (queue
// size <= limit before the pop, push.cpp:38), claim r (the pop,
// push.cpp:40-43), x += r, then scatter (1-a) r / deg_eff to the effective
// out-neighbours with fp64 atomics, 4 independent atomics per lane in flight.
// Entries with more than HEAVY_DEG out-edges are queued for the chunked
// heavy scatter, so a hub never serialises one warp.
__device__ __forceinline__ void pop_entry(const ScatterCtx& C, const uint64_t* off,
                                          const uint32_t* nbr, double* x, double alpha,
                                          uint32_t src_c, unsigned long long limit,
                                          unsigned* col_stop, unsigned long long* col_resv,
                                          uint32_t v, int c, uint64_t pos, uint64_t q,
                                          const LevelAcc& la, HeavyEntry* heavy,
                                          unsigned* heavy_cnt) {
  const int lane = threadIdx.x & 31;
  const uint64_t i = (uint64_t)v * C.K + c;
  const uint32_t d = C.deg[v];
  double r = 0.0;
  if (lane == 0) {
    bool stop = *(volatile unsigned*)(col_stop + c) != 0;
    if (!stop && limit != ~0ull) {
      // appends of the pops before this one are bounded by their out-degrees,
      // reserved at pop time, so concurrent warps see the queue growth at once
      const unsigned long long reserved = atomicAdd(col_resv + c, (unsigned long long)(d ? d : 1));
      if (q - pos + reserved > limit) {
        stop = true;
        col_stop[c] = 1;
      }
    }
    if (!stop) r = __longlong_as_double((long long)atomicExch((unsigned long long*)(C.res + i), 0ull));
  }
  r = __shfl_sync(0xffffffffu, r, 0);
  if (!(r > 0.0)) return;
  const uint64_t de = d ? d : 1;
  const double share = (1.0 - alpha) * r / (double)de;
  const uint64_t b = off[v];
  if (lane == 0) {
    x[i] += r;
    atomicAdd(&la.dr[c], alpha * r);
    atomicAdd(&la.np[c], (unsigned long long)de);
    atomicAdd(&la.nn[c], 1ull);
    if (de > HEAVY_DEG) heavy[atomicAdd(heavy_cnt, 1u)] = HeavyEntry{b, d, (uint32_t)c, share};
  }
  if (de > HEAVY_DEG) return;
  for (uint64_t q0 = 0; q0 < de; q0 += 128) {
    uint32_t t[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t qq = q0 + lane + 32 * k;
      t[k] = qq < de ? (d ? __ldg(nbr + b + qq) : src_c) : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) relax_scatter(C, t[k], c, share, t[k] != 0xFFFFFFFFu, 0xffffffffu);
  }
}

// One level, one warp per frontier entry (host-driven drain: observed or
// traced calls). Per-column counters accumulate in shared memory and are
// flushed once per block.
__global__ void __launch_bounds__(256) k_frontier(const __grid_constant__ FrontierParams P,
                                                  HeavyEntry* heavy, unsigned* heavy_cnt) {
  __shared__ double sh_dr[KMAX];
  __shared__ unsigned long long sh_np[KMAX], sh_nn[KMAX];
  __shared__ double sh_thr[KMAX];
  const int K = P.K;
  for (int i = threadIdx.x; i < K; i += blockDim.x)
    sh_dr[i] = 0, sh_np[i] = 0, sh_nn[i] = 0, sh_thr[i] = P.thr[i];
  __syncthreads();
  const ScatterCtx C{P.res, P.deg, sh_thr, P.stamp, P.level_tag, P.next, P.seg_cap, K, P.col_cnt};
  const LevelAcc la{sh_dr, sh_np, sh_nn};
  const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t w = w0; w < P.total; w += nw) {
    int c = 0;
    while (w >= P.pre[c + 1]) ++c;
    if (!((P.col_live >> c) & 1ull)) continue;
    const uint64_t pos = w - P.pre[c];
    const uint32_t v = P.cur[(uint64_t)c * P.seg_cap + pos];
    pop_entry(C, P.off, P.nbr, P.x, P.alpha, P.src[c], P.limit, P.col_stop, P.col_resv, v, c, pos,
              P.pre[c + 1] - P.pre[c], la, heavy, heavy_cnt);
  }
  __syncthreads();
  for (int cc = threadIdx.x; cc < K; cc += blockDim.x) {
    if (sh_dr[cc] != 0.0) atomicAdd(P.col_dr + cc, sh_dr[cc]);
    if (sh_np[cc]) atomicAdd(P.col_np + cc, sh_np[cc]);
    if (sh_nn[cc]) atomicAdd(P.col_nn + cc, sh_nn[cc]);
  }
}

// The scatter of one HEAVY_CHUNK-edge chunk of a heavy entry by one block,
// four neighbour ids per thread loaded before the first atomic. Every lane of
// a chunk shares the entry's column, so appends group the whole warp.
constexpr uint32_t HEAVY_CHUNK = 1024;
__device__ __forceinline__ void heavy_chunk(const ScatterCtx& C, const uint32_t* nbr,
                                            const HeavyEntry& e, uint32_t first) {
  const uint32_t end = e.deg - first < HEAVY_CHUNK ? e.deg : first + HEAVY_CHUNK;
  const uint32_t q0 = first + threadIdx.x;
  uint32_t t[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t q = q0 + 256u * i;
    t[i] = q < end ? __ldg(nbr + e.begin + q) : 0xFFFFFFFFu;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) relax_scatter(C, t[i], (int)e.c, e.share, t[i] != 0xFFFFFFFFu, 0xffffffffu);
}

struct HeavyChunk {
  uint32_t h;      // heavy entry
  uint32_t first;  // first out-edge of the chunk, relative to the entry
};

// host-built chunk list (host-driven drain), a block per chunk
__global__ void __launch_bounds__(256) k_frontier_heavy_chunks(const __grid_constant__ FrontierParams P,
                                                               const HeavyEntry* heavy,
                                                               const HeavyChunk* chunks,
                                                               unsigned nchunks) {
  __shared__ double sh_thr[KMAX];
  for (int i = threadIdx.x; i < P.K; i += blockDim.x) sh_thr[i] = P.thr[i];
  __syncthreads();
  const ScatterCtx C{P.res, P.deg, sh_thr, P.stamp, P.level_tag, P.next, P.seg_cap, P.K, P.col_cnt};
  for (unsigned ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const HeavyChunk k = chunks[ch];
    heavy_chunk(C, P.nbr, heavy[k.h], k.first);
  }
}

// ---- persistent drain: all levels of a drain in one cooperative launch -----
// (drain_queue, push.cpp:34-59, level by level). The host-driven loop reads
// the level counters back after every level (several round trips per level);
// here every block derives the next level from the reduced counters itself:
//   entries phase (warp per entry, heavy entries queued) | grid barrier |
//   heavy phase (chunks of HEAVY_CHUNK edges, enumerated on the device from
//   a block-wide scan of the heavy entries' chunk counts) | grid barrier |
//   every block: r_sum -= alpha * pushed, queue sizes, stop tests -> next
//   level's live columns and segment prefix.
// Level counters are triple-buffered (slot = level % 3): slot level+1 is
// cleared during `level` by block 0, two barriers after its last reader.
struct DrainCtl {
  GridBarrier gbar;
  unsigned long long cnt[3][KMAX];   // appends per column (next queue size)
  unsigned long long np[3][KMAX];    // edge pushes
  unsigned long long nn[3][KMAX];    // node pushes
  unsigned long long resv[3][KMAX];  // out-degrees reserved by pops (queue-limit test)
  double dr[3][KMAX];                // alpha * pushed residue
  unsigned stop[3][KMAX];            // queue outgrew the limit
  unsigned heavy_cnt[3];
  unsigned levels_run;
  double out_rsum[KMAX];
  unsigned long long out_np[KMAX];
  unsigned out_levels[KMAX];
  unsigned long long out_live;
};

struct DrainParams {
  const uint64_t* off;
  const uint32_t* nbr;
  const uint32_t* deg;
  double* res;
  double* x;
  unsigned* stamp;
  uint32_t* seg[2];                  // level L reads seg[L & 1], appends to seg[(L + 1) & 1]
  uint64_t seg_cap;
  HeavyEntry* heavy;
  DrainCtl* ctl;
  unsigned long long limit;          // queue limit (~0: none)
  unsigned long long live0;          // columns draining
  double lam_stop;                   // r_sum stop (0: none)
  double alpha;
  unsigned tag0;                     // level L stamps tag0 + L + 1 (no wrap: host-checked)
  unsigned max_levels;
  int K;
  uint32_t src[KMAX];
  double thr[KMAX];
  double r_sum0[KMAX];
  unsigned long long q0[KMAX];       // first level's queue sizes
};

constexpr int DRAIN_NT = 256;
constexpr unsigned DRAIN_HSH = 2048;  // heavy entries whose chunk prefix is kept in shared memory

__global__ void __launch_bounds__(DRAIN_NT) k_drain(const __grid_constant__ DrainParams D) {
  __shared__ double s_rsum[KMAX], s_thr[KMAX];
  __shared__ uint32_t s_src[KMAX];
  __shared__ unsigned long long s_q[KMAX], s_pre[KMAX + 1], s_np[KMAX];
  __shared__ unsigned s_lv[KMAX];
  __shared__ unsigned long long s_live;
  __shared__ double sh_dr[KMAX];
  __shared__ unsigned long long sh_np[KMAX], sh_nn[KMAX];
  __shared__ unsigned s_hpre[DRAIN_HSH + 1];
  using Scan = cub::BlockScan<unsigned, DRAIN_NT>;
  __shared__ typename Scan::TempStorage scan_tmp;
  const int tid = threadIdx.x;
  const int K = D.K;
  DrainCtl* ctl = D.ctl;
  if (tid < KMAX) {
    s_rsum[tid] = D.r_sum0[tid];
    s_thr[tid] = D.thr[tid];
    s_src[tid] = D.src[tid];
    s_q[tid] = D.q0[tid];
    s_np[tid] = 0;
    s_lv[tid] = 0;
  }
  if (tid == 0) s_live = D.live0;
  __syncthreads();
  unsigned long long gen = 0;
  uint32_t level = 0;
  for (;; ++level) {
    const int slot = (int)(level % 3);
    if (tid == 0) {
      unsigned long long t = 0;
      for (int c = 0; c < K; ++c) {
        s_pre[c] = t;
        t += ((s_live >> c) & 1ull) ? s_q[c] : 0;
      }
      for (int c = K; c <= KMAX; ++c) s_pre[c] = t;
    }
    if (tid < KMAX) sh_dr[tid] = 0.0, sh_np[tid] = 0, sh_nn[tid] = 0;
    __syncthreads();
    const unsigned long long total = s_pre[K];
    if (total == 0 || level >= D.max_levels) break;  // identical in every block
    if (blockIdx.x == 0 && tid < KMAX) {
      const int ns = (int)((level + 1) % 3);
      ctl->cnt[ns][tid] = 0;
      ctl->np[ns][tid] = 0;
      ctl->nn[ns][tid] = 0;
      ctl->resv[ns][tid] = 0;
      ctl->dr[ns][tid] = 0.0;
      ctl->stop[ns][tid] = 0;
      if (tid == 0) ctl->heavy_cnt[ns] = 0;
    }
    const ScatterCtx C{D.res, D.deg, s_thr, D.stamp, D.tag0 + level + 1, D.seg[(level + 1) & 1],
                       D.seg_cap, K, ctl->cnt[slot]};
    const LevelAcc la{sh_dr, sh_np, sh_nn};
    const uint32_t* cur = D.seg[level & 1];
    {
      const uint64_t w0 = (blockIdx.x * (uint64_t)DRAIN_NT + tid) >> 5;
      const uint64_t nw = ((uint64_t)gridDim.x * DRAIN_NT) >> 5;
      for (uint64_t w = w0; w < total; w += nw) {
        int c = 0;
        while (w >= s_pre[c + 1]) ++c;
        const uint64_t pos = w - s_pre[c];
        const uint32_t v = cur[(uint64_t)c * D.seg_cap + pos];
        pop_entry(C, D.off, D.nbr, D.x, D.alpha, s_src[c], D.limit, ctl->stop[slot], ctl->resv[slot], v,
                  c, pos, s_pre[c + 1] - s_pre[c], la, D.heavy, &ctl->heavy_cnt[slot]);
      }
    }
    __syncthreads();
    if (tid < K) {
      if (sh_dr[tid] != 0.0) atomicAdd(&ctl->dr[slot][tid], sh_dr[tid]);
      if (sh_np[tid]) atomicAdd(&ctl->np[slot][tid], sh_np[tid]);
      if (sh_nn[tid]) atomicAdd(&ctl->nn[slot][tid], sh_nn[tid]);
    }
    grid_barrier2(&ctl->gbar, ++gen);
    const unsigned nh = __ldcg(&ctl->heavy_cnt[slot]);
    if (nh) {
      if (nh <= DRAIN_HSH) {
        // chunk prefix of the heavy entries (every block computes the same)
        unsigned run = 0;
        for (unsigned h0 = 0; h0 < nh; h0 += DRAIN_NT) {
          const unsigned h = h0 + tid;
          const unsigned nc = h < nh ? (__ldcg(&D.heavy[h].deg) + HEAVY_CHUNK - 1) / HEAVY_CHUNK : 0u;
          unsigned excl, agg;
          Scan(scan_tmp).ExclusiveSum(nc, excl, agg);
          if (h < nh) s_hpre[h] = run + excl;
          run += agg;
          __syncthreads();
        }
        if (tid == 0) s_hpre[nh] = run;
        __syncthreads();
        for (unsigned ch = blockIdx.x; ch < run; ch += gridDim.x) {
          unsigned lo = 0, hi = nh - 1;  // last h with s_hpre[h] <= ch
          while (lo < hi) {
            const unsigned mid = (lo + hi + 1) >> 1;
            if (s_hpre[mid] <= ch) lo = mid; else hi = mid - 1;
          }
          HeavyEntry e;
          e.begin = __ldcg(&D.heavy[lo].begin);
          e.deg = __ldcg(&D.heavy[lo].deg);
          e.c = __ldcg(&D.heavy[lo].c);
          e.share = __ldcg(&D.heavy[lo].share);
          heavy_chunk(C, D.nbr, e, (ch - s_hpre[lo]) * HEAVY_CHUNK);
        }
      } else {
        for (unsigned h = blockIdx.x; h < nh; h += gridDim.x) {
          HeavyEntry e;
          e.begin = __ldcg(&D.heavy[h].begin);
          e.deg = __ldcg(&D.heavy[h].deg);
          e.c = __ldcg(&D.heavy[h].c);
          e.share = __ldcg(&D.heavy[h].share);
          for (uint32_t f = 0; f < e.deg; f += HEAVY_CHUNK) heavy_chunk(C, D.nbr, e, f);
        }
      }
      grid_barrier2(&ctl->gbar, ++gen);
    }
    // the next level, identically in every block (drain_queue's loop test)
    if (tid < K && ((s_live >> tid) & 1ull)) {
      s_rsum[tid] -= __ldcg(&ctl->dr[slot][tid]);
      s_np[tid] += __ldcg(&ctl->np[slot][tid]);
      s_lv[tid] += 1;
      const unsigned long long q = __ldcg(&ctl->cnt[slot][tid]);
      s_q[tid] = q;
      const bool still = q > 0 && q <= D.limit && !(D.lam_stop > 0 && s_rsum[tid] <= D.lam_stop);
      if (__ldcg(&ctl->stop[slot][tid]) || !still) atomicAnd(&s_live, ~(1ull << tid));
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && tid < KMAX) {
    ctl->out_rsum[tid] = s_rsum[tid];
    ctl->out_np[tid] = s_np[tid];
    ctl->out_levels[tid] = s_lv[tid];
    if (tid == 0) {
      ctl->out_live = s_live;
      ctl->levels_run = level;
    }
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
