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
#include <cmath>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "internal.h"

namespace pprg {

constexpr int KMAX = 64;
constexpr int EMAX = 64;   // max epochs
#ifndef PPRG_NT
#define PPRG_NT 128
#endif
constexpr int NT = PPRG_NT;             // threads per block for the sweep kernels
constexpr int SWEEP_ELEMS = NT * 8;     // edges x columns per tile (8 per thread)

enum SweepMode : int { M_POWERPUSH = 0, M_POWITR = 1, M_SIMFWD = 2, M_FINAL = 3 };

struct SweepCtl {
  unsigned long long barrier;
  unsigned ticket[3];
  unsigned pad_;
  double pushed[3][KMAX];              // powerpush: pushed mass; powitr: sum of next
  unsigned long long npush[3][KMAX];   // edge pushes (sum deg_eff)
  unsigned long long nnode[3][KMAX];   // node pushes
  double dsum[3][KMAX];                // (1-alpha) * sum_dead x   (or next)
  unsigned long long et[3][KMAX];      // sum of out-degrees over pushed rows (E_t)
  unsigned long long alg_bytes;
  // final state (block 0)
  double out_rsum[KMAX];
  double out_D[KMAX];
  unsigned out_sweeps[KMAX];
  int out_done[KMAX];
  unsigned long long out_pushes[KMAX];
  unsigned total_sweeps;
};

struct ColInit {
  double r_sum;
  double D;
  int epoch;
  int done;
  uint32_t sweeps;
  uint64_t pushes;
};

struct SweepParams {
  uint64_t n, m;
  const uint64_t* in_off;      // compacted transpose rows (in-degree > 0)
  const uint32_t* crow;        // node id of each compacted row
  const uint32_t* cdeg;        // out-degree of each compacted row's node
  const double* cinv;          // 1 / effective out-degree of each compacted row's node
  const uint64_t* in_off_full; // transpose offsets per node
  const uint32_t* in_nbr;
  const uint32_t* deg;
  const double* inv_deg;
  const uint32_t* tile_lo;
  const uint2* desc;           // per tile: (first compact row, rows)
  uint64_t ntiles;
  uint32_t T;
  int k_live;  // real columns (<= K)
  int E;
  double alpha;
  double lambda;               // powitr termination
  double* x;                   // powerpush state / powitr reserve
  double* y[2];                // gather operand (powitr double-buffers)
  double* r[2];                // powitr residues (double-buffered)
  const double* push_res;      // finalize: push-form residues (columns without scan phase)
  double* carry_head;
  double* carry_tail;
  unsigned* split_cnt;
  const uint32_t* split_list;  // compact rows spanning tiles
  uint64_t n_split;
  double* split_acc;           // [2][ntiles+1][K] per-sweep partial sums of split rows
  SweepCtl* ctl;
  double* out_reserve;         // finalize outputs, query-major [c*n + u]
  double* out_residue;
  double* res_inter;           // finalize: explicit residues back into [u*K + c] (SpeedPPR)
  uint32_t max_sweeps;
  uint32_t src[KMAX];
  int final_pull[KMAX];        // finalize: 1 = residue from pull form
  double thr[EMAX];            // epoch r_max (lambda is per call, so shared by columns)
  double lam[EMAX];            // epoch lambda
  ColInit init[KMAX];
};

struct ColSh {
  double r_sum, D;
  int epoch, done;
  unsigned sweeps;
  unsigned long long pushes;
};

// Tile geometry. A tile is T = SWEEP_ELEMS/K consecutive in-edges; thread t
// owns column c = t % K and the SEG = 8 consecutive edges [8 (t/K), 8 (t/K) + 8)
// of the tile, so every thread does identical gather work. The gathered values
// of two tiles (current, next) live in shared memory in an owner-private
// layout vals[i*NT + t]; rows (the transpose's rows with in-degree > 0, so
// none is empty) are staged in chunks of RMAX, double-buffered.
template <int K>
struct Tile {
  static constexpr int T = SWEEP_ELEMS / K;
  static constexpr int SEG = SWEEP_ELEMS / NT;  // 8
  static constexpr int RMAX_ = (2 * NT) / K > 16 ? (2 * NT) / K : 16;
  static constexpr int RMAX = RMAX_ < NT - 1 ? RMAX_ : NT - 1;  // nr + 1 offsets fit one per thread
  static constexpr int RX = RMAX * K;
  // per staging buffer: sinv[RMAX] | sx[RX] | sr[RX] | sacc[RX] (f64) | soff[RMAX+1] (i32) | snode, sdeg [RMAX] (u32)
  static constexpr size_t buf_bytes = 8ull * (RMAX + 3 * RX) + 4ull * (RMAX + 1) + 8ull * RMAX;
  static constexpr size_t buf_stride = (buf_bytes + 15) / 16 * 16;
  static constexpr size_t vals_bytes = 8ull * SWEEP_ELEMS;
  static constexpr size_t bytes = 2 * vals_bytes + 2 * buf_stride;
};

struct Acc {  // per-thread sweep counters for the thread's column
  double push = 0, d = 0;
  unsigned long long np = 0, nn = 0, et = 0;
};

struct BlockAcc {  // shared, per column
  double* push;
  double* d;
  unsigned long long* np;
  unsigned long long* nn;
  unsigned long long* et;
};

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 8 : 0;  // src-size 0 zero-fills
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(sz)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// The per-(row, column) decision: push form of push.cpp:182-193 in pull
// representation, the PowItr update of push.cpp:90-99, or the final explicit
// residue. `acc` is the sum over in-neighbours v of y_v.
template <int K, int MODE>
__device__ __forceinline__ void decide(const SweepParams& P, const ColSh* cs, const double* thr_cur,
                                       uint32_t u, int c, double acc, double xo, double rc,
                                       uint32_t dg, double inv, const double* yg, double* rnxt,
                                       double* ynxt, Acc& a) {
  const uint64_t ix = (uint64_t)u * K + c;
  const bool is_src = u == P.src[c];
  const double alpha = P.alpha, oma = 1.0 - P.alpha;
  if constexpr (MODE == M_POWERPUSH) {
    if (cs[c].done) return;
    const double inflow = acc + (is_src ? 1.0 + cs[c].D : 0.0);
    const double r = inflow - xo;
    if (r > (dg ? (double)dg : 1.0) * thr_cur[c]) {
      P.x[ix] = inflow;
      if (dg) P.y[0][ix] = oma * inflow * inv;
      a.push += r;
      a.np += dg ? dg : 1;
      a.nn += 1;
      a.et += dg;
      xo = inflow;
    }
    if (!dg) a.d += oma * xo;
  } else if constexpr (MODE == M_POWITR || MODE == M_SIMFWD) {
    if (cs[c].done) {
      rnxt[ix] = rc;
      ynxt[ix] = __ldcg(yg + ix);
      return;
    }
    const double nxt = acc + (is_src ? cs[c].D : 0.0);
    P.x[ix] = xo + alpha * rc;  // reserve += alpha * r
    rnxt[ix] = nxt;
    ynxt[ix] = oma * nxt * inv;
    a.push += nxt;  // sum of next = the exact r_sum (push.cpp:101-103)
    if (MODE == M_POWITR || rc != 0.0) {
      a.np += dg ? dg : 1;
      a.nn += 1;
      a.et += dg;
    }
    if (!dg) a.d += oma * nxt;
  } else {  // M_FINAL
    double res;
    if (P.final_pull[c]) {
      const double inflow = acc + (is_src ? 1.0 + cs[c].D : 0.0);
      res = inflow - xo;
      if (res < 0.0) res = 0.0;  // rounding of the implicit form only
    } else {
      res = P.push_res[ix];
    }
    if (P.res_inter) P.res_inter[ix] = res;
    if (c < P.k_live) {
      if (P.out_reserve) P.out_reserve[(uint64_t)c * P.n + u] = alpha * xo;
      if (P.out_residue) P.out_residue[(uint64_t)c * P.n + u] = res;
    }
    a.push += res;
  }
}

// A row straddling tiles adds this tile's per-column partial into the sweep's
// accumulator (fire-and-forget RED, keyed by the row's first tile); the row is
// decided after the grid barrier by split_decide.
template <int K>
__device__ __noinline__ void post_split(const SweepParams& P, uint32_t cr, uint32_t r,
                                        const double* sacc, uint32_t parity) {
  constexpr int T = Tile<K>::T;
  const uint64_t ft = __ldg(P.in_off + cr) / T;
  double* acc = P.split_acc + ((uint64_t)parity * (P.ntiles + 1) + ft) * K;
  for (int cc = 0; cc < K; ++cc) atomicAdd(acc + cc, sacc[r * K + cc]);
}

// Decide every split row from the accumulated partials of sweep `parity`
// (grid-stride; thread column = tid % K as everywhere), and clear them.
template <int K, int MODE>
__device__ __forceinline__ void split_decide(const SweepParams& P, uint32_t parity, const ColSh* cs,
                                             const double* thr_cur, const double* yg,
                                             const double* rcur, double* rnxt, double* ynxt,
                                             Acc& a) {
  constexpr int T = Tile<K>::T;
  const uint64_t total = P.n_split * K;
  for (uint64_t idx = blockIdx.x * (uint64_t)NT + threadIdx.x; idx < total;
       idx += (uint64_t)gridDim.x * NT) {
    const uint32_t cr = P.split_list[idx / K];
    const int c = (int)(idx % K);
    const uint64_t ft = __ldg(P.in_off + cr) / T;
    double* slot = P.split_acc + ((uint64_t)parity * (P.ntiles + 1) + ft) * K + c;
    const double acc = __ldcg(slot);
    *slot = 0.0;
    const uint32_t u = __ldg(P.crow + cr);
    const uint64_t ix = (uint64_t)u * K + c;
    decide<K, MODE>(P, cs, thr_cur, u, c, acc, __ldcg(P.x + ix),
                    (MODE == M_POWITR || MODE == M_SIMFWD) ? __ldcg(rcur + ix) : 0.0,
                    __ldg(P.cdeg + cr), __ldg(P.cinv + cr), yg, rnxt, ynxt, a);
  }
}

// The in-neighbour ids of my 8 edges of tile j (one 32-byte vector load).
template <int K>
__device__ __forceinline__ void load_ids(const SweepParams& P, uint64_t j, uint32_t (&id)[8]) {
  constexpr int T = Tile<K>::T, SEG = Tile<K>::SEG;
  const int32_t seg0 = (threadIdx.x / K) * SEG;
  const uint64_t base = j * (uint64_t)T;
  const int32_t ne = base < P.m ? (int32_t)(P.m - base < (uint64_t)T ? P.m - base : (uint64_t)T) : 0;
  if (seg0 + SEG <= ne) {
    const uint4* p4 = reinterpret_cast<const uint4*>(P.in_nbr + base + seg0);
    const uint4 q0 = __ldg(p4), q1 = __ldg(p4 + 1);
    id[0] = q0.x; id[1] = q0.y; id[2] = q0.z; id[3] = q0.w;
    id[4] = q1.x; id[5] = q1.y; id[6] = q1.z; id[7] = q1.w;
  } else {
#pragma unroll
    for (int i = 0; i < SEG; ++i) id[i] = seg0 + i < ne ? __ldg(P.in_nbr + base + seg0 + i) : ~0u;
  }
}

// Issue my 8 gathers of y for tile j as cp.async into my private slots.
template <int K>
__device__ __forceinline__ void issue_gathers(const double* yg, const uint32_t (&id)[8],
                                              double* vals) {
  const int c = threadIdx.x % K;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const bool ok = id[i] != ~0u;
    cp_async8(vals + i * NT + threadIdx.x, yg + (ok ? (uint64_t)id[i] * K + c : 0), ok);
  }
}

// Row data of one tile's first chunk, prefetched into registers one tile ahead
// (thread t holds row t; thread nr holds only the end offset).
struct RowPre {
  uint64_t off = 0;
  uint32_t node = 0, deg = 0;
  double inv = 0.0;
};

template <int K>
__device__ __forceinline__ void load_rows(const SweepParams& P, uint2 d, RowPre& rp) {
  constexpr int RMAX = Tile<K>::RMAX;
  const uint32_t nr = d.y < (uint32_t)RMAX ? d.y : RMAX;
  const uint32_t t = threadIdx.x;
  if (t <= nr) rp.off = __ldg(P.in_off + d.x + t);
  if (t < nr) {
    rp.node = __ldg(P.crow + d.x + t);
    rp.deg = __ldg(P.cdeg + d.x + t);
    rp.inv = __ldg(P.cinv + d.x + t);
  }
}

// Stage rows [cr0, cr0 + nr) of tile `base` into a staging buffer.
template <int K>
__device__ __forceinline__ void stage_rows_from(const RowPre& rp, uint32_t nr, uint64_t base,
                                                char* buf) {
  using TC = Tile<K>;
  constexpr int T = TC::T, RMAX = TC::RMAX, RX = TC::RX;
  double* sinv = reinterpret_cast<double*>(buf);
  double* sacc = sinv + RMAX + 2 * RX;
  int32_t* soff = reinterpret_cast<int32_t*>(sacc + RX);
  uint32_t* snode = reinterpret_cast<uint32_t*>(soff + RMAX + 1);
  uint32_t* sdeg = snode + RMAX;
  const uint32_t t = threadIdx.x;
  if (t <= nr) {
    const int64_t d = (int64_t)rp.off - (int64_t)base;
    soff[t] = d < 0 ? -1 : (d > T ? T + 1 : (int32_t)d);
  }
  if (t < nr) {
    snode[t] = rp.node;
    sdeg[t] = rp.deg;
    sinv[t] = rp.inv;
#pragma unroll
    for (int cc = 0; cc < K; ++cc) sacc[t * K + cc] = 0.0;
  }
}

template <int K>
__device__ __forceinline__ void stage_rows_sync(const SweepParams& P, uint32_t cr0, uint32_t nr,
                                                uint64_t base, char* buf) {
  for (uint32_t t0 = 0; t0 <= nr; t0 += NT) {
    RowPre rp;
    const uint32_t t = t0 + threadIdx.x;
    if (t <= nr) rp.off = __ldg(P.in_off + cr0 + t);
    if (t < nr) {
      rp.node = __ldg(P.crow + cr0 + t);
      rp.deg = __ldg(P.cdeg + cr0 + t);
      rp.inv = __ldg(P.cinv + cr0 + t);
    }
    // stage_rows_from uses threadIdx.x as the row; emulate the offset t0
    using TC = Tile<K>;
    constexpr int T = TC::T, RMAX = TC::RMAX, RX = TC::RX;
    double* sinv = reinterpret_cast<double*>(buf);
    double* sacc = sinv + RMAX + 2 * RX;
    int32_t* soff = reinterpret_cast<int32_t*>(sacc + RX);
    uint32_t* snode = reinterpret_cast<uint32_t*>(soff + RMAX + 1);
    uint32_t* sdeg = snode + RMAX;
    if (t <= nr) {
      const int64_t d = (int64_t)rp.off - (int64_t)base;
      soff[t] = d < 0 ? -1 : (d > T ? T + 1 : (int32_t)d);
    }
    if (t < nr) {
      snode[t] = rp.node;
      sdeg[t] = rp.deg;
      sinv[t] = rp.inv;
      for (int cc = 0; cc < K; ++cc) sacc[t * K + cc] = 0.0;
    }
  }
}

// Reduce + decide one staged chunk (rows [cr0, cr0+nr)) of tile j whose
// gathered values are in `vals`. Called after the staging barrier.
template <int K, int MODE>
__device__ __forceinline__ void chunk_compute(const SweepParams& P, uint64_t j, const double* vals,
                                              char* smem_buf, uint32_t cr0, uint32_t nr,
                                              bool first_chunk, bool last_chunk, uint32_t parity,
                                              const ColSh* cs,
                                              const double* thr_cur, const double* yg,
                                              const double* rcur, double* rnxt, double* ynxt,
                                              Acc& a, const BlockAcc& ba) {
  using TC = Tile<K>;
  constexpr int T = TC::T, SEG = TC::SEG, RMAX = TC::RMAX, RX = TC::RX;
  double* sinv = reinterpret_cast<double*>(smem_buf);
  double* sr = sinv + RMAX + RX;
  double* sacc = sr + RX;
  int32_t* soff = reinterpret_cast<int32_t*>(sacc + RX);
  uint32_t* snode = reinterpret_cast<uint32_t*>(soff + RMAX + 1);
  uint32_t* sdeg = snode + RMAX;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int c = tid % K;
  const int32_t seg0 = (tid / K) * SEG;
  const uint64_t base = j * (uint64_t)T;
  const int32_t ne = base < P.m ? (int32_t)(P.m - base < (uint64_t)T ? P.m - base : (uint64_t)T) : 0;

  // prefetch the state of my first decision (lands during the reduction)
  double xo0 = 0.0, rc0 = 0.0;
  if ((uint32_t)tid < nr * K) {
    const uint64_t ix = (uint64_t)snode[tid / K] * K + c;
    xo0 = __ldcg(P.x + ix);
    if constexpr (MODE == M_POWITR || MODE == M_SIMFWD) rc0 = __ldcg(rcur + ix);
  }
  if (first_chunk) cp_async_wait<1>();  // my gathers of this tile have landed

  // ---- segmented reduction over my 8 edges ---------------------------------
  {
    constexpr uint32_t SENT = 0xFFFFFFFFu;
    double hp = 0.0, tp = 0.0;
    uint32_t f = SENT, l = SENT;
    bool started = false, cont = false, have = false;
    if (nr > 0) {
      const int32_t cbeg = soff[0] < 0 ? 0 : soff[0];
      int32_t e_hi = seg0 + SEG;
      if (e_hi > ne) e_hi = ne;
      if (e_hi > soff[nr]) e_hi = soff[nr];
      const int32_t e_lo = seg0 > cbeg ? seg0 : cbeg;
      if (e_lo < e_hi) {
        have = true;
        uint32_t lo_r = 0, hi_r = nr;  // last row r with soff[r] <= e_lo
        while (lo_r + 1 < hi_r) {
          const uint32_t mid = (lo_r + hi_r) >> 1;
          if (soff[mid] <= e_lo) lo_r = mid; else hi_r = mid;
        }
        uint32_t r = lo_r;
        f = r;
        started = soff[r] < e_lo;
        int32_t rend = soff[r + 1];
        double part = 0.0;
#pragma unroll
        for (int i = 0; i < SEG; ++i) {
          const int32_t e = seg0 + i;
          if (e >= e_lo && e < e_hi) {
            if (e >= rend) {  // row r ended at e - 1 (rows are never empty)
              if (r == f) hp = part;
              else sacc[r * K + c] = part;  // started and ended inside the segment
              part = 0.0;
              ++r;
              rend = soff[r + 1];
            }
            part += vals[i * NT + tid];
          }
        }
        l = r;
        cont = rend > e_hi;
        if (l == f) hp = part; else tp = part;
        if (l != f && !cont) sacc[l * K + c] = tp;
        if (!started && (l != f || !cont)) sacc[f * K + c] = hp;
      }
    }
    const double carry = cont ? (l == f ? hp : tp) : 0.0;
    const uint32_t key = have ? l : SENT;
    double S = carry;
    double carry_in = 0.0;
    uint32_t f_next = SENT;  // first row of the next segment of my column
    if constexpr (K < 32) {
#pragma unroll
      for (int d = K; d < 32; d <<= 1) {
        const double Sd = __shfl_up_sync(0xffffffffu, S, d);
        const uint32_t kd = __shfl_up_sync(0xffffffffu, key, d);
        if (lane >= d && kd == key) S += Sd;
      }
      const double Sp = __shfl_up_sync(0xffffffffu, S, K);
      const uint32_t kp = __shfl_up_sync(0xffffffffu, key, K);
      if (lane >= K && kp == f) carry_in = Sp;
      f_next = __shfl_down_sync(0xffffffffu, f, K);
    }
    const int first_lane = K < 32 ? lane % K : lane;
    const uint32_t f_first = __shfl_sync(0xffffffffu, f, first_lane);
    const bool st_first = __shfl_sync(0xffffffffu, started, first_lane);
    if (have && started && !(l == f && cont)) {  // I finish row f
      const double val = hp + carry_in;
      if (f == f_first && st_first) atomicAdd(&sacc[f * K + c], val);  // began in an earlier warp
      else sacc[f * K + c] = val;
    }
    if (have && cont && (lane + K >= 32 || f_next != key))
      atomicAdd(&sacc[l * K + c], S);  // row l continues past this warp / chunk
  }
  __syncthreads();

  // ---- rows straddling the tile: post partials --------------------------
  const uint32_t rl = nr ? nr - 1 : 0;
  const bool first_split = first_chunk && nr > 0 && (soff[0] < 0 || soff[1] > T);
  const bool last_split = last_chunk && nr > 0 && !(first_chunk && rl == 0) && soff[rl + 1] > T;
  if (tid == 0 && first_split) post_split<K>(P, cr0, 0, sacc, parity);
  if (tid == 32 && last_split) post_split<K>(P, cr0 + rl, rl, sacc, parity);
  // ---- decisions --------------------------------------------------------
  for (uint32_t fi = tid; fi < nr * K; fi += NT) {
    const uint32_t r = fi / K;
    if (soff[r] < 0 || soff[r + 1] > T) continue;  // straddles the tile: split_row
    double xo = xo0, rc = rc0;
    if (fi != (uint32_t)tid) {
      const uint64_t ix = (uint64_t)snode[r] * K + c;
      xo = __ldcg(P.x + ix);
      if constexpr (MODE == M_POWITR || MODE == M_SIMFWD) rc = __ldcg(rcur + ix);
    }
    decide<K, MODE>(P, cs, thr_cur, snode[r], c, sacc[fi], xo, rc, sdeg[r], sinv[r], yg, rnxt,
                    ynxt, a);
  }
}

// Sources with in-degree 0 are not rows of the compacted transpose; their
// only inflow is the unit start mass plus the dead-end mass D (block 0).
template <int K, int MODE>
__device__ __forceinline__ void source_rows(const SweepParams& P, const ColSh* cs,
                                            const double* thr_cur, const double* yg,
                                            const double* rcur, double* rnxt, double* ynxt,
                                            Acc& a) {
  const int tid = threadIdx.x;
  if (blockIdx.x != 0 || tid >= K) return;
  const uint32_t u = P.src[tid];
  if (__ldg(P.in_off_full + u + 1) != __ldg(P.in_off_full + u)) return;
  const uint64_t ix = (uint64_t)u * K + tid;
  decide<K, MODE>(P, cs, thr_cur, u, tid, 0.0, __ldcg(P.x + ix),
                  (MODE == M_POWITR || MODE == M_SIMFWD) ? __ldcg(rcur + ix) : 0.0, __ldg(P.deg + u),
                  __ldg(P.inv_deg + u), yg, rnxt, ynxt, a);
}

template <int K, int MODE>
#ifndef PPRG_MINB
#define PPRG_MINB 6
#endif
__global__ void __launch_bounds__(NT, PPRG_MINB) k_sweeps(const __grid_constant__ SweepParams P) {
  using TC = Tile<K>;
  extern __shared__ __align__(16) char smem_dyn[];
  __shared__ ColSh cs[K];
  __shared__ double thr_cur[K];
  __shared__ double sh_push[K], sh_d[K];
  __shared__ unsigned long long sh_np[K], sh_nn[K], sh_et[K];
  __shared__ unsigned long long sh_tile[3];
  __shared__ int sh_any;
  const int tid = threadIdx.x;
  SweepCtl* ctl = P.ctl;
  if (tid < K) {
    cs[tid].r_sum = P.init[tid].r_sum;
    cs[tid].D = P.init[tid].D;
    cs[tid].epoch = P.init[tid].epoch;
    cs[tid].done = P.init[tid].done;
    cs[tid].sweeps = P.init[tid].sweeps;
    cs[tid].pushes = P.init[tid].pushes;
  }
  __syncthreads();
  const BlockAcc ba{sh_push, sh_d, sh_np, sh_nn, sh_et};
  unsigned long long gen = 0;
  const int c = tid % K;
  for (uint32_t sweep = 0;; ++sweep) {
    const int buf = sweep % 3;
    if (tid == 0) {
      int any = 0;
      for (int cc = 0; cc < K; ++cc) any |= !cs[cc].done;
      sh_any = any && (MODE == M_FINAL ? sweep == 0 : sweep < P.max_sweeps);
      if (sh_any) {
        sh_tile[0] = atomicAdd(&ctl->ticket[buf], 1u);
        sh_tile[1] = atomicAdd(&ctl->ticket[buf], 1u);
      }
    }
    if (tid < K) {
      thr_cur[tid] = (MODE == M_POWERPUSH && !cs[tid].done) ? P.thr[cs[tid].epoch] : 0.0;
      sh_push[tid] = 0.0;
      sh_d[tid] = 0.0;
      sh_np[tid] = 0;
      sh_nn[tid] = 0;
      sh_et[tid] = 0;
    }
    __syncthreads();
    if (!sh_any) break;
    if (blockIdx.x == 0 && tid == 0 && MODE != M_FINAL) {
      const int nb = (sweep + 1) % 3;  // last read two barriers ago; safe to clear
      ctl->ticket[nb] = 0;
      for (int cc = 0; cc < K; ++cc) {
        ctl->pushed[nb][cc] = 0;
        ctl->npush[nb][cc] = 0;
        ctl->nnode[nb][cc] = 0;
        ctl->dsum[nb][cc] = 0;
        ctl->et[nb][cc] = 0;
      }
    }
    const double* yg = P.y[MODE == M_POWERPUSH || MODE == M_FINAL ? 0 : (sweep & 1)];
    const double* rcur = P.r[sweep & 1];
    double* rnxt = P.r[(sweep + 1) & 1];
    double* ynxt = P.y[(sweep + 1) & 1];
    Acc a;
    if (MODE == M_POWERPUSH && sweep > 0)  // rows straddling tiles, from the last sweep
      split_decide<K, MODE>(P, (sweep - 1) & 1, cs, thr_cur, yg, rcur, rnxt, ynxt, a);
    // Software pipeline. Tickets are fetched two tiles ahead into a 3-slot
    // ring; the ids of tile it+2 are loaded during tile it; the gathers of
    // tile it+1 are issued (cp.async, owner-private slots) before tile it is
    // reduced. Row staging is double-buffered, so consecutive tiles need no
    // block barrier between them.
    uint32_t ids[8];
    RowPre rp;  // rows (first chunk) of the tile about to be processed
    uint2 dcur = make_uint2(0, 0), dnext = make_uint2(0, 0);
    double* vals0 = reinterpret_cast<double*>(smem_dyn);
    double* vals1 = vals0 + SWEEP_ELEMS;
    char* stage0 = smem_dyn + 2 * TC::vals_bytes;
    {
      const unsigned long long j0 = sh_tile[0], j1 = sh_tile[1];
      if (j0 < P.ntiles) {
        dcur = P.desc[j0];
        load_rows<K>(P, dcur, rp);
        load_ids<K>(P, j0, ids);
        issue_gathers<K>(yg, ids, vals0);
      }
      cp_async_commit();
      if (j1 < P.ntiles) {
        dnext = P.desc[j1];
        load_ids<K>(P, j1, ids);
      }
    }
    for (uint32_t it = 0;; ++it) {
      const unsigned long long j = sh_tile[it % 3];
      if (j >= P.ntiles) break;
      const unsigned long long jn = sh_tile[(it + 1) % 3];
      if (jn < P.ntiles) issue_gathers<K>(yg, ids, (it & 1) ? vals0 : vals1);
      cp_async_commit();
      if (tid == 0) sh_tile[(it + 2) % 3] = atomicAdd(&ctl->ticket[buf], 1u);
      char* sbuf = stage0 + (it & 1) * TC::buf_stride;
      const uint64_t base = j * (uint64_t)TC::T;
      const uint2 dthis = dcur;
      const uint32_t nr0 = dthis.y < (uint32_t)TC::RMAX ? dthis.y : TC::RMAX;
      stage_rows_from<K>(rp, nr0, base, sbuf);
      __syncthreads();
      // prefetch: rows of tile it+1, descriptor and ids of tile it+2
      const unsigned long long j2 = sh_tile[(it + 2) % 3];
      if (jn < P.ntiles) load_rows<K>(P, dnext, rp);
      dcur = dnext;
      if (j2 < P.ntiles) {
        dnext = P.desc[j2];
        load_ids<K>(P, j2, ids);
      }
      const double* vals = (it & 1) ? vals1 : vals0;
      chunk_compute<K, MODE>(P, j, vals, sbuf, dthis.x, nr0, true, dthis.y <= (uint32_t)TC::RMAX,
                             sweep & 1, cs, thr_cur, yg, rcur, rnxt, ynxt, a, ba);
      for (uint32_t row0 = TC::RMAX; row0 < dthis.y; row0 += TC::RMAX) {  // rare: many rows
        __syncthreads();
        const uint32_t nr = dthis.y - row0 < (uint32_t)TC::RMAX ? dthis.y - row0 : TC::RMAX;
        stage_rows_sync<K>(P, dthis.x + row0, nr, base, sbuf);
        __syncthreads();
        chunk_compute<K, MODE>(P, j, vals, sbuf, dthis.x + row0, nr, false,
                               row0 + nr >= dthis.y, sweep & 1, cs, thr_cur, yg, rcur, rnxt, ynxt,
                               a, ba);
      }
    }
    cp_async_wait<0>();
    source_rows<K, MODE>(P, cs, thr_cur, yg, rcur, rnxt, ynxt, a);
    if (MODE != M_POWERPUSH) {  // synchronous modes finish their split rows this sweep
      grid_barrier(&ctl->barrier, (++gen) * gridDim.x);
      split_decide<K, MODE>(P, sweep & 1, cs, thr_cur, yg, rcur, rnxt, ynxt, a);
    }
    // block-level flush of this sweep's accumulators: reduce over the lanes of
    // the same column first (shuffles), then one shared atomic per warp/column
    {
      const int lane = tid & 31;
#pragma unroll
      for (int o = 16; o >= K && o > 0; o >>= 1) {
        a.push += __shfl_xor_sync(0xffffffffu, a.push, o);
        a.d += __shfl_xor_sync(0xffffffffu, a.d, o);
        a.np += __shfl_xor_sync(0xffffffffu, a.np, o);
        a.nn += __shfl_xor_sync(0xffffffffu, a.nn, o);
        a.et += __shfl_xor_sync(0xffffffffu, a.et, o);
      }
      if (lane < (K < 32 ? K : 32)) {
        if (a.push != 0.0) atomicAdd(&sh_push[c], a.push);
        if (a.d != 0.0) atomicAdd(&sh_d[c], a.d);
        if (a.np) atomicAdd(&sh_np[c], a.np);
        if (a.nn) atomicAdd(&sh_nn[c], a.nn);
        if (a.et) atomicAdd(&sh_et[c], a.et);
      }
    }
    __syncthreads();
    if (tid < K) {
      if (sh_push[tid] != 0.0) atomicAdd(&ctl->pushed[buf][tid], sh_push[tid]);
      if (sh_d[tid] != 0.0) atomicAdd(&ctl->dsum[buf][tid], sh_d[tid]);
      if (sh_np[tid]) atomicAdd(&ctl->npush[buf][tid], sh_np[tid]);
      if (sh_nn[tid]) atomicAdd(&ctl->nnode[buf][tid], sh_nn[tid]);
      if (sh_et[tid]) atomicAdd(&ctl->et[buf][tid], sh_et[tid]);
    }
    if (MODE == M_FINAL) {
      __syncthreads();
      break;
    }
    grid_barrier(&ctl->barrier, (++gen) * gridDim.x);
    // every block derives the identical next state from the reduced buffers
    if (tid < K) {
      const int cc = tid;
      if (!cs[cc].done) {
        const double pushed = __ldcg(&ctl->pushed[buf][cc]);
        const unsigned long long np = __ldcg(&ctl->npush[buf][cc]);
        cs[cc].sweeps += 1;
        cs[cc].pushes += np;
        cs[cc].D = __ldcg(&ctl->dsum[buf][cc]);
        if (MODE == M_POWERPUSH) {
          cs[cc].r_sum -= P.alpha * pushed;
          if (np == 0) cs[cc].epoch += 1;  // fixpoint: nothing active at this threshold
          while (cs[cc].epoch < P.E && !(cs[cc].r_sum > P.lam[cs[cc].epoch])) cs[cc].epoch += 1;
          if (cs[cc].epoch >= P.E) cs[cc].done = 1;
        } else {
          cs[cc].r_sum = pushed;
          if (!(cs[cc].r_sum > P.lambda)) cs[cc].done = 1;
        }
      }
    }
    if (blockIdx.x == 0 && tid == 0) {
      // B = 8(n+1) + 8 k n + 4 E_t + 24 P_t over the live columns;
      // E_t (rows pushed in any column) is taken as the largest per-column sum.
      unsigned long long live = 0, pt = 0, et = 0;
      for (int cc = 0; cc < P.k_live; ++cc) {
        pt += __ldcg(&ctl->nnode[buf][cc]);
        const unsigned long long e = __ldcg(&ctl->et[buf][cc]);
        et = e > et ? e : et;
        live += 1;
      }
      if (MODE != M_POWERPUSH) et = P.m;
      ctl->alg_bytes += 8ull * (P.n + 1) + 8ull * live * P.n + 4ull * et +
                        (MODE == M_POWERPUSH ? 24ull * pt : 24ull * live * P.n);
      ctl->total_sweeps = sweep + 1;
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && tid < K) {
    ctl->out_rsum[tid] = cs[tid].r_sum;
    ctl->out_D[tid] = cs[tid].D;
    ctl->out_sweeps[tid] = cs[tid].sweeps;
    ctl->out_done[tid] = cs[tid].done;
    ctl->out_pushes[tid] = cs[tid].pushes;
  }
}

// ---- local phase / refine / FIFO: frontier levels in push form ------------
// Entry = linear index i = u*K + c. One warp per entry: claim r with
// atomicExch (the FIFO pop, push.cpp:38-41), x += r, scatter (1-a) r / deg_eff
// with fp64 RED, and append newly active (t, c) once per level (stamp).
struct FrontierParams {
  const uint64_t* off;
  const uint32_t* nbr;
  const uint32_t* deg;
  double* res;
  double* x;
  unsigned* stamp;
  const uint64_t* cur;
  uint64_t ncur;
  uint64_t* next;
  unsigned long long* next_cnt;
  unsigned long long* col_cnt;   // [K] entries appended per column
  double* col_dr;                // [K] alpha * sum r pushed
  unsigned long long* col_np;    // [K] edge pushes
  unsigned long long* col_nn;    // [K] node pushes
  unsigned long long* col_proc;  // [K] entries of live columns processed
  unsigned long long col_live;   // bit c set: column c still in this phase
  unsigned level_tag;
  int K;
  double alpha;
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

// Append (t, c) to the next frontier once per level when it becomes active
// (drain_queue's enqueue test, push.cpp:49-53). Warp-aggregated append.
__device__ __forceinline__ void maybe_append(const FrontierParams& P, bool app, uint64_t ti, int c,
                                             unsigned mask) {
  const unsigned bal = __ballot_sync(mask, app);
  if (app) {
    const int lane = threadIdx.x & 31, leader = __ffs(bal) - 1;
    unsigned long long basepos = 0;
    if (lane == leader) basepos = atomicAdd(P.next_cnt, (unsigned long long)__popc(bal));
    basepos = __shfl_sync(bal, basepos, leader);
    P.next[basepos + __popc(bal & ((1u << lane) - 1u))] = ti;
    atomicAdd(P.col_cnt + c, 1ull);
  }
}

// One warp per frontier entry (v, c): claim r (the FIFO pop, push.cpp:38-41),
// x += r, then scatter (1-a) r / deg_eff to the effective out-neighbours with
// fp64 atomics, 4 independent atomics per lane in flight. Entries with more
// than HEAVY_DEG out-edges are queued for k_frontier_heavy instead, so a hub
// never serialises one warp.
__global__ void __launch_bounds__(256) k_frontier(const __grid_constant__ FrontierParams P,
                                                  HeavyEntry* heavy, unsigned* heavy_cnt) {
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int K = P.K;
  for (uint64_t w = w0; w < P.ncur; w += nw) {
    const uint64_t i = P.cur[w];
    const uint32_t v = (uint32_t)(i / K);
    const int c = (int)(i % K);
    if (!((P.col_live >> c) & 1ull)) continue;
    double r = 0.0;
    if (lane == 0) {
      atomicAdd(P.col_proc + c, 1ull);
      r = __longlong_as_double((long long)atomicExch((unsigned long long*)(P.res + i), 0ull));
    }
    r = __shfl_sync(0xffffffffu, r, 0);
    if (!(r > 0.0)) continue;
    const uint32_t d = P.deg[v];
    const uint64_t de = d ? d : 1;
    const double share = (1.0 - P.alpha) * r / (double)de;
    const uint64_t b = P.off[v];
    if (lane == 0) {
      P.x[i] += r;
      atomicAdd(P.col_dr + c, P.alpha * r);
      atomicAdd(P.col_np + c, (unsigned long long)de);
      atomicAdd(P.col_nn + c, 1ull);
      if (de > HEAVY_DEG) heavy[atomicAdd(heavy_cnt, 1u)] = HeavyEntry{b, d, (uint32_t)c, share};
    }
    if (de > HEAVY_DEG) continue;
    for (uint64_t q0 = 0; q0 < de; q0 += 128) {
      uint64_t ti[4];
      double nv[4];
      uint32_t td[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t q = q0 + lane + 32 * k;
        ti[k] = q < de ? (uint64_t)(d ? __ldg(P.nbr + b + q) : P.src[c]) * K + c : ~0ull;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (ti[k] != ~0ull) {
          nv[k] = atomicAdd(P.res + ti[k], share) + share;
          td[k] = __ldg(P.deg + ti[k] / K);
        }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        bool app = false;
        if (ti[k] != ~0ull && nv[k] > (double)(td[k] ? td[k] : 1) * P.thr[c])
          app = atomicExch(P.stamp + ti[k], P.level_tag) != P.level_tag;
        maybe_append(P, app, ti[k], c, 0xffffffffu);
      }
    }
  }
}

// The scatter of heavy entries, one thread per out-edge over all of them.
__global__ void __launch_bounds__(256) k_frontier_heavy(const __grid_constant__ FrontierParams P,
                                                        const HeavyEntry* heavy,
                                                        const unsigned long long* prefix,
                                                        unsigned nheavy, unsigned long long total) {
  const int K = P.K;
  for (unsigned long long e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
       e - threadIdx.x < total; e += (uint64_t)gridDim.x * blockDim.x) {
    const bool ok = e < total;
    uint64_t ti = 0;
    int c = 0;
    bool app = false;
    if (ok) {
      unsigned lo = 0, hi = nheavy;  // last h with prefix[h] <= e
      while (lo + 1 < hi) {
        const unsigned mid = (lo + hi) >> 1;
        if (prefix[mid] <= e) lo = mid; else hi = mid;
      }
      const HeavyEntry h = heavy[lo];
      c = (int)h.c;
      ti = (uint64_t)__ldg(P.nbr + h.begin + (e - prefix[lo])) * K + c;
      const double nv = atomicAdd(P.res + ti, h.share) + h.share;
      const uint32_t td = __ldg(P.deg + ti / K);
      if (nv > (double)(td ? td : 1) * P.thr[c])
        app = atomicExch(P.stamp + ti, P.level_tag) != P.level_tag;
    }
    maybe_append(P, app, ti, c, 0xffffffffu);
  }
}

// Enqueue every active (u, c) in id order (refine, push.cpp:212-218).
__global__ void k_scan_active(const double* res, const uint32_t* deg, uint64_t n, int K,
                              const double* thr, unsigned long long col_live, unsigned* stamp,
                              unsigned tag, uint64_t* out, unsigned long long* cnt,
                              unsigned long long* col_cnt) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n * K;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % K);
    const uint32_t d = deg[i / K];
    const bool a = ((col_live >> c) & 1ull) && res[i] > (double)(d ? d : 1) * thr[c];
    const unsigned bal = __ballot_sync(0xffffffffu, a);
    if (a) {
      stamp[i] = tag;
      const int lane = threadIdx.x & 31, leader = __ffs(bal) - 1;
      unsigned long long b = 0;
      if (lane == leader) b = atomicAdd(cnt, (unsigned long long)__popc(bal));
      b = __shfl_sync(bal, b, leader);
      out[b + __popc(bal & ((1u << lane) - 1u))] = i;
      atomicAdd(col_cnt + c, 1ull);
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

// ---- per-graph workspace --------------------------------------------------
struct Workspace {
  int K = 0;
  uint64_t n = 0;
  DevBuf<double> x, y0, y1, r0, r1, res;
  DevBuf<unsigned> stamp;
  DevBuf<uint64_t> fa, fb;
  DevBuf<double> carry_h, carry_t;
  DevBuf<unsigned> split_cnt;
  DevBuf<double> split_acc;
  DevBuf<SweepCtl> ctl;
  DevBuf<unsigned long long> counters;  // next_cnt + col_cnt[K] + col_np[K] + col_nn[K]
  DevBuf<double> dcols;                 // col_dr[K], colsum[K], D[K]
  DevBuf<uint32_t> d_src;
  DevBuf<HeavyEntry> heavy;
  DevBuf<unsigned> heavy_cnt;
  DevBuf<unsigned long long> heavy_prefix;
  unsigned level_tag = 0;
  uint64_t ntiles_alloc = 0;
};

static std::mutex g_ws_mu;
static std::map<const Graph*, std::map<int, std::unique_ptr<Workspace>>> g_ws;

static Workspace& workspace(Graph& g, int K, uint64_t ntiles) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  auto& slot = g_ws[&g][K];
  if (!slot) {
    slot = std::make_unique<Workspace>();
    Workspace& w = *slot;
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
    PPRG_CUDA(cudaMemsetAsync(w.stamp.get(), 0, 4 * nk, g.stream));
    w.fa.alloc(nk + 1);
    w.fb.alloc(nk + 1);
    w.ctl.alloc(1);
    w.counters.alloc(1 + 4 * KMAX);
    w.dcols.alloc(3 * KMAX);
    w.d_src.alloc(KMAX);
    w.heavy.alloc((g.m / HEAVY_DEG + 1) * (uint64_t)K + 1);
    w.heavy_cnt.alloc(1);
  }
  Workspace& w = *slot;
  if (ntiles > w.ntiles_alloc) {
    w.carry_h.alloc((ntiles + 1) * K);
    w.carry_t.alloc((ntiles + 1) * K);
    w.split_cnt.alloc(ntiles + 1);
    PPRG_CUDA(cudaMemsetAsync(w.split_cnt.get(), 0, 4 * (ntiles + 1), g.stream));
    w.split_acc.alloc(2 * (ntiles + 1) * K);
    w.ntiles_alloc = ntiles;
  }
  return w;
}

void release_workspaces(const Graph* g) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  g_ws.erase(g);
}

namespace {

inline unsigned grid_for(uint64_t items, int tb = 256) {
  uint64_t b = (items + tb - 1) / tb;
  if (b == 0) b = 1;
  if (b > 65535ull * 32) b = 65535ull * 32;
  return (unsigned)b;
}

template <int K, int MODE>
void launch_sweeps(Graph& g, SweepParams& P, bool cooperative) {
  if (P.split_acc)
    PPRG_CUDA(cudaMemsetAsync(P.split_acc, 0, sizeof(double) * 2 * (P.ntiles + 1) * K, g.stream));
  const size_t smem = Tile<K>::bytes;
  auto kern = k_sweeps<K, MODE>;
  static bool attr_set = false;
  if (!attr_set) {
    PPRG_CUDA(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = true;
  }
  if (cooperative) {
    int per_sm = 0;
    PPRG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
    if (per_sm < 1) fail(EINTERNAL, "sweep kernel cannot be resident");
    const unsigned grid = (unsigned)(per_sm * g.sm_count);
    void* args[] = {(void*)&P};
    PPRG_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3(grid), dim3(NT), args, smem, g.stream));
  } else {
    const uint64_t grid = P.ntiles < (uint64_t)g.sm_count * 8 ? P.ntiles : (uint64_t)g.sm_count * 8;
    kern<<<(unsigned)(grid ? grid : 1), NT, smem, g.stream>>>(P);
  }
  PPRG_CUDA(cudaGetLastError());
}

template <int MODE>
void dispatch_sweeps(Graph& g, int K, SweepParams& P, bool coop) {
  switch (K) {
    case 1: launch_sweeps<1, MODE>(g, P, coop); break;
    case 2: launch_sweeps<2, MODE>(g, P, coop); break;
    case 4: launch_sweeps<4, MODE>(g, P, coop); break;
    case 8: launch_sweeps<8, MODE>(g, P, coop); break;
    case 16: launch_sweeps<16, MODE>(g, P, coop); break;
    case 32: launch_sweeps<32, MODE>(g, P, coop); break;
    case 64: launch_sweeps<64, MODE>(g, P, coop); break;
    default: fail(EINTERNAL, "unsupported column block");
  }
}

int round_k(uint32_t k) {
  int K = 1;
  while (K < (int)k) K <<= 1;
  return K;
}

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
  const uint32_t* tile_lo = nullptr;
  const uint2* desc = nullptr;
  const uint32_t* split_list = nullptr;
  uint64_t n_split = 0;
  double alpha;
  std::vector<uint32_t> src;
  std::vector<double> r_sum;
  std::vector<uint64_t> pushes;
  std::vector<uint32_t> levels;
  std::vector<double> D;
  std::vector<int> scan;
  std::vector<uint32_t> sweeps;
  Block(Graph& g_, Workspace& w_, int K_, uint32_t k_, double a)
      : g(g_), w(w_), K(K_), k(k_), alpha(a), src(KMAX, 0), r_sum(KMAX, 1.0), pushes(KMAX, 0),
        levels(KMAX, 0), D(KMAX, 0.0), scan(KMAX, 0), sweeps(KMAX, 0) {}
};

Block make_block(Graph& g, const uint32_t* sources, uint32_t k, double alpha, bool need_pull) {
  const int K = round_k(k);
  uint64_t ntiles = 0;
  const uint32_t* tl = nullptr;
  const uint2* dsc = nullptr;
  if (need_pull) {
    tl = g.tiles(SWEEP_ELEMS / K, &ntiles);
    dsc = g.tile_desc(SWEEP_ELEMS / K, &ntiles);
  }
  Workspace& w = workspace(g, K, ntiles);
  Block b(g, w, K, k, alpha);
  b.ntiles = ntiles;
  b.tile_lo = tl;
  b.desc = dsc;
  if (need_pull) b.split_list = g.split_rows(SWEEP_ELEMS / K, &b.n_split);
  for (uint32_t c = 0; c < k; ++c) b.src[c] = sources[c];
  for (int c = k; c < K; ++c) b.src[c] = sources[0];  // padding columns are inert
  PPRG_CUDA(cudaMemcpyAsync(w.d_src.get(), b.src.data(), 4 * KMAX, cudaMemcpyHostToDevice, g.stream));
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
  P.ctl = b.w.ctl.get();
  P.k_live = (int)b.k;
  P.max_sweeps = 200000;
  for (int c = 0; c < b.K; ++c) P.src[c] = b.src[c];
  P.in_off = g.cin_off.get();
  P.crow = g.cin_row.get();
  P.cdeg = g.cin_deg.get();
  P.cinv = g.cin_inv.get();
  P.in_off_full = g.in_off.get();
  P.in_nbr = g.in_nbr.get();
  P.tile_lo = b.tile_lo;
  P.desc = b.desc;
  P.ntiles = b.ntiles;
  P.T = SWEEP_ELEMS / b.K;
  P.carry_head = b.w.carry_h.get();
  P.carry_tail = b.w.carry_t.get();
  P.split_cnt = b.w.split_cnt.get();
  P.split_acc = b.w.split_acc.get();
  P.split_list = b.split_list;
  P.n_split = b.n_split;
  return P;
}

// Frontier levels (drain_queue, push.cpp:34-59) for every column in
// `state == 0`. The initial frontier is seed_source (push.cpp:61-66) or, for
// refine, every active node in id order (push.cpp:212-218). A level is
// drained in FIFO-ordered chunks so the reference's loop conditions --
// queue size <= limit and r_sum > lambda_stop, checked before every pop --
// are re-checked every chunk: the queue size of column c at that point is its
// unprocessed entries of this level plus its entries appended to the next.
void drain_levels(Block& b, double r_max, double lam_stop, uint64_t limit, bool from_scan,
                  std::vector<int>& state, CallStats* call) {
  Graph& g = b.g;
  Workspace& w = b.w;
  const int K = b.K;
  const uint64_t n = g.n, nk = n * (uint64_t)K;
  cudaStream_t st = g.stream;
  FrontierParams F;
  std::memset(&F, 0, sizeof F);
  F.off = g.off.get();
  F.nbr = g.nbr.get();
  F.deg = g.deg.get();
  F.res = w.res.get();
  F.x = w.x.get();
  F.stamp = w.stamp.get();
  F.K = K;
  F.alpha = b.alpha;
  for (int c = 0; c < K; ++c) {
    F.src[c] = b.src[c];
    F.thr[c] = r_max;
  }
  const int NC = 1 + 4 * KMAX;
  unsigned long long* next_cnt = w.counters.get();
  unsigned long long* col_cnt = next_cnt + 1;
  unsigned long long* col_np = col_cnt + KMAX;
  unsigned long long* col_nn = col_np + KMAX;
  unsigned long long* col_proc = col_nn + KMAX;
  double* col_dr = w.dcols.get();
  uint64_t* cur = w.fa.get();
  uint64_t* nxt = w.fb.get();
  std::vector<uint64_t> qsize(K, 0);
  uint64_t ncur = 0;
  auto next_tag = [&] {
    if (++w.level_tag == 0) {
      PPRG_CUDA(cudaMemsetAsync(w.stamp.get(), 0, 4 * nk, st));
      w.level_tag = 1;
    }
    return w.level_tag;
  };
  unsigned long long live0 = 0;
  for (uint32_t c = 0; c < b.k; ++c)
    if (state[c] == 0) live0 |= 1ull << c;
  std::vector<unsigned long long> hc(NC);
  if (from_scan) {
    std::vector<double> thr(KMAX, r_max);
    PPRG_CUDA(cudaMemcpyAsync(w.dcols.get() + KMAX, thr.data(), 8 * KMAX, cudaMemcpyHostToDevice, st));
    PPRG_CUDA(cudaMemsetAsync(w.counters.get(), 0, 8 * NC, st));
    k_scan_active<<<grid_for(nk), 256, 0, st>>>(w.res.get(), g.deg.get(), n, K, w.dcols.get() + KMAX,
                                                live0, w.stamp.get(), next_tag(), cur, next_cnt,
                                                col_cnt);
    PPRG_CUDA(cudaMemcpyAsync(hc.data(), w.counters.get(), 8 * NC, cudaMemcpyDeviceToHost, st));
    PPRG_CUDA(cudaStreamSynchronize(st));
    ncur = hc[0];
    for (int c = 0; c < K; ++c) qsize[c] = hc[1 + c];
    call->kernel_launches += 1;
  } else {
    std::vector<uint32_t> hdeg(K);
    for (int c = 0; c < K; ++c)
      PPRG_CUDA(cudaMemcpyAsync(&hdeg[c], g.deg.get() + b.src[c], 4, cudaMemcpyDeviceToHost, st));
    PPRG_CUDA(cudaStreamSynchronize(st));
    std::vector<uint64_t> h;
    for (uint32_t c = 0; c < b.k; ++c)
      if (state[c] == 0 && 1.0 > (double)(hdeg[c] ? hdeg[c] : 1) * r_max) {
        h.push_back((uint64_t)b.src[c] * K + c);
        qsize[c] = 1;
      }
    ncur = h.size();
    if (ncur) PPRG_CUDA(cudaMemcpyAsync(cur, h.data(), 8 * ncur, cudaMemcpyHostToDevice, st));
  }
  const bool bounded = limit != UINT64_MAX;
  const uint64_t chunk_max = bounded ? std::max<uint64_t>(4096, limit / 16) : UINT64_MAX;
  std::vector<double> hdr(KMAX);
  unsigned long long live = 0;
  auto still_live = [&](uint32_t c, uint64_t queued) {
    return queued > 0 && queued <= limit && !(lam_stop > 0 && b.r_sum[c] <= lam_stop);
  };
  for (uint32_t c = 0; c < b.k; ++c) {
    if (state[c] != 0) continue;
    if (still_live(c, qsize[c])) live |= 1ull << c;
    else state[c] = 1;
  }
  while (live && ncur) {
    PPRG_CUDA(cudaMemsetAsync(w.counters.get(), 0, 8 * NC, st));
    const unsigned tag = next_tag();
    uint64_t pos = 0;
    while (pos < ncur && live) {
      const uint64_t chunk = std::min<uint64_t>(chunk_max, ncur - pos);
      PPRG_CUDA(cudaMemsetAsync(col_dr, 0, 8 * KMAX, st));
      PPRG_CUDA(cudaMemsetAsync(col_np, 0, 8 * 2 * KMAX, st));
      F.cur = cur + pos;
      F.ncur = chunk;
      F.next = nxt;
      F.next_cnt = next_cnt;
      F.col_cnt = col_cnt;
      F.col_dr = col_dr;
      F.col_np = col_np;
      F.col_nn = col_nn;
      F.col_proc = col_proc;
      F.col_live = live;
      F.level_tag = tag;
      PPRG_CUDA(cudaMemsetAsync(w.heavy_cnt.get(), 0, 4, st));
      k_frontier<<<grid_for(chunk * 32), 256, 0, st>>>(F, w.heavy.get(), w.heavy_cnt.get());
      PPRG_CUDA(cudaGetLastError());
      call->kernel_launches += 1;
      unsigned nheavy = 0;
      PPRG_CUDA(cudaMemcpyAsync(&nheavy, w.heavy_cnt.get(), 4, cudaMemcpyDeviceToHost, st));
      PPRG_CUDA(cudaStreamSynchronize(st));
      if (nheavy) {
        std::vector<HeavyEntry> hv(nheavy);
        PPRG_CUDA(cudaMemcpyAsync(hv.data(), w.heavy.get(), sizeof(HeavyEntry) * nheavy,
                                  cudaMemcpyDeviceToHost, st));
        PPRG_CUDA(cudaStreamSynchronize(st));
        std::vector<unsigned long long> pre(nheavy + 1, 0);
        for (unsigned h = 0; h < nheavy; ++h) pre[h + 1] = pre[h] + hv[h].deg;
        w.heavy_prefix.ensure(nheavy + 1);
        PPRG_CUDA(cudaMemcpyAsync(w.heavy_prefix.get(), pre.data(), 8 * (nheavy + 1),
                                  cudaMemcpyHostToDevice, st));
        k_frontier_heavy<<<grid_for(pre[nheavy]), 256, 0, st>>>(F, w.heavy.get(),
                                                                w.heavy_prefix.get(), nheavy,
                                                                pre[nheavy]);
        PPRG_CUDA(cudaGetLastError());
        call->kernel_launches += 1;
      }
      PPRG_CUDA(cudaMemcpyAsync(hc.data(), w.counters.get(), 8 * NC, cudaMemcpyDeviceToHost, st));
      PPRG_CUDA(cudaMemcpyAsync(hdr.data(), col_dr, 8 * KMAX, cudaMemcpyDeviceToHost, st));
      PPRG_CUDA(cudaStreamSynchronize(st));
      pos += chunk;
      for (uint32_t c = 0; c < b.k; ++c) {
        if (!((live >> c) & 1ull)) continue;
        b.r_sum[c] -= hdr[c];
        b.pushes[c] += hc[1 + KMAX + c];
        const uint64_t queued = (qsize[c] - hc[1 + 3 * KMAX + c]) + hc[1 + c];
        if (pos < ncur && !still_live(c, queued)) {
          live &= ~(1ull << c);
          state[c] = 1;
        }
      }
    }
    for (uint32_t c = 0; c < b.k; ++c) {
      if (!((live >> c) & 1ull)) continue;
      b.levels[c] += 1;
      qsize[c] = hc[1 + c];
      if (!still_live(c, qsize[c])) {
        live &= ~(1ull << c);
        state[c] = 1;
      }
    }
    std::swap(cur, nxt);
    ncur = hc[0];
  }
  for (uint32_t c = 0; c < b.k; ++c)
    if (state[c] == 0) state[c] = 1;
}

// recompute_r_sum (push.cpp:9-15) over the push-form residues of every column
void exact_rsum(Block& b, const std::vector<int>& which) {
  Graph& g = b.g;
  cudaStream_t st = g.stream;
  const uint64_t nk = g.n * (uint64_t)b.K;
  PPRG_CUDA(cudaMemsetAsync(b.w.dcols.get() + KMAX, 0, 8 * KMAX, st));
  k_colsum<<<grid_for(nk), 256, 0, st>>>(b.w.res.get(), g.n, b.K, b.w.dcols.get() + KMAX);
  std::vector<double> exact(KMAX);
  PPRG_CUDA(cudaMemcpyAsync(exact.data(), b.w.dcols.get() + KMAX, 8 * KMAX, cudaMemcpyDeviceToHost, st));
  PPRG_CUDA(cudaStreamSynchronize(st));
  for (uint32_t c = 0; c < b.k; ++c) {
    if (!which[c]) continue;
    if (std::fabs(exact[c] - b.r_sum[c]) > 1e-6)
      fail(EINTERNAL, "push: r_sum drifted more than 1e-6 from the residues");
    b.r_sum[c] = exact[c];
  }
}

// Global phase: epochs of asynchronous pull sweeps in one persistent
// cooperative kernel (push.cpp:168-197) for the columns with scan[c] set.
void global_phase(Block& b, double lambda, uint32_t E, CallStats* call) {
  Graph& g = b.g;
  Workspace& w = b.w;
  cudaStream_t st = g.stream;
  const uint64_t nk = g.n * (uint64_t)b.K;
  const double m_eff = (double)g.m_eff();
  if (E > EMAX) fail(EINVAL_, "epoch_num exceeds 64");
  PPRG_CUDA(cudaMemsetAsync(w.dcols.get() + 2 * KMAX, 0, 8 * KMAX, st));
  k_init_pull<<<grid_for(nk), 256, 0, st>>>(w.x.get(), g.deg.get(), g.inv_deg.get(), g.n, b.K,
                                            b.alpha, w.y0.get(), w.dcols.get() + 2 * KMAX);
  PPRG_CUDA(cudaMemcpyAsync(b.D.data(), w.dcols.get() + 2 * KMAX, 8 * KMAX, cudaMemcpyDeviceToHost, st));
  PPRG_CUDA(cudaMemsetAsync(w.ctl.get(), 0, sizeof(SweepCtl), st));
  PPRG_CUDA(cudaStreamSynchronize(st));
  SweepParams P = base_params(b);
  for (uint32_t e = 0; e < E; ++e) {
    const double el = std::pow(lambda, static_cast<double>(e + 1) / E);  // push.cpp:176-178
    P.lam[e] = el;
    P.thr[e] = el / m_eff;
  }
  for (int c = 0; c < b.K; ++c) {
    P.init[c].r_sum = b.r_sum[c];
    P.init[c].D = b.D[c];
    int ep = 0;
    while (ep < (int)E && !(b.r_sum[c] > P.lam[ep])) ++ep;
    P.init[c].epoch = ep;
    P.init[c].done = !b.scan[c] || ep >= (int)E;
  }
  P.E = (int)E;
  P.x = w.x.get();
  P.y[0] = P.y[1] = w.y0.get();
  EventTimer tm(st);
  tm.start();
  dispatch_sweeps<M_POWERPUSH>(g, b.K, P, true);
  tm.stop();
  SweepCtl hc;
  PPRG_CUDA(cudaMemcpyAsync(&hc, w.ctl.get(), sizeof hc, cudaMemcpyDeviceToHost, st));
  call->sweep_ms += tm.ms();
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
  cudaStream_t st = g.stream;
  const uint64_t n = g.n, nk = n * (uint64_t)b.K;
  const uint32_t k = b.k;
  const cudaMemcpyKind kind = out.on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  bool any_scan = false;
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
  DevBuf<double> o_res, o_rsd;
  const bool direct = out.on_device;  // write straight into the caller's device buffers
  if (out.reserve && !direct) o_res.alloc(n * k);
  if (out.residue && !direct) o_rsd.alloc(n * k);
  Q.out_reserve = out.reserve ? (direct ? out.reserve : o_res.get()) : nullptr;
  Q.out_residue = out.residue ? (direct ? out.residue : o_rsd.get()) : nullptr;
  // rows with in-degree 0 (other than sources) are never visited: they hold 0
  if (Q.out_reserve) PPRG_CUDA(cudaMemsetAsync(Q.out_reserve, 0, 8 * n * k, st));
  if (Q.out_residue) PPRG_CUDA(cudaMemsetAsync(Q.out_residue, 0, 8 * n * k, st));
  Q.res_inter = residues_inplace ? w.res.get() : nullptr;
  Q.push_res = w.res.get();
  Q.x = w.x.get();
  Q.y[0] = Q.y[1] = w.y0.get();
  for (int c = 0; c < b.K; ++c) {
    Q.final_pull[c] = b.scan[c];
    Q.init[c].r_sum = b.r_sum[c];
    Q.init[c].D = b.D[c];
  }
  PPRG_CUDA(cudaMemsetAsync(w.ctl.get(), 0, sizeof(SweepCtl), st));
  dispatch_sweeps<M_FINAL>(g, b.K, Q, true);
  call->kernel_launches += 1;
  SweepCtl fc;
  PPRG_CUDA(cudaMemcpyAsync(&fc, w.ctl.get(), sizeof fc, cudaMemcpyDeviceToHost, st));
  if (out.reserve && !direct) PPRG_CUDA(cudaMemcpyAsync(out.reserve, o_res.get(), 8 * n * k, kind, st));
  if (out.residue && !direct) PPRG_CUDA(cudaMemcpyAsync(out.residue, o_rsd.get(), 8 * n * k, kind, st));
  PPRG_CUDA(cudaStreamSynchronize(st));
  for (uint32_t c = 0; c < k; ++c) {
    if (!b.scan[c]) continue;
    const double exact = fc.pushed[0][c];
    if (std::fabs(exact - b.r_sum[c]) > 1e-6)
      fail(EINTERNAL, "push: r_sum drifted more than 1e-6 from the residues");
    b.r_sum[c] = exact;
  }
}

void power_push_block(Block& b, double lambda, uint32_t epoch_num, int64_t scan_threshold,
                      CallStats* call) {
  const double m_eff = (double)b.g.m_eff();
  const uint64_t nk = b.g.n * (uint64_t)b.K;
  cudaStream_t st = b.g.stream;
  PPRG_CUDA(cudaMemsetAsync(b.w.x.get(), 0, 8 * nk, st));
  PPRG_CUDA(cudaMemsetAsync(b.w.res.get(), 0, 8 * nk, st));
  k_seed<<<1, KMAX, 0, st>>>(b.w.res.get(), b.w.d_src.get(), b.K, 1.0);
  const double r_max = lambda / m_eff;  // push.cpp:157-160
  const uint64_t limit = scan_threshold < 0 ? b.g.n / 4 : (uint64_t)scan_threshold;
  std::vector<int> state(KMAX, 2);
  for (uint32_t c = 0; c < b.k; ++c) state[c] = 0;
  drain_levels(b, r_max, lambda, limit, false, state, call);
  std::vector<int> all(KMAX, 1);
  exact_rsum(b, all);
  bool any = false;
  for (uint32_t c = 0; c < b.k; ++c) {
    b.scan[c] = b.r_sum[c] > lambda;  // push.cpp:168
    any |= b.scan[c] != 0;
  }
  if (any) global_phase(b, lambda, epoch_num, call);
}

}  // namespace

// Columns per block: the gathered operand y (n*K doubles) and the state x
// should stay L2-resident (126 MB), so K shrinks as n grows. PPRG_COLUMNS
// overrides (power of two <= 64).
uint32_t block_columns(uint64_t n, uint32_t k) {
  if (const char* e = std::getenv("PPRG_COLUMNS")) {
    const long v = std::strtol(e, nullptr, 10);
    if (v >= 1 && v <= KMAX) return (uint32_t)v;
  }
  uint32_t K = KMAX;
  while (K > 1 && 8.0 * (double)n * K > 80e6) K >>= 1;
  return K < k ? K : (k ? k : 1);
}

void run_push_engine(Graph& g, Engine eng, const uint32_t* sources, uint32_t k, double alpha,
                     double lambda, uint32_t epoch_num, int64_t scan_threshold, double r_max_fifo,
                     double lambda_stop_fifo, const Outputs& out, ColumnStats* cols,
                     CallStats* call) {
  DeviceGuard dg(g.device);
  std::lock_guard<std::mutex> lk(g.mu);
  for (uint32_t c = 0; c < k; ++c)
    if (sources[c] >= g.n) fail(EINVAL_, "source out of range");
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
    EventTimer tdev(g.stream);
    tdev.start();
    if (eng == Engine::PowItr || eng == Engine::SimFwdPush) {
      const uint64_t n = g.n, nk = n * (uint64_t)b.K;
      cudaStream_t st = g.stream;
      Workspace& w = b.w;
      PPRG_CUDA(cudaMemsetAsync(w.x.get(), 0, 8 * nk, st));
      PPRG_CUDA(cudaMemsetAsync(w.r0.get(), 0, 8 * nk, st));
      PPRG_CUDA(cudaMemsetAsync(w.r1.get(), 0, 8 * nk, st));  // rows never visited stay 0
      PPRG_CUDA(cudaMemsetAsync(w.y1.get(), 0, 8 * nk, st));
      PPRG_CUDA(cudaMemsetAsync(w.dcols.get() + 2 * KMAX, 0, 8 * KMAX, st));
      k_seed<<<1, KMAX, 0, st>>>(w.r0.get(), w.d_src.get(), b.K, 1.0);
      k_init_pull<<<grid_for(nk), 256, 0, st>>>(w.r0.get(), g.deg.get(), g.inv_deg.get(), n, b.K,
                                                alpha, w.y0.get(), w.dcols.get() + 2 * KMAX);
      PPRG_CUDA(cudaMemcpyAsync(b.D.data(), w.dcols.get() + 2 * KMAX, 8 * KMAX, cudaMemcpyDeviceToHost, st));
      PPRG_CUDA(cudaMemsetAsync(w.ctl.get(), 0, sizeof(SweepCtl), st));
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
      EventTimer tm(st);
      tm.start();
      if (eng == Engine::PowItr) dispatch_sweeps<M_POWITR>(g, b.K, P, true);
      else dispatch_sweeps<M_SIMFWD>(g, b.K, P, true);
      tm.stop();
      SweepCtl hc;
      PPRG_CUDA(cudaMemcpyAsync(&hc, w.ctl.get(), sizeof hc, cudaMemcpyDeviceToHost, st));
      call->sweep_ms += tm.ms();
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
      PPRG_CUDA(cudaMemsetAsync(b.w.x.get(), 0, 8 * nk, g.stream));
      PPRG_CUDA(cudaMemsetAsync(b.w.res.get(), 0, 8 * nk, g.stream));
      k_seed<<<1, KMAX, 0, g.stream>>>(b.w.res.get(), b.w.d_src.get(), b.K, 1.0);
      std::vector<int> state(KMAX, 2);
      for (uint32_t c = 0; c < kb; ++c) state[c] = 0;
      drain_levels(b, r_max_fifo, lambda_stop_fifo, UINT64_MAX, false, state, call);
      std::vector<int> all(KMAX, 1);
      exact_rsum(b, all);
      finalize(b, o, false, call);
    } else {
      power_push_block(b, lambda, epoch_num, scan_threshold, call);
      finalize(b, o, false, call);
    }
    tdev.stop();
    call->device_ms += tdev.ms();
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
  Block b = make_block(g, sources, k, alpha, true);
  power_push_block(b, lambda, 8, -1, call);
  Outputs none;
  finalize(b, none, true, call);
  // refine (push.cpp:208-222): every active node in id order, drain, recompute
  std::vector<int> state(KMAX, 2);
  for (uint32_t c = 0; c < k; ++c) state[c] = 0;
  drain_levels(b, r_max, 0.0, UINT64_MAX, true, state, call);
  std::vector<int> all(KMAX, 1);
  exact_rsum(b, all);
  for (uint32_t c = 0; c < k; ++c) {
    cols[c].r_sum = b.r_sum[c];
    cols[c].pushes = b.pushes[c];
    cols[c].sweeps = b.sweeps[c];
    cols[c].local_levels = b.levels[c];
    cols[c].used_scan_phase = b.scan[c];
  }
  view->K = b.K;
  view->k = k;
  view->x = b.w.x.get();
  view->res = b.w.res.get();
  view->d_src = b.w.d_src.get();
  view->src = b.src;
}

}  // namespace pprg
