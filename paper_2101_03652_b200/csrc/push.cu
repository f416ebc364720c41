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
#include <cmath>
#include <cstdlib>
#include <algorithm>
#include <cstdio>
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
constexpr int NT = PPRG_NT;
#define PPRG_MAX_PEERS 15             // threads per block for the sweep kernels
#ifndef PPRG_TILE_U
#define PPRG_TILE_U 8
#endif
constexpr int TILE_U = PPRG_TILE_U;     // narrow path: gathers per thread per tile
constexpr int SWEEP_ELEMS = NT * TILE_U;  // edges x columns per narrow tile

enum SweepMode : int { M_POWERPUSH = 0, M_POWITR = 1, M_SIMFWD = 2, M_FINAL = 3 };

thread_local TraceSink* g_trace = nullptr;
thread_local StepSink* g_obs = nullptr;

uint64_t host_now_ns() {
  return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

struct SweepCtl {
  unsigned long long barrier;
  GridBarrier gbar;
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
  int out_epoch[KMAX];
  unsigned long long out_pushes[KMAX];
  unsigned total_sweeps;
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
  const TileDesc* desc;        // row-aligned tile plan
  double* hub_acc;             // [ntiles][K] per-piece partial sums of hub rows
  unsigned* hub_cnt;           // [nhubs] arrived pieces
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

  SweepCtl* ctl;
  double* out_reserve;         // finalize outputs, query-major [c*n + u]
  double* out_residue;
  double* res_inter;           // finalize: explicit residues back into [u*K + c] (SpeedPPR)
  uint32_t max_sweeps;
  double* peer_y[PPRG_MAX_PEERS];  // fused exchange: other parts' y buffers (P2P / same device)
  int npeers;
  TracePoint* trace;            // per-sweep progress of column 0 (traced calls), or null
  uint32_t trace_cap;
  uint64_t own_lo, own_hi;      // node range this launch owns (vertex partition; else [0, n))
  unsigned long long handoff_np;  // refine epoch: hand off to the frontier below this many edge pushes
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

// Tile geometry: a row-aligned tile holds at most T = SWEEP_ELEMS/K in-edges
// and at most RMAX rows (host-built plan, Graph::tile_plan). Its gathered
// values vals[e*K + c] and its row data live in shared memory.
template <int K>
struct Tile {
  static constexpr int T = SWEEP_ELEMS / K;
  static constexpr int RMAX = T < 256 ? T : 256;
  static constexpr int LONG = K == 1 ? 32 : 16;  // rows longer than this: warp per row
  // vals[SWEEP_ELEMS] f64 | sinv[RMAX] f64 | hub[NT/32 * K] f64 | soff[RMAX+1] i32 | snode, sdeg, slong [RMAX] u32
  static constexpr size_t bytes = 8ull * (SWEEP_ELEMS + RMAX + (NT / 32) * K) +
                                  4ull * (RMAX + 1) + 12ull * RMAX + 16;
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
      st_state(P.x + ix, inflow);
      if (dg) {
        const double yv = oma * inflow * inv;
        P.y[0][ix] = yv;
        for (int p = 0; p < P.npeers; ++p) P.peer_y[p][ix] = yv;  // fused exchange
      }
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

template <int K, int MODE>
__device__ __forceinline__ void decide_at(const SweepParams& P, const ColSh* cs,
                                          const double* thr_cur, uint32_t u, int c, double acc,
                                          uint32_t dg, double inv, const double* yg,
                                          const double* rcur, double* rnxt, double* ynxt, Acc& a) {
  const uint64_t ix = (uint64_t)u * K + c;
  decide<K, MODE>(P, cs, thr_cur, u, c, acc, __ldcg(P.x + ix),
                  (MODE == M_POWITR || MODE == M_SIMFWD) ? __ldcg(rcur + ix) : 0.0, dg, inv, yg,
                  rnxt, ynxt, a);
}

// One piece of a hub row (more in-edges than a tile holds): the block sums its
// edges per column, adds the piece total into the row's accumulator, and the
// last piece to arrive decides the row (release-ordered counter; the partials
// are read back from L2). Only hub pieces pay this protocol.
template <int K, int MODE>
__device__ __noinline__ void hub_piece(const SweepParams& P, const TileDesc& d, uint64_t j,
                                       double* hubsh, int* flag, const ColSh* cs, const double* thr_cur,
                                       const double* yg, const double* rcur, double* rnxt,
                                       double* ynxt, Acc& a) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = tid % K;
  const uint64_t total = (uint64_t)d.ne * K;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  uint64_t f = tid;
  for (; f + 3 * NT < total; f += 4 * NT) {
    const uint32_t i0 = __ldg(P.in_nbr + d.e0 + f / K);
    const uint32_t i1 = __ldg(P.in_nbr + d.e0 + (f + NT) / K);
    const uint32_t i2 = __ldg(P.in_nbr + d.e0 + (f + 2 * NT) / K);
    const uint32_t i3 = __ldg(P.in_nbr + d.e0 + (f + 3 * NT) / K);
    s0 += yg[(uint64_t)i0 * K + c];
    s1 += yg[(uint64_t)i1 * K + c];
    s2 += yg[(uint64_t)i2 * K + c];
    s3 += yg[(uint64_t)i3 * K + c];
  }
  for (; f < total; f += NT) s0 += yg[(uint64_t)__ldg(P.in_nbr + d.e0 + f / K) * K + c];
  double s = (s0 + s1) + (s2 + s3);
#pragma unroll
  for (int o = 16; o >= K && o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  for (int i = tid; i < (NT / 32) * K; i += NT) hubsh[i] = 0.0;
  __syncthreads();
  if (lane < K) hubsh[warp * K + c] = s;  // the lanes holding this warp's per-column sums
  __syncthreads();
  if (tid < K) {
    double t = 0.0;
    for (int w = 0; w < NT / 32; ++w) t += hubsh[w * K + tid];
    P.hub_acc[j * K + tid] = t;  // this piece's partial (slot = its tile)
  }
  __syncthreads();
  if (tid == 0) {
    unsigned old;
    asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(old) : "l"(P.hub_cnt + d.hub) : "memory");
    *flag = old == d.npieces - 1;
    if (*flag) P.hub_cnt[d.hub] = 0;
  }
  __syncthreads();
  if (*flag && tid < K) {
    // the last piece sums the partials in piece order: deterministic
    const double* part = P.hub_acc + (j - d.piece) * K + tid;
    double acc = 0.0;
    for (uint32_t p = 0; p < d.npieces; ++p) acc += __ldcg(part + (uint64_t)p * K);
    const uint32_t u = __ldg(P.crow + d.r0);
    decide_at<K, MODE>(P, cs, thr_cur, u, tid, acc, __ldg(P.cdeg + d.r0), __ldg(P.cinv + d.r0), yg,
                       rcur, rnxt, ynxt, a);
  }
}

// One row-aligned tile: gather y of every in-edge into shared memory (all
// loads of the tile issued together), then one thread per (row, column) sums
// its row and decides; rows longer than LONG are summed by a whole warp.
template <int K, int MODE>
__device__ __forceinline__ void tile_rows(const SweepParams& P, const TileDesc& d, char* smem,
                                          const ColSh* cs, const double* thr_cur, const double* yg,
                                          const double* rcur, double* rnxt, double* ynxt, Acc& a,
                                          const BlockAcc& ba, uint32_t* nlong,
                                          const unsigned long long* dn_slot, TileDesc* dn) {
  using TC = Tile<K>;
  constexpr int RMAX = TC::RMAX;
  double* vals = reinterpret_cast<double*>(smem);
  double* sinv = vals + SWEEP_ELEMS;
  int32_t* soff = reinterpret_cast<int32_t*>(sinv + RMAX + (NT / 32) * K);
  uint32_t* snode = reinterpret_cast<uint32_t*>(soff + RMAX + 1);
  uint32_t* sdeg = snode + RMAX;
  uint32_t* slong = sdeg + RMAX;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = tid % K;
  const uint32_t nr = d.nr;
  // ---- stage rows and gather (one memory latency) -------------------------
  for (uint32_t t = tid; t <= nr; t += NT) soff[t] = (int32_t)(__ldg(P.in_off + d.r0 + t) - d.e0);
  for (uint32_t t = tid; t < nr; t += NT) {
    snode[t] = __ldg(P.crow + d.r0 + t);
    sdeg[t] = __ldg(P.cdeg + d.r0 + t);
    sinv[t] = __ldg(P.cinv + d.r0 + t);
    const uint64_t len = __ldg(P.in_off + d.r0 + t + 1) - __ldg(P.in_off + d.r0 + t);
    if (len > (uint64_t)TC::LONG) slong[atomicAdd(nlong, 1u)] = t;
  }
  {
    const uint32_t total = d.ne * K;
    constexpr int U = TILE_U;
    for (uint32_t f0 = 0; f0 < total; f0 += U * NT) {
      uint32_t id[U];
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const uint32_t f = f0 + tid + i * NT;
        id[i] = f < total ? __ldg(P.in_nbr + d.e0 + f / K) : 0u;
      }
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const uint32_t f = f0 + tid + i * NT;
        if (f < total) vals[f] = yg[(uint64_t)id[i] * K + (f % K)];
      }
    }
  }
  __syncthreads();
  if (dn_slot) *dn = P.desc[*dn_slot < P.ntiles ? *dn_slot : 0];  // next tile's descriptor
  // ---- short rows: one thread per (row, column) ------------------------------
  for (uint32_t fi = tid; fi < nr * K; fi += NT) {
    const uint32_t r = fi / K;
    const int32_t b = soff[r], e = soff[r + 1];
    if (e - b > TC::LONG) continue;
    const uint32_t u = snode[r];
    const uint64_t ix = (uint64_t)u * K + c;
    const double xo = __ldcg(P.x + ix);  // issued before the sum: lands meanwhile
    const double rc = (MODE == M_POWITR || MODE == M_SIMFWD) ? __ldcg(rcur + ix) : 0.0;
    double s0 = 0.0, s1 = 0.0;
    int32_t q = b;
    for (; q + 1 < e; q += 2) {
      s0 += vals[q * K + c];
      s1 += vals[(q + 1) * K + c];
    }
    if (q < e) s0 += vals[q * K + c];
    decide<K, MODE>(P, cs, thr_cur, u, c, s0 + s1, xo, rc, sdeg[r], sinv[r], yg, rnxt, ynxt, a);
  }
  // ---- long rows: one warp per row -----------------------------------------
  {
    constexpr int KC = K < 32 ? K : 32;
    constexpr int CPL = K / KC;
    constexpr int ES = 32 / KC;  // edge slots per warp
    const int es = lane / KC, kc = lane % KC;
    const uint32_t nl = *nlong;
    for (uint32_t li = warp; li < nl; li += NT / 32) {
      const uint32_t r = slong[li];
      const int32_t b = soff[r], e = soff[r + 1];
      double s[CPL];
#pragma unroll
      for (int q = 0; q < CPL; ++q) s[q] = 0.0;
      for (int32_t p = b + es; p < e; p += ES)
#pragma unroll
        for (int q = 0; q < CPL; ++q) s[q] += vals[p * K + kc + q * KC];
#pragma unroll
      for (int q = 0; q < CPL; ++q)
#pragma unroll
        for (int o = KC; o < 32; o <<= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], o);
      if (es == 0) {
        if constexpr (CPL == 1) {
          decide_at<K, MODE>(P, cs, thr_cur, snode[r], kc, s[0], sdeg[r], sinv[r], yg, rcur, rnxt,
                             ynxt, a);
        } else {  // K = 64: lane kc decides columns kc and kc+32; counters via shared atomics
#pragma unroll
          for (int q = 0; q < CPL; ++q) {
            Acc b2;
            const int cc = kc + q * KC;
            decide_at<K, MODE>(P, cs, thr_cur, snode[r], cc, s[q], sdeg[r], sinv[r], yg, rcur,
                               rnxt, ynxt, b2);
            if (b2.push != 0.0) atomicAdd(&ba.push[cc], b2.push);
            if (b2.d != 0.0) atomicAdd(&ba.d[cc], b2.d);
            if (b2.np) atomicAdd(&ba.np[cc], b2.np);
            if (b2.nn) atomicAdd(&ba.nn[cc], b2.nn);
            if (b2.et) atomicAdd(&ba.et[cc], b2.et);
          }
        }
      }
    }
  }
  __syncthreads();
  if (tid == 0) *nlong = 0;
}

// Wide column blocks (K >= WIDE_K): tiles of up to WIDE_T in-edges and
// RMAX_W rows; warps take rows from a shared counter and gather each in-edge's
// K contiguous values straight into registers (lanes = edge slots x columns),
// so no value staging in shared memory and no per-tile hub split below WIDE_T.
constexpr int WIDE_K = 4;
#ifndef PPRG_WIDE_T
#define PPRG_WIDE_T 4096
#endif
#ifndef PPRG_RMAX_W
#define PPRG_RMAX_W 256
#endif
constexpr uint32_t WIDE_T = PPRG_WIDE_T;
constexpr uint32_t RMAX_W = PPRG_RMAX_W;

// Sum of y over the in-edges [b, e) of one row for my columns, by one warp.
// Lanes = ES edge slots x KC column lanes (x CPL contiguous columns). The ids
// of 32 consecutive edges are loaded once, coalesced, and broadcast by shuffle;
// the gathers are then issued G at a time into registers before any add, so
// each warp keeps G row-loads in flight (tail slots re-load the last edge and
// are masked out of the sum).
#ifndef PPRG_G
#define PPRG_G 8
#endif
template <int K>
__device__ __forceinline__ void warp_row_sum(const SweepParams& P, const double* yg, uint64_t b,
                                             uint64_t e, double (&s)[(K < 32 ? 1 : K / 32)],
                                             bool have_first = false, uint32_t first_id = 0) {
  constexpr int KC = K < 32 ? K : 32;
  constexpr int CPL = K / KC;
  constexpr int ES = 32 / KC;
  constexpr int G = PPRG_G;
  const int lane = threadIdx.x & 31, es = lane / KC, kc = lane % KC;
  const double* ybase = yg + kc * CPL;
  double acc[CPL][2];
#pragma unroll
  for (int q = 0; q < CPL; ++q) acc[q][0] = acc[q][1] = 0.0;
  for (uint64_t p0 = b; p0 < e; p0 += 32) {
    const uint64_t pl = p0 + lane;
    const uint32_t myid = (have_first && p0 == b) ? first_id : (pl < e ? ld_stream(P.in_nbr + pl) : 0u);
    const int cnt = e - p0 < 32 ? (int)(e - p0) : 32;
    for (int j0 = 0; j0 < cnt; j0 += G * ES) {
      double v[G][CPL];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int j = j0 + g * ES + es;
        const uint32_t id = __shfl_sync(0xffffffffu, myid, j < cnt ? j : cnt - 1);
        const double* src = ybase + (uint64_t)id * K;
        if constexpr (CPL == 2) {
          const double2 v2 = ld_gather2(src);
          v[g][0] = v2.x;
          v[g][1] = v2.y;
        } else {
          v[g][0] = ld_gather(src);
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const bool ok = j0 + g * ES + es < cnt;
#pragma unroll
        for (int q = 0; q < CPL; ++q) acc[q][g & 1] += ok ? v[g][q] : 0.0;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < CPL; ++q) {
    s[q] = acc[q][0] + acc[q][1];
#pragma unroll
    for (int o = KC; o < 32; o <<= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], o);
  }
}

template <int K, int MODE>
__device__ __forceinline__ void decide_cols(const SweepParams& P, const ColSh* cs,
                                            const double* thr_cur, uint32_t u, const double* s,
                                            const double* xo, const double* rc, uint32_t dg,
                                            double inv, const double* yg, double* rnxt,
                                            double* ynxt, Acc& a, const BlockAcc& ba) {
  constexpr int KC = K < 32 ? K : 32;
  constexpr int CPL = K / KC;
  const int kc = (threadIdx.x & 31) % KC;
  if constexpr (CPL == 1) {
    decide<K, MODE>(P, cs, thr_cur, u, kc, s[0], xo[0], rc[0], dg, inv, yg, rnxt, ynxt, a);
  } else {  // K = 64: lane kc owns columns 2kc, 2kc+1; counters via shared atomics
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      Acc b2;
      const int cc = kc * CPL + q;
      decide<K, MODE>(P, cs, thr_cur, u, cc, s[q], xo[q], rc[q], dg, inv, yg, rnxt, ynxt, b2);
      if (b2.push != 0.0) atomicAdd(&ba.push[cc], b2.push);
      if (b2.d != 0.0) atomicAdd(&ba.d[cc], b2.d);
      if (b2.np) atomicAdd(&ba.np[cc], b2.np);
      if (b2.nn) atomicAdd(&ba.nn[cc], b2.nn);
      if (b2.et) atomicAdd(&ba.et[cc], b2.et);
    }
  }
}

// Long-row counter slot of the wide layout (zeroed at kernel start).
template <int K>
__device__ __forceinline__ uint32_t* wide_long_count(char* smem) {
  uint64_t* soff = reinterpret_cast<uint64_t*>(smem);
  double* sinv = reinterpret_cast<double*>(soff + RMAX_W + 1);
  double* spart = sinv + RMAX_W;
  uint32_t* snode = reinterpret_cast<uint32_t*>(spart + (NT / 32) * K);
  return snode + 3 * RMAX_W;
}

// Wide column blocks: warps take rows from a shared counter and sum each row
// with warp_row_sum; rows longer than LONG_W in-edges are summed by all warps
// of the block together (partials in shared memory) so no warp lags the tile.
#ifndef PPRG_LONG_W
#define PPRG_LONG_W 384
#endif
constexpr uint32_t LONG_W = PPRG_LONG_W;

template <int K, int MODE>
__device__ __forceinline__ void tile_rows_wide(const SweepParams& P, const TileDesc& d, char* smem,
                                               const ColSh* cs, const double* thr_cur,
                                               const double* yg, const double* rcur, double* rnxt,
                                               double* ynxt, Acc& a, const BlockAcc& ba,
                                               uint32_t* rowctr,
                                               const unsigned long long* dn_slot, TileDesc* dn) {
  constexpr int KC = K < 32 ? K : 32;
  constexpr int CPL = K / KC;
  constexpr int NW = NT / 32;
  uint64_t* soff = reinterpret_cast<uint64_t*>(smem);
  double* sinv = reinterpret_cast<double*>(soff + RMAX_W + 1);
  double* spart = sinv + RMAX_W;                       // [NW][K] long-row partials
  uint32_t* snode = reinterpret_cast<uint32_t*>(spart + NW * K);
  uint32_t* sdeg = snode + RMAX_W;
  uint32_t* slong = sdeg + RMAX_W;                     // [RMAX_W] long rows; slong[RMAX_W] = count
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int es0 = lane < KC;  // lanes holding the reduced sums
  const int kc = lane % KC;
  const uint32_t nr = d.nr;
  for (uint32_t t = tid; t <= nr; t += NT) soff[t] = __ldg(P.in_off + d.r0 + t);
  for (uint32_t t = tid; t < nr; t += NT) {
    snode[t] = __ldg(P.crow + d.r0 + t);
    sdeg[t] = __ldg(P.cdeg + d.r0 + t);
    sinv[t] = __ldg(P.cinv + d.r0 + t);
    const uint64_t len = __ldg(P.in_off + d.r0 + t + 1) - __ldg(P.in_off + d.r0 + t);
    if (len > LONG_W) slong[atomicAdd(&slong[RMAX_W], 1u)] = t;
  }
  __syncthreads();
  if (dn_slot) *dn = P.desc[*dn_slot < P.ntiles ? *dn_slot : 0];  // next tile's descriptor
  // ---- short rows: one warp per row, dynamic -----------------------------
  // Rows are taken one ahead: the next row's first 32 in-edge ids are loaded
  // before this row's gathers, so their latency hides behind the gathers.
  auto grab = [&]() -> uint32_t {
    uint32_t r = 0;
    if (lane == 0) r = atomicAdd(rowctr, 1u);
    return __shfl_sync(0xffffffffu, r, 0);
  };
  auto first_ids = [&](uint32_t r) -> uint32_t {
    if (r >= nr) return 0u;
    const uint64_t b = soff[r], e = soff[r + 1];
    return (e - b <= LONG_W && b + lane < e) ? ld_stream(P.in_nbr + b + lane) : 0u;
  };
  uint32_t r = grab();
  uint32_t ids = first_ids(r);
  while (r < nr) {
    const uint64_t b = soff[r], e = soff[r + 1];
    const uint32_t rn = grab();
    const uint32_t ids_n = first_ids(rn);
    if (e - b <= LONG_W) {
      const uint32_t u = snode[r];
      double xo[CPL], rc[CPL], s[CPL];
#pragma unroll
      for (int q = 0; q < CPL; ++q) {  // issued early; lands during the edge loop
        const uint64_t ix = (uint64_t)u * K + kc * CPL + q;
        xo[q] = es0 ? ld_state(P.x + ix) : 0.0;
        rc[q] = (es0 && (MODE == M_POWITR || MODE == M_SIMFWD)) ? __ldcg(rcur + ix) : 0.0;
      }
      warp_row_sum<K>(P, yg, b, e, s, true, ids);
      if (es0) decide_cols<K, MODE>(P, cs, thr_cur, u, s, xo, rc, sdeg[r], sinv[r], yg, rnxt, ynxt, a, ba);
    }
    r = rn;
    ids = ids_n;
  }
  // ---- long rows: all warps split the edges ---------------------------------
  const uint32_t nl = slong[RMAX_W];
  for (uint32_t li = 0; li < nl; ++li) {
    const uint32_t r = slong[li];
    const uint64_t b = soff[r], e = soff[r + 1];
    const uint64_t chunk = ((e - b) + NW - 1) / NW;
    const uint64_t wb = b + warp * chunk, we = wb + chunk < e ? wb + chunk : e;
    double s[CPL];
    warp_row_sum<K>(P, yg, wb < e ? wb : e, we, s);
    if (es0)
#pragma unroll
      for (int q = 0; q < CPL; ++q) spart[warp * K + kc * CPL + q] = s[q];
    __syncthreads();
    if (warp == 0 && es0) {
      const uint32_t u = snode[r];
      double xo[CPL], rc[CPL];
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const uint64_t ix = (uint64_t)u * K + kc * CPL + q;
        xo[q] = __ldcg(P.x + ix);
        rc[q] = (MODE == M_POWITR || MODE == M_SIMFWD) ? __ldcg(rcur + ix) : 0.0;
        double t = 0.0;
        for (int w = 0; w < NW; ++w) t += spart[w * K + kc * CPL + q];
        s[q] = t;
      }
      decide_cols<K, MODE>(P, cs, thr_cur, u, s, xo, rc, sdeg[r], sinv[r], yg, rnxt, ynxt, a, ba);
    }
    __syncthreads();
  }
  __syncthreads();
  if (tid == 0) {
    *rowctr = 0;
    slong[RMAX_W] = 0;
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
  if (u < P.own_lo || u >= P.own_hi) return;  // another partition's row
  if (__ldg(P.in_off_full + u + 1) != __ldg(P.in_off_full + u)) return;
  const uint64_t ix = (uint64_t)u * K + tid;
  decide<K, MODE>(P, cs, thr_cur, u, tid, 0.0, __ldcg(P.x + ix),
                  (MODE == M_POWITR || MODE == M_SIMFWD) ? __ldcg(rcur + ix) : 0.0, __ldg(P.deg + u),
                  __ldg(P.inv_deg + u), yg, rnxt, ynxt, a);
}

template <int K, int MODE>
#ifndef PPRG_MINB
#define PPRG_MINB 8
#endif
#ifndef PPRG_MINB_NARROW
#define PPRG_MINB_NARROW PPRG_MINB
#endif
__global__ void __launch_bounds__(NT, (K >= 4 ? PPRG_MINB : PPRG_MINB_NARROW))
    k_sweeps(const __grid_constant__ SweepParams P) {
  using TC = Tile<K>;
  extern __shared__ __align__(16) char smem_dyn[];
  __shared__ ColSh cs[K];
  __shared__ double thr_cur[K];
  __shared__ double sh_push[K], sh_d[K];
  __shared__ unsigned long long sh_np[K], sh_nn[K], sh_et[K];
  __shared__ unsigned long long sh_tile[3];
  __shared__ int sh_any;
  __shared__ double sh_hub[(NT / 32) * K];
  __shared__ int sh_flag;
  __shared__ uint32_t sh_nlong;
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
      if (sh_any) sh_tile[0] = atomicAdd(&ctl->ticket[buf], 1u);
      sh_nlong = 0;
      if constexpr (K >= WIDE_K) *wide_long_count<K>(smem_dyn) = 0;
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
    // Tiles in ticket (= id) order; the next ticket is fetched one tile ahead
    // and the next descriptor is loaded inside the current tile.
    unsigned long long j = sh_tile[0];
    TileDesc d = P.desc[j < P.ntiles ? j : 0];
    for (uint32_t it = 0;; ++it) {
      if (j >= P.ntiles) break;
      if (tid == 0) sh_tile[(it + 1) & 1] = atomicAdd(&ctl->ticket[buf], 1u);
      TileDesc dn = d;
      if (d.npieces > 1) {
        hub_piece<K, MODE>(P, d, j, sh_hub, &sh_flag, cs, thr_cur, yg, rcur, rnxt, ynxt, a);
        dn = P.desc[sh_tile[(it + 1) & 1] < P.ntiles ? sh_tile[(it + 1) & 1] : 0];
        __syncthreads();
      } else if constexpr (K >= WIDE_K) {
        tile_rows_wide<K, MODE>(P, d, smem_dyn, cs, thr_cur, yg, rcur, rnxt, ynxt, a, ba,
                                &sh_nlong, &sh_tile[(it + 1) & 1], &dn);
      } else {
        tile_rows<K, MODE>(P, d, smem_dyn, cs, thr_cur, yg, rcur, rnxt, ynxt, a, ba, &sh_nlong,
                           &sh_tile[(it + 1) & 1], &dn);
      }
      j = sh_tile[(it + 1) & 1];
      d = dn;
    }
    source_rows<K, MODE>(P, cs, thr_cur, yg, rcur, rnxt, ynxt, a);
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
    grid_barrier2(&ctl->gbar, ++gen);
    // every block derives the identical next state from the reduced buffers
    if (tid < K) {
      const int cc = tid;
      if (!cs[cc].done) {
        const double pushed = __ldcg(&ctl->pushed[buf][cc]);
        const unsigned long long np = __ldcg(&ctl->npush[buf][cc]);
        cs[cc].sweeps += 1;
        cs[cc].pushes += np;
        cs[cc].D = __ldcg(&ctl->dsum[buf][cc]);
        if (P.trace && cc == 0 && blockIdx.x == 0 && sweep < P.trace_cap) {
          unsigned long long t;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
          const double rs = MODE == M_POWERPUSH ? cs[cc].r_sum - P.alpha * pushed : pushed;
          P.trace[sweep] = TracePoint{cs[cc].pushes, rs, t};
        }
        if (MODE == M_POWERPUSH) {
          cs[cc].r_sum -= P.alpha * pushed;
          if (np == 0) cs[cc].epoch += 1;  // fixpoint: nothing active at this threshold
          else if (cs[cc].epoch == P.E - 1 && np < P.handoff_np) cs[cc].epoch += 1;  // refine tail
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
  if (MODE == M_POWERPUSH && P.npeers) __threadfence_system();  // peer y stores performed
  if (blockIdx.x == 0 && tid < K) {
    ctl->out_rsum[tid] = cs[tid].r_sum;
    ctl->out_D[tid] = cs[tid].D;
    ctl->out_sweeps[tid] = cs[tid].sweeps;
    ctl->out_done[tid] = cs[tid].done;
    ctl->out_epoch[tid] = cs[tid].epoch;
    ctl->out_pushes[tid] = cs[tid].pushes;
  }
}

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
// Entries with more than HEAVY_DEG out-edges are queued for k_frontier_heavy,
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

// The scatter of heavy entries, one thread per out-edge over all of them.
__global__ void __launch_bounds__(256) k_frontier_heavy(const __grid_constant__ FrontierParams P,
                                                        const HeavyEntry* heavy,
                                                        const unsigned long long* prefix,
                                                        unsigned nheavy, unsigned long long total) {
  for (unsigned long long e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
       e - threadIdx.x < total; e += (uint64_t)gridDim.x * blockDim.x) {
    const bool ok = e < total;
    uint32_t t = 0;
    int c = 0;
    double share = 0.0;
    if (ok) {
      unsigned lo = 0, hi = nheavy;  // last h with prefix[h] <= e
      while (lo + 1 < hi) {
        const unsigned mid = (lo + hi) >> 1;
        if (prefix[mid] <= e) lo = mid; else hi = mid;
      }
      const HeavyEntry h = heavy[lo];
      c = (int)h.c;
      share = h.share;
      t = __ldg(P.nbr + h.begin + (e - prefix[lo]));
    }
    // all lanes of a ballot group must share the column: group by column
    const unsigned same = __match_any_sync(0xffffffffu, ok ? c : -1);
    if (ok) relax_scatter(P, t, c, share, true, same);
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

inline uint32_t tile_edges(int K) { return K >= WIDE_K ? WIDE_T : (uint32_t)(SWEEP_ELEMS / K); }
inline uint32_t tile_rmax(int K) {
  if (K >= WIDE_K) return RMAX_W;
  const int T = SWEEP_ELEMS / K;
  return T < 256 ? T : 256;
}

// ---- per-graph workspace --------------------------------------------------
struct Workspace {
  int K = 0;
  uint64_t n = 0;
  DevBuf<double> x, y0, y1, r0, r1, res;
  DevBuf<unsigned> stamp;
  DevBuf<uint32_t> fa, fb;  // frontier segments [K][n] of node ids
  DevBuf<double> carry_h, carry_t;
  DevBuf<unsigned> split_cnt;
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
  DevBuf<SweepCtl> ctl;
  DevBuf<unsigned long long> counters;  // next_cnt + col_cnt[K] + col_np[K] + col_nn[K]
  DevBuf<double> dcols;                 // col_dr[K], colsum[K], D[K]
  DevBuf<uint32_t> d_src;
  DevBuf<HeavyEntry> heavy;
  DevBuf<unsigned> heavy_cnt;
  DevBuf<unsigned> col_stop;
  DevBuf<unsigned long long> heavy_prefix;
  unsigned level_tag = 0;
  uint64_t ntiles_alloc = 0;
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
  PPRG_CUDA(cudaMemsetAsync(w.stamp.get(), 0, 4 * nk, g.stream));
  w.fa.alloc(nk + 1);
  w.fb.alloc(nk + 1);
  w.ctl.alloc(1);
  w.counters.alloc(1 + 5 * KMAX);
  w.col_stop.alloc(KMAX);
  w.dcols.alloc(3 * KMAX);
  w.d_src.alloc(KMAX);
  w.heavy.alloc((g.m / HEAVY_DEG + 1) * (uint64_t)K + 1);
  w.heavy_cnt.alloc(1);
}

static void ws_tiles(Workspace& w, Graph& g, uint64_t ntiles, uint64_t nhubs) {
  const int K = w.K;
  if (ntiles > w.ntiles_alloc) {
    w.carry_h.alloc((ntiles + 1) * K);
    w.carry_t.alloc((ntiles + 1) * K);
    w.split_cnt.alloc(ntiles + 1);
    PPRG_CUDA(cudaMemsetAsync(w.split_cnt.get(), 0, 4 * (ntiles + 1), g.stream));
    w.ntiles_alloc = ntiles;
  }
  if ((ntiles + 1) * K > w.hub_acc.n) w.hub_acc.alloc((ntiles + 1) * K);
  if (nhubs + 1 > w.hub_cnt.n) {
    w.hub_cnt.alloc(nhubs + 1);
    PPRG_CUDA(cudaMemsetAsync(w.hub_cnt.get(), 0, 4 * (nhubs + 1), g.stream));
  }
}

static Workspace& workspace(Graph& g, int K, uint64_t ntiles, uint64_t nhubs) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  auto& slot = g_ws[&g][K];
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

template <int K, int MODE>
void launch_sweeps(Graph& g, SweepParams& P, bool cooperative) {

  const size_t wide_bytes = 8ull * (RMAX_W + 1) + 8ull * RMAX_W + 8ull * (NT / 32) * K +
                            4ull * (3 * RMAX_W + 1) + 16;
  const size_t smem = K >= WIDE_K ? wide_bytes : Tile<K>::bytes;
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
  k_stamp<<<1, 1, 0, g.stream>>>(t.get());
  unsigned long long h = 0;
  PPRG_CUDA(cudaMemcpyAsync(&h, t.get(), 8, cudaMemcpyDeviceToHost, g.stream));
  PPRG_CUDA(cudaStreamSynchronize(g.stream));
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

void d2h_small(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (!bytes) return;
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
  const TileDesc* desc = nullptr;
  uint64_t nhubs = 0;
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

Block make_block(Graph& g, const uint32_t* sources, uint32_t k, double alpha, bool need_pull,
                 Workspace* own = nullptr) {
  const int K = round_k(k);
  uint64_t ntiles = 0;
  const uint32_t* tl = nullptr;
  const TileDesc* dsc = nullptr;
  uint64_t nhubs = 0;
  if (need_pull) {
    const Graph::Plan& pl = g.tile_plan(tile_edges(K), tile_rmax(K));
    dsc = pl.tiles.get();
    ntiles = pl.ntiles;
    nhubs = pl.nhubs;
  }
  if (own) {
    if (!own->K) ws_alloc(*own, g, K);
    ws_tiles(*own, g, ntiles, nhubs);
  }
  Workspace& w = own ? *own : workspace(g, K, ntiles, nhubs);
  Block b(g, w, K, k, alpha);
  b.ntiles = ntiles;
  b.tile_lo = tl;
  b.desc = dsc;
  b.nhubs = nhubs;
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
  P.own_lo = 0;
  P.own_hi = g.n;
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
  P.hub_acc = b.w.hub_acc.get();
  P.hub_cnt = b.w.hub_cnt.get();
  return P;
}

// Observed calls: column 0's reserve / residue (device, interleaved with the
// block's K) to the host sink.
void emit_step(Block& b, const double* reserve_src, double reserve_scale, const double* residue_src,
               double r_sum, uint64_t pushes) {
  if (!g_obs) return;
  Graph& g = b.g;
  const uint64_t n = g.n, nk = n * (uint64_t)b.K;
  cudaStream_t st = g.stream;
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
  F.seg_cap = n;
  F.limit = limit == UINT64_MAX ? ~0ull : (unsigned long long)limit;
  for (int c = 0; c < K; ++c) {
    F.src[c] = b.src[c];
    F.thr[c] = r_max;
  }
  const int NC = 1 + 5 * KMAX;
  unsigned long long* col_cnt = w.counters.get() + 1;
  unsigned long long* col_np = col_cnt + KMAX;
  unsigned long long* col_nn = col_np + KMAX;
  double* col_dr = w.dcols.get();
  unsigned* d_stop = w.col_stop.get();
  uint32_t* cur = w.fa.get();
  uint32_t* nxt = w.fb.get();
  std::vector<uint64_t> qsize(K, 0);
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
                                                live0, w.stamp.get(), next_tag(), cur, n, col_cnt);
    d2h_small(hc.data(), w.counters.get(), 8 * NC, st);
    PPRG_CUDA(cudaStreamSynchronize(st));
    for (int c = 0; c < K; ++c) qsize[c] = hc[1 + c];
    call->kernel_launches += 1;
  } else {
    std::vector<uint32_t> hdeg(K);
    for (int c = 0; c < K; ++c)
      d2h_small(&hdeg[c], g.deg.get() + b.src[c], 4, st);
    PPRG_CUDA(cudaStreamSynchronize(st));
    for (uint32_t c = 0; c < b.k; ++c)  // seed_source, push.cpp:61-66
      if (state[c] == 0 && 1.0 > (double)(hdeg[c] ? hdeg[c] : 1) * r_max) {
        PPRG_CUDA(cudaMemcpyAsync(cur + (uint64_t)c * n, &b.src[c], 4, cudaMemcpyHostToDevice, st));
        qsize[c] = 1;
      }
  }
  std::vector<double> hdr(KMAX);
  std::vector<unsigned> hstop(KMAX);
  unsigned long long live = 0;
  auto still_live = [&](uint32_t c, uint64_t queued) {
    return queued > 0 && queued <= limit && !(lam_stop > 0 && b.r_sum[c] <= lam_stop);
  };
  for (uint32_t c = 0; c < b.k; ++c) {
    if (state[c] != 0) continue;
    if (still_live(c, qsize[c])) live |= 1ull << c;
    else state[c] = 1;
  }
  while (live) {
    uint64_t total = 0;
    for (int c = 0; c < K; ++c) {
      F.pre[c] = total;
      total += ((live >> c) & 1ull) ? qsize[c] : 0;
    }
    F.pre[K] = total;
    for (int c = K + 1; c <= KMAX; ++c) F.pre[c] = total;
    if (!total) break;
    PPRG_CUDA(cudaMemsetAsync(w.counters.get(), 0, 8 * NC, st));
    PPRG_CUDA(cudaMemsetAsync(col_dr, 0, 8 * KMAX, st));
    PPRG_CUDA(cudaMemsetAsync(d_stop, 0, 4 * KMAX, st));
    PPRG_CUDA(cudaMemsetAsync(w.heavy_cnt.get(), 0, 4, st));
    // the segments of the live columns are read in place (pre[] skips the others)
    F.cur = cur;
    F.next = nxt;
    F.total = total;
    F.col_cnt = col_cnt;
    F.col_dr = col_dr;
    F.col_np = col_np;
    F.col_nn = col_nn;
    F.col_stop = d_stop;
    F.col_resv = col_nn + KMAX;
    F.col_live = live;
    F.level_tag = next_tag();
    // live columns are contiguous in pre[] but their segments sit at c*n: the
    // kernel maps (c, pos) -> cur[c*n + pos]
    k_frontier<<<grid_for(total * 32), 256, 0, st>>>(F, w.heavy.get(), w.heavy_cnt.get());
    PPRG_CUDA(cudaGetLastError());
    call->kernel_launches += 1;
    unsigned nheavy = 0;
    d2h_small(&nheavy, w.heavy_cnt.get(), 4, st);
    PPRG_CUDA(cudaStreamSynchronize(st));
    if (nheavy) {
      std::vector<HeavyEntry> hv(nheavy);
      d2h_small(hv.data(), w.heavy.get(), sizeof(HeavyEntry) * nheavy, st);
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
    d2h_small(hc.data(), w.counters.get(), 8 * NC, st);
    d2h_small(hdr.data(), col_dr, 8 * KMAX, st);
    d2h_small(hstop.data(), d_stop, 4 * KMAX, st);
    PPRG_CUDA(cudaStreamSynchronize(st));
    if (std::getenv("PPRG_DEBUG_LOCAL")) {
      unsigned long long nn = 0, np = 0, app = 0;
      for (uint32_t c = 0; c < b.k; ++c) nn += hc[1 + 2 * KMAX + c], np += hc[1 + KMAX + c], app += hc[1 + c];
      std::fprintf(stderr, "level: entries %llu heavy %u node_pushes %llu edge_pushes %llu appended %llu\n",
                   (unsigned long long)total, nheavy, nn, np, app);
    }
    const bool observed_col0 = g_obs && (live & 1ull);
    for (uint32_t c = 0; c < b.k; ++c) {
      if (!((live >> c) & 1ull)) continue;
      b.r_sum[c] -= hdr[c];
      b.pushes[c] += hc[1 + KMAX + c];
      b.levels[c] += 1;
      if (g_trace && c == 0)
        g_trace->pts.push_back(TracePoint{b.pushes[0], b.r_sum[0], host_now_ns() - g_trace->host_t0});
      qsize[c] = hc[1 + c];
      if (hstop[c] || !still_live(c, qsize[c])) {
        live &= ~(1ull << c);
        state[c] = 1;
      }
    }
    if (observed_col0) emit_step(b, w.x.get(), b.alpha, w.res.get(), b.r_sum[0], b.pushes[0]);
    std::swap(cur, nxt);
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
  k_colsum<<<grid_reduce(nk), 256, 0, st>>>(b.w.res.get(), g.n, b.K, b.w.dcols.get() + KMAX);
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

// Global phase: epochs of asynchronous pull sweeps in one persistent
// cooperative kernel (push.cpp:168-197) for the columns with scan[c] set.
// refine_rmax > 0 appends a refine epoch (push.cpp:208-222): threshold
// refine_rmax, no r_sum target, ends at the sweep that pushes nothing — the
// fixpoint where every residue is <= deg_eff * refine_rmax, refine's postcondition.
void global_phase(Block& b, double lambda, uint32_t E, CallStats* call, double refine_rmax = 0.0) {
  Graph& g = b.g;
  Workspace& w = b.w;
  cudaStream_t st = g.stream;
  const uint64_t nk = g.n * (uint64_t)b.K;
  const double m_eff = (double)g.m_eff();
  if (E + (refine_rmax > 0.0) > EMAX) fail(EINVAL_, "epoch_num exceeds 64");
  PPRG_CUDA(cudaMemsetAsync(w.dcols.get() + 2 * KMAX, 0, 8 * KMAX, st));
  k_init_pull<<<grid_reduce(nk), 256, 0, st>>>(w.x.get(), g.deg.get(), g.inv_deg.get(), g.n, b.K,
                                            b.alpha, w.y0.get(), w.dcols.get() + 2 * KMAX);
  d2h_small(b.D.data(), w.dcols.get() + 2 * KMAX, 8 * KMAX, st);
  PPRG_CUDA(cudaMemsetAsync(w.ctl.get(), 0, sizeof(SweepCtl), st));
  PPRG_CUDA(cudaStreamSynchronize(st));
  SweepParams P = base_params(b);
  for (uint32_t e = 0; e < E; ++e) {
    const double el = std::pow(lambda, static_cast<double>(e + 1) / E);  // push.cpp:176-178
    P.lam[e] = el;
    P.thr[e] = el / m_eff;
  }
  const int Et = (int)E + (refine_rmax > 0.0);
  if (refine_rmax > 0.0) {
    P.lam[E] = -1.0;
    P.thr[E] = refine_rmax;
    // a sweep costs a pass over every in-edge; once the refine tail pushes
    // fewer than m_eff/64 edges per sweep the frontier kernels finish it
    double f = 1.0 / 64;
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
  P.y[0] = P.y[1] = w.y0.get();
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
      for (int c = 0; c < b.K; ++c) Q.init[c] = stv[c];
      PPRG_CUDA(cudaMemsetAsync(w.ctl.get(), 0, sizeof(SweepCtl), st));
      dispatch_sweeps<M_POWERPUSH>(g, b.K, Q, true);
      SweepCtl one;
      d2h_small(&one, w.ctl.get(), sizeof one, st);
      PPRG_CUDA(cudaStreamSynchronize(st));
      hc.alg_bytes += one.alg_bytes;
      hc.total_sweeps = sweep + 1;
      for (int c = 0; c < b.K; ++c)
        stv[c] = ColInit{one.out_rsum[c], one.out_D[c], one.out_epoch[c], one.out_done[c],
                         one.out_sweeps[c], one.out_pushes[c]};
      // explicit residues of the pull form (the final pass, outputs only)
      SweepParams F = base_params(b);
      F.x = w.x.get();
      F.y[0] = F.y[1] = w.y0.get();
      F.push_res = w.res.get();
      F.out_reserve = snap.get();
      F.out_residue = snap.get() + g.n;
      for (int c = 0; c < b.K; ++c) {
        F.final_pull[c] = 1;
        F.init[c].r_sum = stv[c].r_sum;
        F.init[c].D = stv[c].D;
      }
      PPRG_CUDA(cudaMemsetAsync(snap.get(), 0, 16 * g.n, st));
      PPRG_CUDA(cudaMemsetAsync(w.ctl.get(), 0, sizeof(SweepCtl), st));
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
  } else {
    tm.start();
    dispatch_sweeps<M_POWERPUSH>(g, b.K, P, true);
    tm.stop();
    d2h_small(&hc, w.ctl.get(), sizeof hc, st);
  }
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
  EventTimer tf(st);
  tf.start();
  dispatch_sweeps<M_FINAL>(g, b.K, Q, true);
  tf.stop();
  call->kernel_launches += 1;
  SweepCtl fc;
  d2h_small(&fc, w.ctl.get(), sizeof fc, st);
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
    const double exact = fc.pushed[0][c];
    if (std::fabs(exact - b.r_sum[c]) > 1e-6)
      fail(EINTERNAL, "push: r_sum drifted more than 1e-6 from the residues");
    b.r_sum[c] = exact;
  }
}

void power_push_block(Block& b, double lambda, uint32_t epoch_num, int64_t scan_threshold,
                      CallStats* call, double refine_rmax = 0.0) {
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
  EventTimer tl(st);
  tl.start();
  drain_levels(b, r_max, lambda, limit, false, state, call);
  std::vector<int> all(KMAX, 1);
  exact_rsum(b, all);
  tl.stop();
  call->local_ms += tl.ms();
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
  std::lock_guard<std::mutex> lk(g.mu);
  if (!(r_max > 0.0)) fail(EINVAL_, "refine: r_max must be positive");  // push.cpp:210
  for (uint32_t c = 0; c < k; ++c)
    if (sources[c] >= g.n) fail(EINVAL_, "source out of range");
  const uint64_t n = g.n;
  for (uint32_t b0 = 0; b0 < k; b0 += KMAX) {
    const uint32_t kb = k - b0 < (uint32_t)KMAX ? k - b0 : (uint32_t)KMAX;
    Block b = make_block(g, sources + b0, kb, alpha, false);
    cudaStream_t st = g.stream;
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
    std::vector<int> all(KMAX, 1);
    std::fill(b.r_sum.begin(), b.r_sum.end(), 0.0);
    {  // r_sum of the incoming state (no drift check: it is the caller's)
      PPRG_CUDA(cudaMemsetAsync(b.w.dcols.get() + KMAX, 0, 8 * KMAX, st));
      k_colsum<<<grid_reduce(nk), 256, 0, st>>>(b.w.res.get(), n, b.K, b.w.dcols.get() + KMAX);
      d2h_small(b.r_sum.data(), b.w.dcols.get() + KMAX, 8 * KMAX, st);
      PPRG_CUDA(cudaStreamSynchronize(st));
    }
    std::vector<int> state(KMAX, 2);
    for (uint32_t c = 0; c < kb; ++c) state[c] = 0;
    EventTimer tl(st);
    tl.start();
    drain_levels(b, r_max, 0.0, UINT64_MAX, true, state, call);
    exact_rsum(b, all);  // push.cpp:221
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
      k_init_pull<<<grid_reduce(nk), 256, 0, st>>>(w.r0.get(), g.deg.get(), g.inv_deg.get(), n, b.K,
                                                alpha, w.y0.get(), w.dcols.get() + 2 * KMAX);
      d2h_small(b.D.data(), w.dcols.get() + 2 * KMAX, 8 * KMAX, st);
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
          PPRG_CUDA(cudaMemsetAsync(w.ctl.get(), 0, sizeof(SweepCtl), st));
          if (eng == Engine::PowItr) dispatch_sweeps<M_POWITR>(g, b.K, Q, true);
          else dispatch_sweeps<M_SIMFWD>(g, b.K, Q, true);
          SweepCtl one;
          d2h_small(&one, w.ctl.get(), sizeof one, st);
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
        d2h_small(&hc, w.ctl.get(), sizeof hc, st);
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
    if (b0 + kb >= k) sync_host_copies(g);
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
  // PowerPush to lambda, then refine (push.cpp:208-222) as a final sweep
  // epoch at r_max run to its fixpoint, so the refine is pull sweeps over the
  // tile plan rather than a scattered frontier over millions of nodes.
  power_push_block(b, lambda, 8, -1, call, r_max);
  Outputs none;
  finalize(b, none, true, call);
  // the tail: every node still above deg_eff * r_max in id order, drained
  std::vector<int> state(KMAX, 2);
  for (uint32_t c = 0; c < k; ++c) state[c] = 0;
  EventTimer tl(g.stream);
  tl.start();
  drain_levels(b, r_max, 0.0, UINT64_MAX, true, state, call);
  std::vector<int> all(KMAX, 1);
  exact_rsum(b, all);
  tl.stop();
  call->local_ms += tl.ms();
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
  std::lock_guard<std::mutex> lk(g.mu);
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
  const Graph::Plan& pl = g.tile_plan(tile_edges(K), tile_rmax(K));
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
  cudaStream_t st = g.stream;
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
  std::lock_guard<std::mutex> lk(g.mu);
  Block& b = *s->b;
  const int K = b.K;
  const double m_eff = (double)g.m_eff();
  s->lam.assign(EMAX, 0.0);
  s->thr.assign(EMAX, 0.0);
  for (uint32_t e = 0; e < s->E; ++e) {
    s->lam[e] = std::pow(s->lambda, static_cast<double>(e + 1) / s->E);  // push.cpp:176-178
    s->thr[e] = s->lam[e] / m_eff;
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
    k_part_y<<<grid_for((s->hi - s->lo) * K), 256, 0, g.stream>>>(b.w.x.get(), g.inv_deg.get(), s->lo,
                                                                  s->hi, K, b.alpha, b.w.y0.get(), ps);
  PPRG_CUDA(cudaGetLastError());
  PPRG_CUDA(cudaStreamSynchronize(g.stream));
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
  std::lock_guard<std::mutex> lk(g.mu);
  Block& b = *s->b;
  const int K = b.K;
  SweepParams P = part_params(s);
  P.max_sweeps = 1;
  P.E = (int)s->E;
  for (uint32_t e = 0; e < s->E; ++e) {
    P.lam[e] = s->lam[e];
    P.thr[e] = s->thr[e];
  }
  cudaStream_t st = g.stream;
  PPRG_CUDA(cudaMemsetAsync(b.w.ctl.get(), 0, sizeof(SweepCtl), st));
  EventTimer tm(st);
  tm.start();
  dispatch_sweeps<M_POWERPUSH>(g, K, P, true);
  tm.stop();
  k_pack_counters<<<1, KMAX, 0, st>>>(b.w.ctl.get(), K, s->counters.get());
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
  std::lock_guard<std::mutex> lk(g.mu);
  Block& b = *s->b;
  cudaStream_t st = g.stream;
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
  PPRG_CUDA(cudaMemsetAsync(b.w.ctl.get(), 0, sizeof(SweepCtl), st));
  EventTimer tf(st);
  tf.start();
  dispatch_sweeps<M_FINAL>(g, b.K, Q, true);
  tf.stop();
  SweepCtl fc;
  d2h_small(&fc, b.w.ctl.get(), sizeof fc, st);
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
int part_device(const PartSession* s) { return s->g->device; }

void part_destroy(PartSession* s) {
  if (!s) return;
  DeviceGuard dg(s->g->device);
  delete s;
}

}  // namespace pprg
