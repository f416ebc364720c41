// Device side of the global sweeps: the persistent k_sweeps<K, MODE> kernel
// (PowerPush epochs, PowItr / SimFwdPush iterations, the final residue pass)
// and its tile / row machinery. Included by push.cu only (one translation unit).
#pragma once
#include <cub/cub.cuh>
#include <math_constants.h>

#include <cstdint>

#include "internal.h"

namespace pprg {

constexpr int KMAX = 64;
constexpr int EMAX = 64;   // max epochs
constexpr int WMAX = 16;   // max waves of a deterministic sweep
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
thread_local bool t_det = false;

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
  // final pass: implicit residues below zero (rounding of inflow - x only;
  // clamped to 0 in the outputs, counted and summed here and checked on the host)
  unsigned long long neg_count;
  double neg_sum;
  double out_scale[KMAX];              // final pass: pushed[0][c] / out_scale[c] = residue sum
  unsigned wticket[3][WMAX];           // deterministic sweeps: tile ticket of each wave
  int out_scan[KMAX];                  // column ran the global phase (push.cpp:168)
  unsigned wdone[3][64];               // delta sweeps: finished tiles of each wave
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
  const TileDesc* desc;        // row-aligned tile plan
  double* hub_acc;             // [ntiles][K] per-piece partial sums of hub rows
  unsigned* hub_cnt;           // [nhubs] arrived pieces
  uint64_t ntiles;
  uint32_t T;
  int k_live;  // real columns (<= K)
  int k1w;     // K = 1: warp tasks (sweep_k1_warps) instead of block tiles
  int E;
  double alpha;
  double lambda;               // powitr termination
  double* x;                   // powerpush state / powitr reserve
  double* y[2];                // gather operand (powitr double-buffers)
  double* r[2];                // powitr residues (double-buffered)
  const double* push_res;      // finalize: push-form residues (columns without scan phase)
  const double* D_dev;         // if set: each column's initial D on the device (else init[].D)
  // Device-decided starts (no host round trip between the phases of a block):
  // from_drain: the global phase takes each column's r_sum from the local
  // phase's exact sum and decides scan / epoch / done itself (push.cpp:168,
  // 176-180: scan iff r_sum > scan_lambda, or every column with scan_all);
  // from_sweeps: the final pass takes r_sum, D and the scan flag from the
  // global phase's outputs.
  const double* from_drain;    // [KMAX] exact r_sum after the local phase
  const SweepCtl* from_sweeps;
  double scan_lambda;
  int scan_all;

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
  // deterministic sweeps: the tile list cut into nwaves waves of contiguous
  // rows; wave w = tiles [wave_tile[w], wave_tile[w+1]), whose rows start at
  // node wave_node[w]
  uint32_t nwaves;
  uint64_t wave_tile[WMAX + 1];
  uint32_t wave_node[WMAX];
  uint32_t src[KMAX];
  int final_pull[KMAX];        // finalize: 1 = residue from pull form
  double thr[EMAX];            // epoch r_max (lambda is per call, so shared by columns)
  double lam[EMAX];            // epoch lambda
  ColInit init[KMAX];
};

// (56 bytes = 14 words: lanes reading cs[c] for 32 different columns meet at
// most 2-way shared bank conflicts; a 64-byte stride would make them 16-way)
struct ColSh {
  double r_sum, D;
  double scp, scd;  // deterministic sweeps: fixed-point scales 2^S of this sweep's pushed / D sums
  int epoch;
  short done;
  short pull;  // final pass: residue from the pull form (the column ran the global phase)
  unsigned sweeps;
  uint32_t src;  // the column's source (a shared copy: P.src[c] with a per-lane c
                 // would be a divergent, serialised constant-bank load)
  unsigned long long pushes;
};

static_assert(sizeof(ColSh) == 56, "ColSh stride");

// Gather operand of a sweep. Fast mode: one y, updated in place (rows read
// whatever value a neighbour's row has when the gather lands). Deterministic
// sweeps: rows of the earlier waves of this sweep are read from this sweep's
// buffer yn, every other row from the previous sweep's yo, so no inflow
// depends on timing.
struct YG {
  const double* yo;
  const double* yn;
  uint32_t lo;  // first node of the current wave
};
template <bool DET>
__device__ __forceinline__ const double* ysrc(const YG& y, uint32_t id) {
  if constexpr (DET) return id < y.lo ? y.yn : y.yo;
  else return y.yo;
}
// One term of a per-column sum. Deterministic sweeps sum integers (term *
// 2^S rounded, exact in fp64 while every partial sum stays below 2^53), so
// the fp64 atomics that combine them give the same bits in any order.
template <bool DET>
__device__ __forceinline__ double qterm(double v, double sc) {
  if constexpr (DET) return rint(v * sc);
  else return v;
}

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
  // two-columns-per-lane decisions (K = 32, 64): node pushes and edge pushes
  // packed into one 64-bit add (nn << 40 | np; per block and sweep np < 2^40 and
  // nn < 2^24, since n <= 6.2M at these widths), and dead-end pushes counted
  // separately (et = np - dead) - one 64-bit shared atomic (a CAS loop on
  // sm_100) per push instead of three
  unsigned long long* pk;
  unsigned* nd;
};
constexpr int PK_SHIFT = 40;
#ifndef PPRG_PUSH_REG
#define PPRG_PUSH_REG 1
#endif

// The per-(row, column) decision: push form of push.cpp:182-193 in pull
// representation, the PowItr update of push.cpp:90-99, or the final explicit
// residue. `acc` is the sum over in-neighbours v of y_v.
template <int K, int MODE, bool DET>
__device__ __forceinline__ void decide(const SweepParams& P, const ColSh* cs, const double* thr_cur,
                                       uint32_t u, int c, double acc, double xo, double rc,
                                       uint32_t dg, double inv, const YG& yg, double* rnxt,
                                       double* ynxt, Acc& a) {
  const uint64_t ix = (uint64_t)u * K + c;
  const bool is_src = u == cs[c].src;
  const double alpha = P.alpha, oma = 1.0 - P.alpha;
  if constexpr (MODE == M_POWERPUSH) {
    if (cs[c].done) {
      if (DET && dg) ynxt[ix] = oma * xo * inv;  // every row's y into this sweep's buffer
      return;
    }
    const double inflow = acc + (is_src ? 1.0 + cs[c].D : 0.0);
    const double r = inflow - xo;
    if (r > (dg ? (double)dg : 1.0) * thr_cur[c]) {
      st_state(P.x + ix, inflow);
      if (!DET && dg) {
        const double yv = oma * inflow * inv;
        P.y[0][ix] = yv;
        for (int p = 0; p < P.npeers; ++p) P.peer_y[p][ix] = yv;  // fused exchange
      }
      a.push += qterm<DET>(r, cs[c].scp);
      a.np += dg ? dg : 1;
      a.nn += 1;
      a.et += dg;
      xo = inflow;
    }
    if (DET && dg) ynxt[ix] = oma * xo * inv;  // the same bits as the pushed value
    if (!dg) a.d += qterm<DET>(oma * xo, cs[c].scd);
  } else if constexpr (MODE == M_POWITR || MODE == M_SIMFWD) {
    if (cs[c].done) {
      rnxt[ix] = rc;
      ynxt[ix] = __ldcg(yg.yo + ix);
      return;
    }
    const double nxt = acc + (is_src ? cs[c].D : 0.0);
    P.x[ix] = xo + alpha * rc;  // reserve += alpha * r
    rnxt[ix] = nxt;
    ynxt[ix] = oma * nxt * inv;
    a.push += qterm<DET>(nxt, cs[c].scp);  // sum of next = the exact r_sum (push.cpp:101-103)
    if (MODE == M_POWITR || rc != 0.0) {
      a.np += dg ? dg : 1;
      a.nn += 1;
      a.et += dg;
    }
    if (!dg) a.d += qterm<DET>(oma * nxt, cs[c].scd);
  } else {  // M_FINAL
    double res;
    if (cs[c].pull) {
      const double inflow = acc + (is_src ? 1.0 + cs[c].D : 0.0);
      res = inflow - xo;
      if (res < 0.0) {  // rounding of the implicit form only: counted, checked on the host
        atomicAdd(&P.ctl->neg_count, 1ull);
        atomicAdd(&P.ctl->neg_sum, res);
        res = 0.0;
      }
    } else {
      res = P.push_res[ix];
    }
    if (P.res_inter) P.res_inter[ix] = res;
    if (c < P.k_live) {
      if (P.out_reserve) P.out_reserve[(uint64_t)c * P.n + u] = alpha * xo;
      if (P.out_residue) P.out_residue[(uint64_t)c * P.n + u] = res;
    }
    a.push += qterm<DET>(res, cs[c].scp);
  }
}

template <int K, int MODE, bool DET>
__device__ __forceinline__ void decide_at(const SweepParams& P, const ColSh* cs,
                                          const double* thr_cur, uint32_t u, int c, double acc,
                                          uint32_t dg, double inv, const YG& yg,
                                          const double* rcur, double* rnxt, double* ynxt, Acc& a) {
  const uint64_t ix = (uint64_t)u * K + c;
  decide<K, MODE, DET>(P, cs, thr_cur, u, c, acc, __ldcg(P.x + ix),
                  (MODE == M_POWITR || MODE == M_SIMFWD) ? __ldcg(rcur + ix) : 0.0, dg, inv, yg,
                  rnxt, ynxt, a);
}

// One piece of a hub row (more in-edges than a tile holds): the block sums its
// edges per column, adds the piece total into the row's accumulator, and the
// last piece to arrive decides the row (acq_rel counter: each piece releases
// its partial, the last arriver acquires all of them before the block barrier
// hands them to the deciding threads; partials read back from L2). Only hub
// pieces pay this protocol.
template <int K, int MODE, bool DET>
__device__ __noinline__ void hub_piece(const SweepParams& P, const TileDesc& d, uint64_t j,
                                       double* hubsh, int* flag, const ColSh* cs, const double* thr_cur,
                                       const YG& yg, const double* rcur, double* rnxt,
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
    s0 += ysrc<DET>(yg, i0)[(uint64_t)i0 * K + c];
    s1 += ysrc<DET>(yg, i1)[(uint64_t)i1 * K + c];
    s2 += ysrc<DET>(yg, i2)[(uint64_t)i2 * K + c];
    s3 += ysrc<DET>(yg, i3)[(uint64_t)i3 * K + c];
  }
  for (; f < total; f += NT) {
    const uint32_t i0 = __ldg(P.in_nbr + d.e0 + f / K);
    s0 += ysrc<DET>(yg, i0)[(uint64_t)i0 * K + c];
  }
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
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
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
    decide_at<K, MODE, DET>(P, cs, thr_cur, u, tid, acc, __ldg(P.cdeg + d.r0), __ldg(P.cinv + d.r0),
                            yg, rcur, rnxt, ynxt, a);
  }
}

// One row-aligned tile: gather y of every in-edge into shared memory (all
// loads of the tile issued together), then one thread per (row, column) sums
// its row and decides; rows longer than LONG are summed by a whole warp.
template <int K, int MODE, bool DET>
__device__ __forceinline__ void tile_rows(const SweepParams& P, const TileDesc& d, char* smem,
                                          const ColSh* cs, const double* thr_cur, const YG& yg,
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
        if (f < total) vals[f] = ysrc<DET>(yg, id[i])[(uint64_t)id[i] * K + (f % K)];
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
    decide<K, MODE, DET>(P, cs, thr_cur, u, c, s0 + s1, xo, rc, sdeg[r], sinv[r], yg, rnxt, ynxt, a);
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
          decide_at<K, MODE, DET>(P, cs, thr_cur, snode[r], kc, s[0], sdeg[r], sinv[r], yg, rcur,
                                  rnxt, ynxt, a);
        } else {  // K = 64: lane kc decides columns kc and kc+32; counters via shared atomics
#pragma unroll
          for (int q = 0; q < CPL; ++q) {
            Acc b2;
            const int cc = kc + q * KC;
            decide_at<K, MODE, DET>(P, cs, thr_cur, snode[r], cc, s[q], sdeg[r], sinv[r], yg, rcur,
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

// One-column sweeps (K = 1) by independent warps (PPRG_K1W). The tile plan is
// cut into warp tasks: <= 256 in-edges and <= 64 whole rows, or one whole row
// of <= K1W_H in-edges, or one K1W_H-edge piece of a longer row. Warps take
// tasks in id order, CH at a time from the sweep's ticket (fetched one chunk
// ahead), with no block barrier anywhere; the next task's descriptor is
// loaded one ahead. Per 256-edge round a task's in-edge ids (8 per lane,
// coalesced) and gathers are issued before its row data (2 rows per lane:
// offset, node, degree, x) is needed; per 32-edge window the row starts are
// OR-reduced into a bit mask, each lane's row key is a popcount of it, and a
// segmented shuffle reduction leaves every row segment's sum in its first
// lane, which adds it into the warp's row accumulator in shared memory.
// Pieces meet through the hub protocol of hub_piece (partial slot,
// release-ordered counter, the last piece sums the partials in piece order).
#ifndef PPRG_K1W
#define PPRG_K1W 1
#endif
#ifndef PPRG_K1W_H
#define PPRG_K1W_H 1024
#endif
#ifndef PPRG_K1W_CH
#define PPRG_K1W_CH 2
#endif
constexpr uint32_t K1W_T = 256;         // packed-task edges (32 lanes x 8 gathers per round)
constexpr uint32_t K1W_R = 64;          // packed-task rows (2 per lane)
constexpr uint32_t K1W_H = PPRG_K1W_H;  // longest whole-row task; longer rows are pieces
constexpr uint32_t K1W_CH = PPRG_K1W_CH;
constexpr size_t k1w_bytes = 8ull * (NT / 32) * K1W_R;

__device__ __forceinline__ uint32_t le_mask(int j) { return 0xFFFFFFFFu >> (31 - j); }

template <int MODE, bool DET>
__device__ __forceinline__ void sweep_k1_warps(const SweepParams& P, const ColSh* cs,
                                               const double* thr_cur, const YG& yg,
                                               const double* rcur, double* rnxt, double* ynxt,
                                               Acc& a, double* sacc_all, unsigned* ticket,
                                               uint64_t t0, uint64_t t1) {
  constexpr int G = K1W_T / 32;
  constexpr bool RC = MODE == M_POWITR || MODE == M_SIMFWD;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* sacc = sacc_all + warp * K1W_R;
  const uint64_t nt = t1;  // tasks [t0, t1)
  auto grab = [&]() -> uint64_t {
    unsigned b = 0;
    if (lane == 0) b = atomicAdd(ticket, K1W_CH);
    return t0 + __shfl_sync(0xffffffffu, b, 0);
  };
  uint64_t base = grab();
  uint64_t nbase = base < nt ? grab() : nt;
  TileDesc d{};
  if (base < nt) d = P.desc[base];
  while (base < nt) {
    for (uint32_t ci = 0; ci < K1W_CH; ++ci) {
      const uint64_t t = base + ci;
      if (t >= nt) break;
      const uint64_t tn = (ci + 1 < K1W_CH && t + 1 < nt) ? t + 1 : nbase;
      TileDesc dn = d;
      if (tn < nt) dn = P.desc[tn];  // next task, one ahead
      if (d.npieces > 1) {  // one piece of a row longer than K1W_H
        double sum = 0.0;
        for (uint32_t rb = 0; rb < d.ne; rb += K1W_T) {
          uint32_t id[G];
          double v[G];
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const uint32_t pe = rb + 32 * g + lane;
            id[g] = pe < d.ne ? ld_stream(P.in_nbr + d.e0 + pe) : 0u;
          }
#pragma unroll
          for (int g = 0; g < G; ++g)
            v[g] = rb + 32 * g + lane < d.ne ? ld_gather(ysrc<DET>(yg, id[g]) + id[g]) : 0.0;
          sum += ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        int last = 0;
        if (lane == 0) {
          P.hub_acc[t] = sum;
          unsigned old;
          asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                       : "=r"(old) : "l"(P.hub_cnt + d.hub) : "memory");
          last = old == d.npieces - 1;
          if (last) P.hub_cnt[d.hub] = 0;
        }
        __syncwarp();  // orders lane 0's acquire before the other lanes' partial reads
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {  // the partials in piece order (lane-strided, then a fixed tree)
          const double* part = P.hub_acc + (t - d.piece);
          double acc = 0.0;
          for (uint32_t p = lane; p < d.npieces; p += 32) acc += __ldcg(part + p);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          if (lane == 0) {
            const uint32_t u = __ldg(P.crow + d.r0);
            decide<1, MODE, DET>(P, cs, thr_cur, u, 0, acc, __ldcg(P.x + u),
                            RC ? __ldcg(rcur + u) : 0.0, __ldg(P.cdeg + d.r0),
                            __ldg(P.cinv + d.r0), yg, rnxt, ynxt, a);
          }
        }
        d = dn;
        continue;
      }
      // rows: lane holds rows lane and lane + 32 of the task
      uint32_t st0 = 0xFFFFFFFFu, st1 = 0xFFFFFFFFu, u0 = 0, u1 = 0, dg0 = 0, dg1 = 0;
      double inv0 = 0.0, inv1 = 0.0, xo0 = 0.0, xo1 = 0.0, rc0 = 0.0, rc1 = 0.0;
      if ((uint32_t)lane < d.nr) {
        const uint64_t r = d.r0 + lane;
        st0 = (uint32_t)(__ldg(P.in_off + r) - d.e0);
        u0 = __ldg(P.crow + r);
        dg0 = __ldg(P.cdeg + r);
        inv0 = __ldg(P.cinv + r);
        xo0 = __ldcg(P.x + u0);
        if constexpr (RC) rc0 = __ldcg(rcur + u0);
      }
      if ((uint32_t)lane + 32 < d.nr) {
        const uint64_t r = d.r0 + lane + 32;
        st1 = (uint32_t)(__ldg(P.in_off + r) - d.e0);
        u1 = __ldg(P.crow + r);
        dg1 = __ldg(P.cdeg + r);
        inv1 = __ldg(P.cinv + r);
        xo1 = __ldcg(P.x + u1);
        if constexpr (RC) rc1 = __ldcg(rcur + u1);
      }
      sacc[lane] = 0.0;
      sacc[lane + 32] = 0.0;
      __syncwarp();
      int before = 0;  // rows started before the window
      for (uint32_t rb = 0; rb < d.ne; rb += K1W_T) {
        uint32_t id[G];
        double v[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const uint32_t pe = rb + 32 * g + lane;
          id[g] = pe < d.ne ? ld_stream(P.in_nbr + d.e0 + pe) : 0u;
        }
#pragma unroll
        for (int g = 0; g < G; ++g)
          v[g] = rb + 32 * g + lane < d.ne ? ld_gather(ysrc<DET>(yg, id[g]) + id[g]) : 0.0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const uint32_t w0 = rb + 32 * g;
          if (w0 >= d.ne) break;  // warp-uniform
          uint32_t bit = 0;
          if (st0 - w0 < 32u) bit |= 1u << (st0 - w0);
          if (st1 - w0 < 32u) bit |= 1u << (st1 - w0);
          const uint32_t M = __reduce_or_sync(0xffffffffu, bit);
          const int key = before - 1 + __popc(M & le_mask(lane));
          double x = v[g];
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const double xn = __shfl_down_sync(0xffffffffu, x, o);
            // lane + o is in my segment iff no row starts in (lane, lane + o]
            if (lane + o < 32 && !(M & le_mask(lane + o) & ~le_mask(lane))) x += xn;
          }
          if (w0 + lane < d.ne && (lane == 0 || ((M >> lane) & 1u))) sacc[key] += x;
          __syncwarp();
          before += __popc(M);
        }
      }
      if ((uint32_t)lane < d.nr)
        decide<1, MODE, DET>(P, cs, thr_cur, u0, 0, sacc[lane], xo0, rc0, dg0, inv0, yg, rnxt, ynxt, a);
      if ((uint32_t)lane + 32 < d.nr)
        decide<1, MODE, DET>(P, cs, thr_cur, u1, 0, sacc[lane + 32], xo1, rc1, dg1, inv1, yg, rnxt,
                             ynxt, a);
      __syncwarp();
      d = dn;
    }
    base = nbase;
    nbase = base < nt ? grab() : nt;
  }
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

// Column lanes of the wide layout: each lane loads CPL = K / KC contiguous
// columns of an in-edge's row. K = 64: 32 lanes x 16 B; K = 32 (PPRG_VEC2):
// 16 lanes x 16 B, two in-edges per warp load instruction (5.5% faster per
// sweep than 32 lanes x 8 B on configs[2]; for K = 4..16 the same split was
// 12-40% slower, so they keep one column per lane).
// Round 2 (PPRG_VEC4, sm_100's 32-byte LDG.E.ENL2.256): K = 64 as 16 lanes x
// 32 B and K = 32 as 8 lanes x 32 B -- two (four) in-edges per warp load
// instruction at the same registers in flight (4 loads of 4 doubles per
// lane). The bare gather over the configs[2] transpose: 2.73 instead of 3.16
// ms per 64-column sweep (profiles/r02_microbench_narrow_k_v2.log).
#ifndef PPRG_VEC2
#define PPRG_VEC2 1
#endif
#ifndef PPRG_VEC4
#define PPRG_VEC4 1
#endif
template <int K>
__host__ __device__ constexpr int wide_kc() {
  return (PPRG_VEC4 && K >= 32) ? K / 4
         : K >= 64              ? 32
         : (PPRG_VEC2 && K == 32) ? 16
                                  : (K < 32 ? K : 32);
}

// Sum of y over the in-edges [b, e) of one row for my columns, by one warp.
// Lanes = ES edge slots x KC column lanes (x CPL contiguous columns). The ids
// of 32 consecutive edges are loaded once, coalesced, and broadcast by shuffle;
// the gathers are then issued G at a time into registers before any add, so
// each warp keeps G row-loads in flight (tail slots re-load the last edge and
// are masked out of the sum).
#ifndef PPRG_G
#define PPRG_G 8
#endif
#ifndef PPRG_G4
#define PPRG_G4 4  // row loads in flight per lane with 32-byte lanes (same registers as 8 x 16 B)
#endif
template <int K, bool DET>
__device__ __forceinline__ void warp_row_sum(const SweepParams& P, const YG& yg, uint64_t b,
                                             uint64_t e, double (&s)[K / wide_kc<K>()],
                                             bool have_first = false, uint32_t first_id = 0) {
  constexpr int KC = wide_kc<K>();
  constexpr int CPL = K / KC;
  constexpr int ES = 32 / KC;
  constexpr int G = CPL == 4 ? PPRG_G4 : PPRG_G;
  constexpr int NA = CPL == 4 ? 1 : 2;  // accumulators per column (register budget)
  const int lane = threadIdx.x & 31, es = lane / KC, kc = lane % KC;
  const double* ybase = yg.yo + kc * CPL;  // (fast mode: one y)
  double acc[CPL][NA];
#pragma unroll
  for (int q = 0; q < CPL; ++q)
#pragma unroll
    for (int t = 0; t < NA; ++t) acc[q][t] = 0.0;
  // the ids of the next 32 in-edges are loaded one chunk ahead, so their
  // latency hides behind this chunk's gathers (rows longer than 32 in-edges)
  uint32_t nextid = have_first ? first_id : (b + lane < e ? ld_stream(P.in_nbr + b + lane) : 0u);
  for (uint64_t p0 = b; p0 < e; p0 += 32) {
    const uint32_t myid = nextid;
    if (p0 + 32 < e) nextid = p0 + 32 + lane < e ? ld_stream(P.in_nbr + p0 + 32 + lane) : 0u;
    const int cnt = e - p0 < 32 ? (int)(e - p0) : 32;
    for (int j0 = 0; j0 < cnt; j0 += G * ES) {
      double v[G][CPL];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int j = j0 + g * ES + es;
        const uint32_t id = __shfl_sync(0xffffffffu, myid, j < cnt ? j : cnt - 1);
        const double* src = (DET ? ysrc<DET>(yg, id) + kc * CPL : ybase) + (uint64_t)id * K;
        if constexpr (CPL == 4) {
          const dbl4 v4 = ld_gather4(src);
#pragma unroll
          for (int q = 0; q < 4; ++q) v[g][q] = v4.v[q];
        } else if constexpr (CPL == 2) {
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
        for (int q = 0; q < CPL; ++q) acc[q][g % NA] += ok ? v[g][q] : 0.0;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < CPL; ++q) {
    s[q] = NA == 2 ? acc[q][0] + acc[q][NA - 1] : acc[q][0];
#pragma unroll
    for (int o = KC; o < 32; o <<= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], o);
  }
}

// A hub piece in the wide layout: each warp sums a contiguous quarter of the
// piece's in-edges with warp_row_sum (one 8K-byte row per load instruction,
// G loads in flight), the warps' per-column partials meet in shared memory,
// and the piece protocol of hub_piece follows (partial slot, release-ordered
// counter, last piece decides from the partials in piece order). Measured on
// configs[2]: sweep kernel -4% against the column-per-thread hub_piece.
template <int K, int MODE, bool DET>
__device__ __noinline__ void hub_piece_wide(const SweepParams& P, const TileDesc d, uint64_t j,
                                            double* hubsh, int* flag, const ColSh* cs,
                                            const double* thr_cur, const YG& yg,
                                            const double* rcur, double* rnxt, double* ynxt,
                                            double* sh_push, double* sh_d,
                                            unsigned long long* sh_np, unsigned long long* sh_nn,
                                            unsigned long long* sh_et) {
  // (no by-reference locals: the deciding thread's counters go straight to
  // the block's shared per-column sums, so the call needs no stack frame)
  constexpr int KC = wide_kc<K>();
  constexpr int CPL = K / KC;
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t chunk = ((uint64_t)d.ne + NW - 1) / NW;
  const uint64_t b = d.e0 + (uint64_t)warp * chunk;
  const uint64_t e0 = d.e0 + d.ne;
  const uint64_t e = b + chunk < e0 ? b + chunk : e0;
  double s[CPL];
  warp_row_sum<K, DET>(P, yg, b < e ? b : e, e, s);
  if (lane < KC)
#pragma unroll
    for (int q = 0; q < CPL; ++q) hubsh[warp * K + (lane % KC) * CPL + q] = s[q];
  __syncthreads();
  if (tid < K) {
    double t = 0.0;
    for (int w = 0; w < NW; ++w) t += hubsh[w * K + tid];
    P.hub_acc[j * K + tid] = t;  // this piece's partial (slot = its tile)
  }
  __syncthreads();
  if (tid == 0) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(old) : "l"(P.hub_cnt + d.hub) : "memory");
    *flag = old == d.npieces - 1;
    if (*flag) P.hub_cnt[d.hub] = 0;
  }
  __syncthreads();
  if (*flag && tid < K) {
    const double* part = P.hub_acc + (j - d.piece) * K + tid;
    double acc = 0.0;
    for (uint32_t p = 0; p < d.npieces; ++p) acc += __ldcg(part + (uint64_t)p * K);
    const uint32_t u = __ldg(P.crow + d.r0);
    Acc a;
    decide_at<K, MODE, DET>(P, cs, thr_cur, u, tid, acc, __ldg(P.cdeg + d.r0), __ldg(P.cinv + d.r0), yg,
                            rcur, rnxt, ynxt, a);
    if (a.push != 0.0) atomicAdd(&sh_push[tid], a.push);
    if (a.d != 0.0) atomicAdd(&sh_d[tid], a.d);
    if (a.np) atomicAdd(&sh_np[tid], a.np);
    if (a.nn) atomicAdd(&sh_nn[tid], a.nn);
    if (a.et) atomicAdd(&sh_et[tid], a.et);
  }
}

// decide<K, M_POWERPUSH> with the column's threshold and source in registers
// (thr = +inf: the column is done).
template <int K, bool DET>
__device__ __forceinline__ void decide_pp(const SweepParams& P, const ColSh* cs, double thr,
                                          uint32_t src, uint32_t u, int c, double acc, double xo,
                                          uint32_t dg, double inv, double* ynxt, Acc& a) {
  const uint64_t ix = (uint64_t)u * K + c;
  const double oma = 1.0 - P.alpha;
  if (thr == CUDART_INF) {
    if (DET && dg) ynxt[ix] = oma * xo * inv;  // every row's y into this sweep's buffer
    return;
  }
  const double inflow = acc + (u == src ? 1.0 + cs[c].D : 0.0);
  const double r = inflow - xo;
  if (r > (dg ? (double)dg : 1.0) * thr) {
    st_state(P.x + ix, inflow);
    if (!DET && dg) {
      const double yv = oma * inflow * inv;
      P.y[0][ix] = yv;
      for (int p = 0; p < P.npeers; ++p) P.peer_y[p][ix] = yv;  // fused exchange
    }
    a.push += qterm<DET>(r, cs[c].scp);
    a.np += dg ? dg : 1;
    a.nn += 1;
    a.et += dg;
    xo = inflow;
  }
  if (DET && dg) ynxt[ix] = oma * xo * inv;
  if (!dg) a.d += qterm<DET>(oma * xo, cs[c].scd);
}

// Decision layout of the wide path: the columns a lane decides for a row.
// 16-byte and 8-byte lanes (CPL <= 2) decide the columns they loaded. With
// 32-byte lanes (CPL = 4) only KC = K/4 lanes load a row's columns, but after
// warp_row_sum's xor reduction every lane holds every sum of its kc, so all 32
// lanes decide: DPL = K/32 columns each, starting at dc0.
template <int K>
struct DecLayout {
  static constexpr int KC = wide_kc<K>();
  static constexpr int CPL = K / KC;
  static constexpr int DPL = CPL == 4 ? K / 32 : CPL;  // columns decided per lane
  int sb;   // index of the lane's first decided column in its s[CPL]
  int dc0;  // the lane's first decided column
  bool on;  // this lane decides
  __device__ __forceinline__ DecLayout() {
    const int lane = threadIdx.x & 31, kc = lane % KC;
    sb = CPL == 4 ? DPL * (lane / KC) : 0;
    dc0 = kc * CPL + sb;
    on = CPL == 4 ? true : lane < KC;
  }
};

template <int K, int MODE, bool DET>
__device__ __forceinline__ void decide_cols(const SweepParams& P, const ColSh* cs,
                                            const double* thr_cur, const uint32_t* csrc,
                                            uint32_t u, const DecLayout<K>& L, const double* s,
                                            const double* xo, const double* rc, uint32_t dg,
                                            double inv, const YG& yg, double* rnxt,
                                            double* ynxt, Acc& a, const BlockAcc& ba,
                                            double* pacc = nullptr) {
  constexpr int CPL = DecLayout<K>::CPL;
  constexpr int DPL = DecLayout<K>::DPL;
  if constexpr (CPL == 1) {  // one column per lane: the thread's own counters (column = tid % K)
    decide<K, MODE, DET>(P, cs, thr_cur, u, L.dc0, s[0], xo[0], rc[0], dg, inv, yg, rnxt, ynxt, a);
  } else {  // counters via shared atomics
    // the lane's thresholds and sources in one vector shared load each (a
    // done column's threshold is +inf)
    double th[DPL];
    uint32_t sr[DPL];
    if constexpr (DPL == 2) {
      const double2 t2 = reinterpret_cast<const double2*>(thr_cur)[L.dc0 / 2];
      const uint2 s2 = reinterpret_cast<const uint2*>(csrc)[L.dc0 / 2];
      th[0] = t2.x, th[1] = t2.y, sr[0] = s2.x, sr[1] = s2.y;
    } else {
      th[0] = thr_cur[L.dc0];
      sr[0] = csrc[L.dc0];
    }
#pragma unroll
    for (int q = 0; q < DPL; ++q) {
      Acc b2;
      const int cc = L.dc0 + q;
      if constexpr (MODE == M_POWERPUSH)
        decide_pp<K, DET>(P, cs, th[q], sr[q], u, cc, s[q], xo[q], dg, inv, ynxt, b2);
      else
        decide<K, MODE, DET>(P, cs, thr_cur, u, cc, s[q], xo[q], rc[q], dg, inv, yg, rnxt, ynxt, b2);
      if (PPRG_PUSH_REG && pacc) pacc[q] += b2.push;  // flushed once per tile
      else if (b2.push != 0.0) atomicAdd(&ba.push[cc], b2.push);
      if (b2.d != 0.0) atomicAdd(&ba.d[cc], b2.d);
      if (b2.nn) {
        atomicAdd(&ba.pk[cc], (b2.nn << PK_SHIFT) | b2.np);
        if (!b2.et) atomicAdd(&ba.nd[cc], 1u);  // a dead end's push (np 1, no out-edges)
      }
    }
  }
}

// the lane's DPL decided sums out of its CPL row sums, by selects (a dynamic
// index would put s[] in local memory)
template <int K>
__device__ __forceinline__ void pick_sums(const DecLayout<K>& L, const double* s, double* sd) {
  constexpr int CPL = DecLayout<K>::CPL;
  constexpr int DPL = DecLayout<K>::DPL;
#pragma unroll
  for (int q = 0; q < DPL; ++q) {
    double v = s[q];
#pragma unroll
    for (int j = 1; j < CPL / DPL; ++j) v = L.sb == j * DPL ? s[j * DPL + q] : v;
    sd[q] = v;
  }
}

// the lane's DPL state values of row u (issued early; they land during the gathers)
template <int K, int DPL>
__device__ __forceinline__ void load_cols(const double* a, uint32_t u, int dc0, bool on, double* out) {
  const double* p = a + (uint64_t)u * K + dc0;
  if constexpr (DPL == 2) {
    const double2 v = on ? ld_state2(p) : make_double2(0.0, 0.0);
    out[0] = v.x;
    out[1] = v.y;
  } else {
    out[0] = on ? ld_state(p) : 0.0;
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

template <int K, int MODE, bool DET>
__device__ __forceinline__ void tile_rows_wide(const SweepParams& P, const TileDesc& d, char* smem,
                                               const ColSh* cs, const double* thr_cur,
                                               const uint32_t* csrc,
                                               const YG& yg, const double* rcur, double* rnxt,
                                               double* ynxt, Acc& a, const BlockAcc& ba,
                                               uint32_t* rowctr,
                                               const unsigned long long* dn_slot, TileDesc* dn) {
  constexpr int KC = wide_kc<K>();
  constexpr int CPL = K / KC;
  constexpr int NW = NT / 32;
  uint64_t* soff = reinterpret_cast<uint64_t*>(smem);
  double* sinv = reinterpret_cast<double*>(soff + RMAX_W + 1);
  double* spart = sinv + RMAX_W;                       // [NW][K] long-row partials
  uint32_t* snode = reinterpret_cast<uint32_t*>(spart + NW * K);
  uint32_t* sdeg = snode + RMAX_W;
  uint32_t* slong = sdeg + RMAX_W;                     // [RMAX_W] long rows; slong[RMAX_W] = count
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int es0 = lane < KC;  // lanes holding the reduced sums of their kc (first edge slot)
  const int kc = lane % KC;
  const DecLayout<K> L;
  constexpr int DPL = DecLayout<K>::DPL;
  double pacc[DPL];  // pushed mass of my decided columns in this tile (PPRG_PUSH_REG)
#pragma unroll
  for (int q = 0; q < DPL; ++q) pacc[q] = 0.0;
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
      double xo[DPL], rc[DPL], s[CPL];
      load_cols<K, DPL>(P.x, u, L.dc0, L.on, xo);  // issued early; lands during the edge loop
      if constexpr (MODE == M_POWITR || MODE == M_SIMFWD) load_cols<K, DPL>(rcur, u, L.dc0, L.on, rc);
      else
#pragma unroll
        for (int q = 0; q < DPL; ++q) rc[q] = 0.0;
      warp_row_sum<K, DET>(P, yg, b, e, s, true, ids);
      double sd[DPL];
      pick_sums<K>(L, s, sd);
      if (L.on)
        decide_cols<K, MODE, DET>(P, cs, thr_cur, csrc, u, L, sd, xo, rc, sdeg[r], sinv[r], yg, rnxt, ynxt,
                                  a, ba, pacc);
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
    warp_row_sum<K, DET>(P, yg, wb < e ? wb : e, we, s);
    if (es0)
#pragma unroll
      for (int q = 0; q < CPL; ++q) spart[warp * K + kc * CPL + q] = s[q];
    __syncthreads();
    if (warp == 0 && L.on) {
      const uint32_t u = snode[r];
      double xo[DPL], rc[DPL], sd[DPL];
#pragma unroll
      for (int q = 0; q < DPL; ++q) {
        const uint64_t ix = (uint64_t)u * K + L.dc0 + q;
        xo[q] = __ldcg(P.x + ix);
        rc[q] = (MODE == M_POWITR || MODE == M_SIMFWD) ? __ldcg(rcur + ix) : 0.0;
        double t = 0.0;
        for (int w = 0; w < NW; ++w) t += spart[w * K + L.dc0 + q];
        sd[q] = t;
      }
      decide_cols<K, MODE, DET>(P, cs, thr_cur, csrc, u, L, sd, xo, rc, sdeg[r], sinv[r], yg, rnxt, ynxt, a,
                                ba, pacc);
    }
    __syncthreads();
  }
  if (PPRG_PUSH_REG && L.on)
#pragma unroll
    for (int q = 0; q < DPL; ++q)
      if (pacc[q] != 0.0) atomicAdd(&ba.push[L.dc0 + q], pacc[q]);
  __syncthreads();
  if (tid == 0) {
    *rowctr = 0;
    slong[RMAX_W] = 0;
  }
}

// Sources with in-degree 0 are not rows of the compacted transpose; their
// only inflow is the unit start mass plus the dead-end mass D (block 0).
template <int K, int MODE, bool DET>
__device__ __forceinline__ void source_rows(const SweepParams& P, const ColSh* cs,
                                            const double* thr_cur, const YG& yg,
                                            const double* rcur, double* rnxt, double* ynxt,
                                            Acc& a) {
  const int tid = threadIdx.x;
  if (blockIdx.x != 0 || tid >= K) return;
  const uint32_t u = P.src[tid];
  if (u < P.own_lo || u >= P.own_hi) return;  // another partition's row
  if (__ldg(P.in_off_full + u + 1) != __ldg(P.in_off_full + u)) return;
  const uint64_t ix = (uint64_t)u * K + tid;
  decide<K, MODE, DET>(P, cs, thr_cur, u, tid, 0.0, __ldcg(P.x + ix),
                  (MODE == M_POWITR || MODE == M_SIMFWD) ? __ldcg(rcur + ix) : 0.0, __ldg(P.deg + u),
                  __ldg(P.inv_deg + u), yg, rnxt, ynxt, a);
}

#ifndef PPRG_MINB
#define PPRG_MINB 8
#endif
#ifndef PPRG_MINB_NARROW
#define PPRG_MINB_NARROW PPRG_MINB
#endif
#ifndef PPRG_MINB_K1
#define PPRG_MINB_K1 6
#endif
// Fixed-point scale 2^(52 - e) for a per-column sum bounded by `bound` < 2^e:
// every scaled term and partial sum stays an integer below 2^53.
__device__ __forceinline__ double det_scale(double bound) {
  int e;
  frexp(bound > 1e-280 ? bound : 1e-280, &e);
  return ldexp(1.0, 52 - e);
}

// The persistent sweep kernel: every epoch and sweep of a query block in one
// cooperative launch (see DESIGN 3). DET: deterministic sweeps -- the tile
// list runs as P.nwaves waves of contiguous rows separated by grid barriers;
// a row of wave w gathers this sweep's y for rows of waves < w and the
// previous sweep's y for all others (y double-buffered: every row writes its
// y into this sweep's buffer, pushed or not), and the per-column sums are
// fixed-point integers (qterm). Results are then a function of the inputs
// alone: no timing, no atomic order.
template <int K, int MODE, bool DET>
__global__ void __launch_bounds__(NT, (K >= 4 ? PPRG_MINB : K == 1 ? PPRG_MINB_K1 : PPRG_MINB_NARROW))
    k_sweeps(const __grid_constant__ SweepParams P) {
  using TC = Tile<K>;
  extern __shared__ __align__(16) char smem_dyn[];
  __shared__ ColSh cs[K];
  __shared__ __align__(16) double thr_cur[K];
  __shared__ __align__(16) uint32_t csrc[K];  // column sources (lane-pair loads in decide_cols)
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
    cs[tid].D = P.D_dev ? P.D_dev[tid] : P.init[tid].D;
    cs[tid].epoch = P.init[tid].epoch;
    cs[tid].done = P.init[tid].done;
    cs[tid].sweeps = P.init[tid].sweeps;
    cs[tid].pushes = P.init[tid].pushes;
    cs[tid].src = P.src[tid];
    cs[tid].scp = cs[tid].scd = 1.0;
    cs[tid].pull = P.final_pull[tid];
    csrc[tid] = P.src[tid];
    if (P.from_drain) {  // push.cpp:168-180, decided here instead of on the host
      const double rs = __ldcg(P.from_drain + tid);
      const int scan = tid < P.k_live && (P.scan_all || rs > P.scan_lambda);
      int ep = 0;
      while (ep < P.E && !(rs > P.lam[ep])) ++ep;
      cs[tid].r_sum = rs;
      cs[tid].epoch = ep;
      cs[tid].done = !scan || ep >= P.E;
      cs[tid].pull = scan;
    }
    if (P.from_sweeps) {  // the final pass after a device-started global phase
      cs[tid].r_sum = __ldcg(&P.from_sweeps->out_rsum[tid]);
      cs[tid].D = __ldcg(&P.from_sweeps->out_D[tid]);
      cs[tid].pull = __ldcg(&P.from_sweeps->out_scan[tid]);
    }
  }
  __syncthreads();
  __shared__ unsigned long long sh_pk[K];
  __shared__ unsigned sh_nd[K];
  const BlockAcc ba{sh_push, sh_d, sh_np, sh_nn, sh_et, sh_pk, sh_nd};
  unsigned long long gen = 0;
  const int c = tid % K;
  for (uint32_t sweep = 0;; ++sweep) {
    const int buf = sweep % 3;
    if (tid == 0) {
      int any = 0;
      for (int cc = 0; cc < K; ++cc) any |= !cs[cc].done;
      sh_any = any && (MODE == M_FINAL ? sweep == 0 : sweep < P.max_sweeps);
      if (!DET && sh_any && !P.k1w) sh_tile[0] = atomicAdd(&ctl->ticket[buf], 1u);
      sh_nlong = 0;
      if constexpr (K >= WIDE_K) *wide_long_count<K>(smem_dyn) = 0;
    }
    if (tid < K) {
      // a done column's threshold is +inf (decide_pp's done test); decide()
      // checks cs[].done itself
      thr_cur[tid] = MODE != M_POWERPUSH ? 0.0 : cs[tid].done ? CUDART_INF : P.thr[cs[tid].epoch];
      if constexpr (DET) {
        // bounds of this sweep's sums (identical in every block): PowerPush
        // pushes at most r_sum / alpha (Gauss-Seidel within a sweep), D grows by
        // at most that; PowItr / the final pass sum at most r_sum
        const double rs = cs[tid].r_sum > 0 ? cs[tid].r_sum : 0.0;
        const double bp = MODE == M_POWERPUSH ? 2.0 * rs / P.alpha : 2.0 * rs;
        cs[tid].scp = det_scale(bp);
        cs[tid].scd = det_scale(MODE == M_POWERPUSH ? cs[tid].D + bp : bp);
      }
      sh_push[tid] = 0.0;
      sh_d[tid] = 0.0;
      sh_np[tid] = 0;
      sh_nn[tid] = 0;
      sh_et[tid] = 0;
      sh_pk[tid] = 0;
      sh_nd[tid] = 0;
    }
    __syncthreads();
    if (!sh_any) break;
    if (blockIdx.x == 0 && tid == 0 && MODE != M_FINAL) {
      const int nb = (sweep + 1) % 3;  // last read two barriers ago; safe to clear
      ctl->ticket[nb] = 0;
      if (DET)
        for (int w = 0; w < WMAX; ++w) ctl->wticket[nb][w] = 0;
      for (int cc = 0; cc < K; ++cc) {
        ctl->pushed[nb][cc] = 0;
        ctl->npush[nb][cc] = 0;
        ctl->nnode[nb][cc] = 0;
        ctl->dsum[nb][cc] = 0;
        ctl->et[nb][cc] = 0;
      }
    }
    const int par = (MODE == M_POWERPUSH && !DET) || MODE == M_FINAL ? 0 : (int)(sweep & 1);
    YG yg{P.y[par], P.y[par ^ 1], 0u};
    const double* rcur = P.r[sweep & 1];
    double* rnxt = P.r[(sweep + 1) & 1];
    double* ynxt = P.y[(sweep + 1) & 1];
    Acc a;
    // Tiles [t0, t1) in ticket (= id) order from counter ctr; the next ticket
    // is fetched one tile ahead and the next descriptor loaded inside the
    // current tile. The first ticket is in sh_tile[0].
    auto run_tiles = [&](unsigned* ctr, uint64_t t0, uint64_t t1) {
      if (K == 1 && PPRG_K1W && P.k1w) {
        sweep_k1_warps<MODE, DET>(P, cs, thr_cur, yg, rcur, rnxt, ynxt, a,
                                  reinterpret_cast<double*>(smem_dyn), ctr, t0, t1);
        return;
      }
      unsigned long long j = sh_tile[0];
      TileDesc d = P.desc[j < t1 ? j : 0];
      for (uint32_t it = 0;; ++it) {
        if (j >= t1) break;
        if (tid == 0) sh_tile[(it + 1) & 1] = t0 + atomicAdd(ctr, 1u);
        TileDesc dn = d;
        if (d.npieces > 1) {
          if constexpr (K >= WIDE_K)
            hub_piece_wide<K, MODE, DET>(P, d, j, sh_hub, &sh_flag, cs, thr_cur, yg, rcur, rnxt, ynxt,
                                         sh_push, sh_d, sh_np, sh_nn, sh_et);
          else
            hub_piece<K, MODE, DET>(P, d, j, sh_hub, &sh_flag, cs, thr_cur, yg, rcur, rnxt, ynxt, a);
          dn = P.desc[sh_tile[(it + 1) & 1] < t1 ? sh_tile[(it + 1) & 1] : 0];
          __syncthreads();
        } else if constexpr (K >= WIDE_K) {
          tile_rows_wide<K, MODE, DET>(P, d, smem_dyn, cs, thr_cur, csrc, yg, rcur, rnxt, ynxt, a, ba,
                                       &sh_nlong, &sh_tile[(it + 1) & 1], &dn);
        } else {
          tile_rows<K, MODE, DET>(P, d, smem_dyn, cs, thr_cur, yg, rcur, rnxt, ynxt, a, ba, &sh_nlong,
                                  &sh_tile[(it + 1) & 1], &dn);
        }
        j = sh_tile[(it + 1) & 1];
        d = dn;
      }
    };
    if constexpr (!DET) {
      if (K == 1 && PPRG_K1W && P.k1w) {
        sweep_k1_warps<MODE, DET>(P, cs, thr_cur, yg, rcur, rnxt, ynxt, a,
                                  reinterpret_cast<double*>(smem_dyn), &ctl->ticket[buf], 0, P.ntiles);
      } else {
        unsigned long long j = sh_tile[0];
        TileDesc d = P.desc[j < P.ntiles ? j : 0];
        for (uint32_t it = 0;; ++it) {
          if (j >= P.ntiles) break;
          if (tid == 0) sh_tile[(it + 1) & 1] = atomicAdd(&ctl->ticket[buf], 1u);
          TileDesc dn = d;
          if (d.npieces > 1) {
            if constexpr (K >= WIDE_K)
              hub_piece_wide<K, MODE, DET>(P, d, j, sh_hub, &sh_flag, cs, thr_cur, yg, rcur, rnxt, ynxt,
                                           sh_push, sh_d, sh_np, sh_nn, sh_et);
            else
              hub_piece<K, MODE, DET>(P, d, j, sh_hub, &sh_flag, cs, thr_cur, yg, rcur, rnxt, ynxt, a);
            dn = P.desc[sh_tile[(it + 1) & 1] < P.ntiles ? sh_tile[(it + 1) & 1] : 0];
            __syncthreads();
          } else if constexpr (K >= WIDE_K) {
            tile_rows_wide<K, MODE, DET>(P, d, smem_dyn, cs, thr_cur, csrc, yg, rcur, rnxt, ynxt, a, ba,
                                         &sh_nlong, &sh_tile[(it + 1) & 1], &dn);
          } else {
            tile_rows<K, MODE, DET>(P, d, smem_dyn, cs, thr_cur, yg, rcur, rnxt, ynxt, a, ba, &sh_nlong,
                                    &sh_tile[(it + 1) & 1], &dn);
          }
          j = sh_tile[(it + 1) & 1];
          d = dn;
        }
      }
      source_rows<K, MODE, DET>(P, cs, thr_cur, yg, rcur, rnxt, ynxt, a);
    } else {
      // sources without in-edges first (their inflow does not depend on the
      // sweep's other rows); then the waves
      source_rows<K, MODE, DET>(P, cs, thr_cur, yg, rcur, rnxt, ynxt, a);
      const uint32_t nwv = MODE == M_POWERPUSH && P.nwaves > 1 ? P.nwaves : 1;
      for (uint32_t wv = 0; wv < nwv; ++wv) {
        const uint64_t t0 = nwv > 1 ? P.wave_tile[wv] : 0, t1 = nwv > 1 ? P.wave_tile[wv + 1] : P.ntiles;
        yg.lo = nwv > 1 ? P.wave_node[wv] : 0u;  // wave_node[0] = 0: sources without in-edges are in yn
        if (tid == 0 && !P.k1w) sh_tile[0] = t0 + atomicAdd(&ctl->wticket[buf][wv], 1u);
        __syncthreads();
        run_tiles(&ctl->wticket[buf][wv], t0, t1);
        if (wv + 1 < nwv) grid_barrier2(&ctl->gbar, ++gen);
      }
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
    if (tid < K && sh_pk[tid]) {  // unpack the two-columns-per-lane counters
      const unsigned long long np = sh_pk[tid] & ((1ull << PK_SHIFT) - 1);
      sh_np[tid] += np;
      sh_nn[tid] += sh_pk[tid] >> PK_SHIFT;
      sh_et[tid] += np - sh_nd[tid];
    }
    if (tid < K) {
      if (sh_push[tid] != 0.0) atomicAdd(&ctl->pushed[buf][tid], sh_push[tid]);
      if (sh_d[tid] != 0.0) atomicAdd(&ctl->dsum[buf][tid], sh_d[tid]);
      if (sh_np[tid]) atomicAdd(&ctl->npush[buf][tid], sh_np[tid]);
      if (sh_nn[tid]) atomicAdd(&ctl->nnode[buf][tid], sh_nn[tid]);
      if (sh_et[tid]) atomicAdd(&ctl->et[buf][tid], sh_et[tid]);
    }
    if (MODE == M_FINAL) {
      if (blockIdx.x == 0 && tid < K) ctl->out_scale[tid] = cs[tid].scp;
      __syncthreads();
      break;
    }
    grid_barrier2(&ctl->gbar, ++gen);
    // every block derives the identical next state from the reduced buffers
    if (tid < K) {
      const int cc = tid;
      if (!cs[cc].done) {
        const double pushed = __ldcg(&ctl->pushed[buf][cc]) / cs[cc].scp;
        const unsigned long long np = __ldcg(&ctl->npush[buf][cc]);
        cs[cc].sweeps += 1;
        cs[cc].pushes += np;
        cs[cc].D = __ldcg(&ctl->dsum[buf][cc]) / cs[cc].scd;
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
    ctl->out_scan[tid] = cs[tid].pull;
    ctl->out_rsum[tid] = cs[tid].r_sum;
    ctl->out_D[tid] = cs[tid].D;
    ctl->out_sweeps[tid] = cs[tid].sweeps;
    ctl->out_done[tid] = cs[tid].done;
    ctl->out_epoch[tid] = cs[tid].epoch;
    ctl->out_pushes[tid] = cs[tid].pushes;
  }
}

}  // namespace pprg
