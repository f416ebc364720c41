// Delta sweeps: the PowerPush global phase (push.cpp:168-197) for wide column
// blocks on graphs whose gather operand does not fit in L2. Included by
// push.cu after sweep_kernel.cuh.
//
// k_sweeps gathers, per in-edge, the neighbour's cumulative y row (8K bytes:
// 512 B at 64 columns). Here the residue is explicit and a push publishes only
// this sweep's *increment* per out-edge, as a 16-bit float (e8m8, unsigned):
// 2K bytes per in-edge (one 128-byte line at 64 columns), a quarter of the
// gather traffic, and the gathered array (n x K x 2 B) is a quarter of y.
//
// Exactness. A push of row u with residue r (push.cpp:17-27) moves r' <= r:
//     h  = e8m8 of (1-a) r / deg_eff, rounded DOWN        (the published share)
//     r' = value(h) * deg_eff / (1-a)                     (the mass that leaves)
//     x_u += r' (reserve = a x), r_u -= r', every out-neighbour later adds value(h).
// The rounding remainder (< 2^-8 of r) simply stays in r_u, so mass is
// conserved to fp64 rounding, residues stay >= 0, r_sum -= a r' (push.cpp:25)
// stays exact, and the loop still ends at r_sum <= lambda: the 16-bit format
// costs convergence rate (<0.4% of a row's residue left behind per push), not
// accuracy. Sums of shares are formed in fp64 (a share's fp64 high word is
// h << 12: decode is one widening multiply per share, no conversion
// instruction; see add_shares for the two shares of a word).
//
// Exactly-once. Every published share must be added by every out-neighbour
// exactly once, so the asynchronous "read whatever is there" of k_sweeps is
// not available. Rows are cut into W waves of contiguous ids (equal in-edges);
// shares are double-buffered by sweep parity; a row of wave w in sweep t reads
//     d[t & 1][v]        if wave(v) <= w - L   (published earlier in this sweep)
//     d[(t-1) & 1][v]    otherwise             (published in the previous sweep)
// with lag L >= 2 (default: 64 waves, L = 6): a task of wave w starts once
// every task of the waves <= w-L has finished (per-wave completion counters,
// release adds and one acquire per block and wave), so a wave's tail overlaps
// the next waves' start and no grid barrier sits between waves. One grid
// barrier per sweep closes the sweep (counters, epoch decisions), as in
// k_sweeps. Gauss-Seidel between waves: 50 sweeps on configs[2] against 44.
// After the last pushing sweep one more sweep consumes the shares in flight.
// Work units are warp tasks (delta_task); the blocks only share per-column
// state and the per-sweep sums.
#pragma once
#include "sweep_kernel.cuh"

namespace pprg {

#ifndef PPRG_DS_NT
#define PPRG_DS_NT 128
#endif
constexpr int DS_NT = PPRG_DS_NT;
constexpr int DS_NW = DS_NT / 32;
#ifndef PPRG_DS_G
#define PPRG_DS_G 8
#endif
constexpr int DS_G = PPRG_DS_G;  // 16-byte row loads in flight per lane
constexpr uint32_t DS_IDS = 512;    // in-edges per task at most
constexpr uint32_t DS_TASK_R = 32;  // rows per task (lane i holds row i's data)
#ifndef PPRG_DS_SHORT
#define PPRG_DS_SHORT 64
#endif
constexpr uint32_t DS_SHORT = PPRG_DS_SHORT;  // rows up to this many in-edges: one lane group each
constexpr int DS_WMAX = 64;         // waves per sweep
constexpr int DS_EXP = 769;         // value(h) = fp64{h << 12, 0} * 2^769: e8m8 spans 2^-253 .. 4
// A/B switches (tools/build_variant.sh; measured in profiles/r02_delta_history.txt)
#ifndef PPRG_DS_PFROWS
#define PPRG_DS_PFROWS 1   // a task's share rows prefetched into L2 when its ids are staged
#endif
#ifndef PPRG_DS_PFTASK
#define PPRG_DS_PFTASK 1   // the next task's ids and row data prefetched into L2
#endif
#ifndef PPRG_DS_L1STATE
#define PPRG_DS_L1STATE 1  // state rows (r, x) prefetched into and read through L1 (0: L2)
#endif
#ifndef PPRG_DS_MINB
#define PPRG_DS_MINB 5     // blocks per SM (96 registers); 4 and 6 are both slower
#endif

struct DeltaParams {
  uint64_t n, m;
  const uint64_t* in_off;   // compacted transpose rows
  const uint32_t* crow;
  const uint32_t* cdeg;
  const double* cinv;
  const uint64_t* in_off_full;
  const uint32_t* in_nbr;
  const uint32_t* deg;
  const double* inv_deg;
  const TileDesc* desc;
  uint64_t ntiles;
  double* hub_acc;          // [ntiles][K] raw partial sums of hub pieces
  unsigned* hub_cnt;
  int k_live, E;
  double alpha, inv_oma;    // inv_oma = 1 / (1 - alpha)
  double* x;                // [n][K] pushed mass
  double* r;                // [n][K] explicit residues
  uint4* dsh;               // [n][2][K] u16 shares: row v of sweep parity p at 2 v + p
  const double* from_drain; // exact r_sum after the local phase
  double scan_lambda;
  int scan_all;                   // refine epoch appended: every live column runs the sweeps
  unsigned long long handoff_np;  // refine epoch: hand off to the frontier below this many edge pushes
  SweepCtl* ctl;
  uint32_t max_sweeps;
  uint32_t nwaves, lag;
  uint32_t wave_tile[DS_WMAX + 1];
  uint32_t wave_node[DS_WMAX + 1];
  uint32_t src[KMAX];
  double thr[EMAX], lam[EMAX];
};

#ifndef PPRG_DS_GATHER_NA
#define PPRG_DS_GATHER_NA 0  // 1: share gathers do not allocate in L1
#endif
__device__ __forceinline__ uint4 ld_share(const uint4* p) {
  uint4 v;
#if PPRG_DS_GATHER_NA
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
#endif
  asm volatile("ld.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
// A 32-bit word holds two shares: A (even column) in its low half, B (odd
// column) in its high half. Decode is one widening multiply each, straight
// into an aligned register pair (no masks, no zero words: 2.5 instead of 3.6
// instructions per share):
//   A: fp64 bits = (w << 16) * 2^28 = A << 44      -> hi = A << 12, lo = 0: exact
//   B: fp64 bits =  w        * 2^28                -> hi = B << 12 | A >> 4, lo = A << 28
// so B's value carries A's bits below its 8 mantissa bits. The row that
// publishes the word computes B's value the same way and rounds B's field
// down one more step (share_field), so value_b(w) <= the share it wanted and
// the mass it deducts is exactly what its out-neighbours add. (B = 0 beside
// A != 0 decodes to a subnormal below 2^-253: 1e-76 of unaccounted mass.)
__device__ __forceinline__ double share_value(uint32_t h) {  // raw (unscaled) value of a clean share
  return __hiloint2double((int)(h << 12), 0);
}
__device__ __forceinline__ double value_b(uint32_t w) {  // raw value of the word's odd-column share
  return __longlong_as_double((long long)((unsigned long long)w * 0x10000000ull));
}
// the field of a wanted raw share q (an fp64 below 2^(256-1023)): e8m8 rounded
// down, one step lower for odd columns; 0 = below the format (no push)
__device__ __forceinline__ uint32_t share_field(double q, bool odd) {
  uint32_t h = (uint32_t)__double2hiint(q) >> 12;
  h = h > 0xFFFFu ? 0xFFFFu : h;
  if (odd) return h >= 257u ? h - 1u : 0u;
  return h >= 256u ? h : 0u;
}
// the 8 shares of one 16-byte group added to their columns' sums
__device__ __forceinline__ void add_shares(double (&acc)[8], const uint4& v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    acc[2 * i] += __longlong_as_double((long long)((unsigned long long)(w[i] << 16) * 0x10000000ull));
    acc[2 * i + 1] += value_b(w[i]);
  }
}

// Per-block shared state of the delta sweeps (the warps of a block work
// independently; the block only shares the per-column state and sums).
template <int K>
struct DeltaSh {
  static constexpr int LPR = K / 8;    // lanes per row (16 B = 8 columns each)
  static constexpr int ES = 32 / LPR;  // rows (lane groups) per warp instruction
  // Per-lane sums of a sweep, [warp][column-in-lane q][lane]: every lane owns its
  // 8 entries (no atomics) and a warp's accesses for one q are 32 consecutive
  // words (no bank conflicts; as [lane group][column] arrays the same adds were
  // 16-way conflicted and, with the shared atomics of the counters, kept the LSU
  // data pipe 67% busy). Column c = 8 kc + q of lane group es sits at lane es LPR + kc.
  double pacc[DS_NW][8][32];           // pushed mass
  double pdead[DS_NW][8][32];          // (1-a) x mass pushed by dead-end rows (to the source next sweep)
  unsigned long long pcnt[DS_NW][8][32];  // node pushes << 40 | edge pushes
  uint32_t sids[DS_NW][DS_IDS];        // each warp's task: its in-edge ids
  double thr[LPR * 10];                // this sweep's thresholds, column c at (c/8)*10 + c%8
  double dd[K];                        // dead-end mass of the previous sweep (to the source)
  double srcpush[K];                   // mass pushed by sources without in-edges
  double r_sum[K];
  unsigned long long pushes[K];
  uint32_t csrc[K];
  unsigned nd[K];                      // dead-end pushes (rare enough for shared atomics)
  double srcdead[K];                   // dead-end mass pushed by sources without in-edges
  unsigned srcnn[K], srcnp[K];
  unsigned sweeps[K];
  int epoch[K];
  int done[K];
  uint32_t bloom[64];                  // 2048 bits: (node & 2047) of every source
  int any;
  uint32_t known;                      // leading waves of this sweep known complete (by some warp)
};

// Gather operand of one task. The two share buffers are interleaved by row
// (row v of parity p at index 2 v + p), so the buffer choice is an index bit;
// the staged ids already carry it (row()), so a gather address is one multiply-add.
template <int K>
struct DRow {
  const uint4* base;  // shares + this lane's 16-byte column group
  uint32_t bound;     // ids below: published earlier in this sweep (parity par), others par ^ 1
  uint32_t par;
  __device__ __forceinline__ uint32_t row(uint32_t id) const {
    return 2u * id + (id < bound ? par : par ^ 1u);
  }
  __device__ __forceinline__ const uint4* at(uint32_t row) const {
    return base + (uint64_t)row * (K / 8);
  }
};
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// State rows (r, x) are touched by exactly one warp per sweep and every sweep
// starts with an L1 invalidation (the grid barrier's fence), so they may be
// prefetched into and read through L1.
__device__ __forceinline__ void prefetch_state(const void* p) {
#if PPRG_DS_L1STATE
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
#else
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
#endif
}
__device__ __forceinline__ dbl4 ld_rowstate4(const double* p) {
#if PPRG_DS_L1STATE
  return ld_gather4(p);
#else
  return ld_state4(p);
#endif
}

// Raw share sums of ES short rows at once: lane group es sums the in-edges
// ids[0 .. len) of its row (len = 0: no row). ids: the task's in-edge ids in
// shared memory (staged once per task, so no id load sits in a gather chain).
template <int K>
__device__ __forceinline__ void group_sum(const DRow<K>& X, const uint32_t* ids, uint32_t len,
                                          uint32_t maxlen, double (&acc)[8]) {
  for (uint32_t p0 = 0; p0 < maxlen; p0 += DS_G) {
    uint4 v[DS_G];
#pragma unroll
    for (int g = 0; g < DS_G; ++g)
      v[g] = p0 + g < len ? ld_share(X.at(ids[p0 + g])) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int g = 0; g < DS_G; ++g) add_shares(acc, v[g]);
  }
}

// Raw share sums of the in-edges ids[0 .. ne) by the whole warp: lane groups
// take every ES-th edge, DS_G loads per lane in flight. Afterwards every lane
// holds the totals of its 8 columns.
template <int K>
__device__ __forceinline__ void warp_sum(const DRow<K>& X, const uint32_t* ids, uint32_t ne,
                                         double (&acc)[8]) {
  constexpr int LPR = K / 8, ES = 32 / LPR;
  constexpr uint32_t BE = ES * DS_G;  // edges per batch: 16 at K = 64, 32 at K = 32
  const uint32_t es = (threadIdx.x & 31) / LPR;
  for (uint32_t t0 = 0; t0 < ne; t0 += BE) {
    uint4 v[DS_G];
#pragma unroll
    for (int g = 0; g < DS_G; ++g) {
      const uint32_t j = t0 + g * ES + es;
      v[g] = j < ne ? ld_share(X.at(ids[j])) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int g = 0; g < DS_G; ++g) add_shares(acc, v[g]);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q)
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
}

// The decision for 8 columns [8 kc, 8 kc + 8) of row u by one lane: add the
// gathered shares to the residues, push the columns above their threshold
// (push.cpp:182-193) in the share format, write this sweep's shares.
// acc: raw share sums. slot: the calling lane's index in its warp's sum planes
// (lane group es, column group kc -> es LPR + kc), warp: its warp.
template <int K>
__device__ __noinline__ void decide8(const DeltaParams& P, DeltaSh<K>& S, uint4* dcur, uint32_t u,
                                     uint32_t dg, double inv, double a0, double a1, double a2,
                                     double a3, double a4, double a5, double a6, double a7, int kc,
                                     int slot) {
  const double acc[8] = {a0, a1, a2, a3, a4, a5, a6, a7};
  const uint64_t ix = (uint64_t)u * K + kc * 8;
  const dbl4 ra = ld_rowstate4(P.r + ix), rb = ld_rowstate4(P.r + ix + 4);
  // (x too, before any decision: one memory latency per row instead of two; nearly
  // every visited row pushes in some column)
  const dbl4 xa = ld_rowstate4(P.x + ix), xb = ld_rowstate4(P.x + ix + 4);
  double rr[8];
  const double up = ldexp(1.0, DS_EXP);
  bool chg = false;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    rr[q] = fma(acc[q], up, q < 4 ? ra.v[q] : rb.v[q - 4]);
    chg |= acc[q] != 0.0;
  }
  if ((S.bloom[(u >> 5) & 63] >> (u & 31)) & 1u) {  // maybe a source: last sweep's dead-end mass
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (u == S.csrc[kc * 8 + q] && S.dd[kc * 8 + q] != 0.0) {
        rr[q] += S.dd[kc * 8 + q];
        chg = true;
      }
  }
  const double dthr = dg ? (double)dg : 1.0;
  unsigned pm = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) pm |= (rr[q] > dthr * S.thr[kc * 10 + q]) ? 1u << q : 0u;
  uint32_t w[4] = {0u, 0u, 0u, 0u};
  if (pm) {
    double xx[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) xx[q] = q < 4 ? xa.v[q] : xb.v[q - 4];
    const double oma = 1.0 - P.alpha;
    const double c1 = oma * inv * ldexp(1.0, -DS_EXP);  // residue -> raw share
    const double c2 = dthr * P.inv_oma * up;            // raw share -> mass leaving the row
    const int wp = threadIdx.x >> 5;
    double* pa = &S.pacc[wp][0][slot];            // my column q at pa[32 q]
    unsigned long long* pc = &S.pcnt[wp][0][slot];
    if (dg) {
      // the words first (an odd column's value depends on its even neighbour's field)
      uint32_t hf[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        hf[q] = ((pm >> q) & 1u) ? share_field(rr[q] * c1, q & 1) : 0u;
        w[q >> 1] |= hf[q] << (16 * (q & 1));
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (!hf[q]) continue;  // (below the format's range: stays a residue)
        const double val = (q & 1) ? value_b(w[q >> 1]) : share_value(hf[q]);
        const double rp = fmin(val * c2, rr[q]);
        xx[q] += rp;
        rr[q] -= rp;
        pa[32 * q] += rp;
        pc[32 * q] += (1ull << 40) | dg;
      }
    } else {  // dead end: everything leaves, (1-a) of it to the source next sweep
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (!((pm >> q) & 1u)) continue;
        const double rp = rr[q];
        S.pdead[wp][q][slot] += oma * rp;
        atomicAdd(&S.nd[kc * 8 + q], 1u);
        xx[q] += rp;
        rr[q] -= rp;
        pa[32 * q] += rp;
        pc[32 * q] += (1ull << 40) | 1ull;
      }
    }
    dbl4 oa, ob;
#pragma unroll
    for (int q = 0; q < 4; ++q) oa.v[q] = xx[q], ob.v[q] = xx[q + 4];
    st_state4(P.x + ix, oa);
    st_state4(P.x + ix + 4, ob);
    chg = true;
  }
  if (chg) {
    dbl4 oa, ob;
#pragma unroll
    for (int q = 0; q < 4; ++q) oa.v[q] = rr[q], ob.v[q] = rr[q + 4];
    st_state4(P.r + ix, oa);
    st_state4(P.r + ix + 4, ob);
  }
  if (dg) dcur[(uint64_t)(2u * u) * (K / 8) + kc] = make_uint4(w[0], w[1], w[2], w[3]);
}

// One warp task (a TileDesc of the warp-task plan): a bundle of <= 32 whole
// rows with <= DS_TASK_E in-edges, or one whole longer row, or one piece of a
// row cut into DS_PIECE-edge pieces. No block barrier anywhere: lane i holds
// bundle row i's data (offsets, node, degree) and hands it out by shuffle;
// rows of <= DS_SHORT in-edges run ES at a time in lane groups, longer ones one
// at a time over the whole warp; pieces leave raw partial sums in hub_acc and
// the last piece to arrive decides the row.
template <int K>
__device__ __forceinline__ void delta_task(const DeltaParams& P, DeltaSh<K>& S, const TileDesc& d,
                                           uint64_t j, const DRow<K>& X, uint4* dcur) {
  constexpr int LPR = K / 8, ES = 32 / LPR;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kc = lane % LPR, es = lane / LPR;
  // the task's in-edge ids into shared memory, every load in flight at once
  uint32_t* ids = S.sids[warp];
#pragma unroll 4
  for (uint32_t i = lane; i < d.ne; i += 32) {
    const uint32_t row = X.row(ld_stream(P.in_nbr + d.e0 + i));
    ids[i] = row;
#if PPRG_DS_PFROWS
    prefetch_l2(X.at(row));  // its share row on the way into L2
#endif
  }
  __syncwarp();
  if (d.npieces > 1) {  // ---- a piece of a hub row ------------------------------
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    warp_sum<K>(X, ids, d.ne, acc);
    if (es == 0)
#pragma unroll
      for (int q = 0; q < 8; ++q) P.hub_acc[j * K + kc * 8 + q] = acc[q];
    __syncwarp();
    unsigned old = 0;
    if (lane == 0) {
      // (release only: an acquire invalidates the SM's L1, so only the last
      // arriver, who reads the other pieces' partials, pays for one)
      asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;"
                   : "=r"(old) : "l"(P.hub_cnt + d.hub) : "memory");
      if (old == d.npieces - 1) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        P.hub_cnt[d.hub] = 0;
      }
    }
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old != d.npieces - 1) return;
    __syncwarp();
    {  // the last piece to arrive: the partials of all pieces, lane groups taking every ES-th
      const double* part = P.hub_acc + (j - d.piece) * K + kc * 8;
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = 0.0;
      for (uint32_t p = es; p < d.npieces; p += ES) {
        const dbl4 a = ld_state4(part + (uint64_t)p * K), b = ld_state4(part + (uint64_t)p * K + 4);
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] += a.v[q], acc[q + 4] += b.v[q];
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int o = LPR; o < 32; o <<= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
    }
    if (es == 0)
      decide8<K>(P, S, dcur, __ldg(P.crow + d.r0), __ldg(P.cdeg + d.r0), __ldg(P.cinv + d.r0),
                 acc[0], acc[1], acc[2], acc[3], acc[4], acc[5], acc[6], acc[7], kc, lane);
    return;
  }
  // ---- whole rows: lane i holds row i --------------------------------------
  uint32_t loff = 0, llen = 0, lnode = 0, ldeg = 0;
  double linv = 0.0;
  if ((uint32_t)lane < d.nr) {
    const uint64_t o = __ldg(P.in_off + d.r0 + lane);
    loff = (uint32_t)(o - d.e0);
    llen = (uint32_t)(__ldg(P.in_off + d.r0 + lane + 1) - o);
    lnode = __ldg(P.crow + d.r0 + lane);
    ldeg = __ldg(P.cdeg + d.r0 + lane);
    linv = __ldg(P.cinv + d.r0 + lane);
  }
  const unsigned longm = __ballot_sync(0xffffffffu, llen > DS_SHORT);
  // short rows, ES per pass; the next pass's first in-edge ids are loaded and its
  // state rows prefetched into L2 before this pass's gathers
  auto prep = [&](uint32_t g0, uint32_t& off, uint32_t& len, uint32_t& node) {
    const int srcl = (int)(g0 + es) & 31;
    off = __shfl_sync(0xffffffffu, loff, srcl);
    len = __shfl_sync(0xffffffffu, llen, srcl);
    node = __shfl_sync(0xffffffffu, lnode, srcl);
    if (g0 + es >= d.nr || len > DS_SHORT) len = 0;
    if (!len) return;
    const uint64_t ix = (uint64_t)node * K + kc * 8;
    prefetch_state(P.r + ix);
    prefetch_state(P.x + ix);
  };
  if (d.nr > 1 || !longm) {
    uint32_t off, len, node;
    prep(0, off, len, node);
    for (uint32_t g0 = 0; g0 < d.nr; g0 += ES) {
      uint32_t offn = 0, lenn = 0, noden = 0;
      if (g0 + ES < d.nr) prep(g0 + ES, offn, lenn, noden);
      const uint32_t maxlen = __reduce_max_sync(0xffffffffu, len);
      if (maxlen) {
        double acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = 0.0;
        group_sum<K>(X, ids + off, len, maxlen, acc);
        const int srcl = (int)(g0 + es) & 31;
        const uint32_t dg = __shfl_sync(0xffffffffu, ldeg, srcl);
        const double inv = __shfl_sync(0xffffffffu, linv, srcl);
        if (len)
          decide8<K>(P, S, dcur, node, dg, inv, acc[0], acc[1], acc[2], acc[3], acc[4], acc[5],
                     acc[6], acc[7], kc, lane);
      }
      off = offn;
      len = lenn;
      node = noden;
    }
  }
  // longer rows, one at a time over the whole warp
  for (unsigned m = longm; m; m &= m - 1) {
    const int rl = __ffs(m) - 1;
    const uint32_t off = __shfl_sync(0xffffffffu, loff, rl);
    const uint32_t len = __shfl_sync(0xffffffffu, llen, rl);
    const uint32_t node = __shfl_sync(0xffffffffu, lnode, rl);
    const uint32_t dg = __shfl_sync(0xffffffffu, ldeg, rl);
    const double inv = __shfl_sync(0xffffffffu, linv, rl);
    if (es == 0) {
      const uint64_t ix = (uint64_t)node * K + kc * 8;
      prefetch_state(P.r + ix);
      prefetch_state(P.x + ix);
    }
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    warp_sum<K>(X, ids + off, len, acc);
    if (es == 0)
      decide8<K>(P, S, dcur, node, dg, inv, acc[0], acc[1], acc[2], acc[3], acc[4], acc[5], acc[6],
                 acc[7], kc, lane);
  }
}

// The in-edge ids and row data of a task this warp will run next, into L2.
__device__ __forceinline__ void prefetch_task(const DeltaParams& P, const TileDesc& d) {
  const uint32_t lane = threadIdx.x & 31;
  if (lane < 16) {
    if (lane * 32 < d.ne) prefetch_l2(P.in_nbr + d.e0 + lane * 32);
  } else if (d.npieces == 1) {
    const uint32_t l = lane - 16, last = d.nr - 1;
    if (l < 3) prefetch_l2(P.in_off + d.r0 + (l * 16 < d.nr ? l * 16 : d.nr));
    else if (l < 5) prefetch_l2(P.crow + d.r0 + (l == 3 ? 0 : last));
    else if (l < 7) prefetch_l2(P.cdeg + d.r0 + (l == 5 ? 0 : last));
    else if (l < 10) prefetch_l2(P.cinv + d.r0 + (l == 7 ? 0 : l == 8 ? (last < 16 ? last : 16) : last));
  }
}

// Sources without in-edges are not rows of the compacted transpose: their only
// inflow is the dead-end mass. Run by the warp that takes task 0 (wave 0).
template <int K>
__device__ __forceinline__ void delta_source_rows(const DeltaParams& P, DeltaSh<K>& S,
                                                  uint4* dcur) {
  const int lane = threadIdx.x & 31;
  for (int c = lane; c < K; c += 32) {
    const uint32_t u = S.csrc[c];
    // (the loop is warp-uniform: K / 32 rounds; lanes without such a row idle through it)
    const bool on = __ldg(P.in_off_full + u + 1) == __ldg(P.in_off_full + u);
    const uint64_t ix = (uint64_t)u * K + c;
    double rr = __ldcg(P.r + ix) + S.dd[c];
    const uint32_t dg = __ldg(P.deg + u);
    const double dthr = dg ? (double)dg : 1.0;
    const double oma = 1.0 - P.alpha;
    const double c1 = dg ? oma * __ldg(P.inv_deg + u) * ldexp(1.0, -DS_EXP) : 0.0;
    auto field = [&](int cc, double res) -> uint32_t {
      return res > dthr * S.thr[(cc / 8) * 10 + cc % 8] ? share_field(res * c1, cc & 1) : 0u;
    };
    uint32_t h = 0;
    double rp = 0.0;
    if (on && rr > dthr * S.thr[(c / 8) * 10 + c % 8]) {
      if (dg) {
        h = field(c, rr);
        double val = share_value(h);
        if ((c & 1) && h) {  // the even column of my word, if this node is its source too
          const uint32_t a = S.csrc[c - 1] == u ? field(c - 1, __ldcg(P.r + ix - 1) + S.dd[c - 1]) : 0u;
          val = value_b(a | (h << 16));
        }
        rp = h ? fmin(val * (dthr * P.inv_oma * ldexp(1.0, DS_EXP)), rr) : 0.0;
      } else {
        rp = rr;
        atomicAdd(&S.srcdead[c], oma * rp);
        atomicAdd(&S.nd[c], 1u);
      }
    }
    __syncwarp();  // (every lane has read its neighbour's residue before any is updated)
    if (rp > 0.0) {
      P.x[ix] = __ldcg(P.x + ix) + rp;
      rr -= rp;
      atomicAdd(&S.srcpush[c], rp);
      atomicAdd(&S.srcnn[c], 1u);
      atomicAdd(&S.srcnp[c], dg ? dg : 1u);
    }
    if (on) P.r[ix] = rr;
    // (other columns of this node's share row stay 0: it has no in-edges, so
    // it holds residue only in the columns it is the source of)
    if (on) reinterpret_cast<uint16_t*>(dcur)[2 * (uint64_t)u * K + c] = (uint16_t)h;
  }
  __syncwarp();
}

template <int K>
__global__ void __launch_bounds__(DS_NT, PPRG_DS_MINB) k_dsweeps(const __grid_constant__ DeltaParams P) {
  constexpr int LPR = K / 8, ES = 32 / LPR;
  extern __shared__ __align__(16) char ds_smem[];
  DeltaSh<K>& S = *reinterpret_cast<DeltaSh<K>*>(ds_smem);
  const int tid = threadIdx.x, lane = tid & 31;
  SweepCtl* ctl = P.ctl;
  for (int i = tid; i < 64; i += DS_NT) S.bloom[i] = 0;
  __syncthreads();
  if (tid < K) {
    const double rs = __ldcg(P.from_drain + tid);
    const int scan = tid < P.k_live && (P.scan_all || rs > P.scan_lambda);  // push.cpp:168
    int ep = 0;
    while (ep < P.E && !(rs > P.lam[ep])) ++ep;
    S.r_sum[tid] = rs;
    S.epoch[tid] = ep;
    S.done[tid] = !scan || ep >= P.E;
    S.sweeps[tid] = 0;
    S.pushes[tid] = 0;
    S.csrc[tid] = P.src[tid];
    S.dd[tid] = 0.0;
    atomicOr(&S.bloom[(P.src[tid] >> 5) & 63], 1u << (P.src[tid] & 31));
    if (blockIdx.x == 0) ctl->out_scan[tid] = scan;
  }
  __syncthreads();
  unsigned long long gen = 0;
  bool draining = false;  // the extra sweep that only consumes the shares in flight
  for (uint32_t sweep = 0;; ++sweep) {
    const int buf = sweep % 3;
    if (tid == 0) {
      int any = 0;
      for (int c = 0; c < K; ++c) any |= !S.done[c];
      S.any = any;
      S.known = 0;
    }
    for (int i = tid; i < DS_NW * 8 * 32; i += DS_NT) {
      (&S.pacc[0][0][0])[i] = 0.0;
      (&S.pdead[0][0][0])[i] = 0.0;
      (&S.pcnt[0][0][0])[i] = 0ull;
    }
    if (tid < K) {
      S.thr[(tid / 8) * 10 + tid % 8] = S.done[tid] ? CUDART_INF : P.thr[S.epoch[tid]];
      S.srcdead[tid] = 0.0;
      S.srcpush[tid] = 0.0;
      S.srcnn[tid] = S.srcnp[tid] = S.nd[tid] = 0;
    }
    __syncthreads();
    if (!S.any) {
      if (draining || sweep == 0) break;
      draining = true;
    }
    if (sweep >= P.max_sweeps) break;
    if (blockIdx.x == 0 && tid == 0) {
      const int nb = (sweep + 1) % 3;  // last read two barriers ago
      ctl->ticket[nb] = 0;
      for (int w = 0; w < DS_WMAX; ++w) ctl->wdone[nb][w] = 0;
      for (int c = 0; c < K; ++c) {
        ctl->pushed[nb][c] = 0;
        ctl->npush[nb][c] = 0;
        ctl->nnode[nb][c] = 0;
        ctl->dsum[nb][c] = 0;
        ctl->et[nb][c] = 0;
      }
    }
    // ---- the sweep: every warp takes tasks in id order, two per ticket -----
    const uint32_t par = sweep & 1u;
    uint4* dcur = P.dsh + par * LPR;  // row u of this sweep: dcur[2 u LPR + kc]
    auto grab = [&]() -> unsigned long long {
      unsigned t = 0;
      if (lane == 0) t = atomicAdd(&ctl->ticket[buf], 2u);
      return __shfl_sync(0xffffffffu, t, 0);
    };
    uint32_t wave = 0, known = 0, pending = 0;
    unsigned long long base = grab();
    while (base < P.ntiles) {
      const unsigned long long nbase = grab();  // one ahead
      if (nbase < P.ntiles) prefetch_l2(P.desc + nbase);
      for (unsigned long long j = base; j < base + 2 && j < P.ntiles; ++j) {
        const TileDesc d = P.desc[j];
#if PPRG_DS_PFTASK
        {  // the following task's ids and row data on their way into L2
          const unsigned long long jn = (j == base && j + 1 < P.ntiles) ? j + 1 : nbase;
          if (jn < P.ntiles) prefetch_task(P, P.desc[jn]);
        }
#endif
        while (j >= P.wave_tile[wave + 1]) ++wave;
        // every task of the waves <= wave - lag must have finished (their shares
        // are read from this sweep's buffer)
        const uint32_t need = wave >= P.lag ? wave - P.lag + 1 : 0;
        if (known < need) {
          // One acquire per block and wave (it invalidates the SM's L1): the
          // first warp to need a wave waits for it and publishes it to the
          // block's other warps through shared memory.
          if (lane == 0) {
            uint32_t kn = *(volatile uint32_t*)&S.known;
            if (kn < need) {
              for (; kn < need; ++kn) {
                const unsigned full = P.wave_tile[kn + 1] - P.wave_tile[kn];
                while (ld_acquire32(&ctl->wdone[buf][kn]) < full) __nanosleep(200);
              }
              __threadfence_block();
              atomicMax(&S.known, need);
            } else {
              __threadfence_block();
            }
          }
          __syncwarp();
          known = need;
        }
        DRow<K> X{P.dsh + lane % LPR, need ? P.wave_node[need] : 0u, par};
        if (j == 0) delta_source_rows<K>(P, S, dcur);
        delta_task<K>(P, S, d, j, X, dcur);
        // this task's shares are published: signalled once per pair of tasks (or
        // when the wave changes in between)
        const bool last = j + 1 >= base + 2 || j + 1 >= P.ntiles;
        ++pending;
        if (last || j + 1 >= P.wave_tile[wave + 1]) {
          __syncwarp();
          if (lane == 0)  // (a release, not a fence: no L1 invalidation on the publishing side)
            asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(&ctl->wdone[buf][wave]), "r"(pending) : "memory");
          pending = 0;
        }
      }
      base = nbase;
    }
    __syncthreads();
    // flush the block's sums: lane-group arrays -> one value per column
    if (tid < K) {
      double p = S.srcpush[tid], dm = S.srcdead[tid];
      unsigned long long np = S.srcnp[tid], nn = S.srcnn[tid];
      const int kq = tid % 8, kk = tid / 8;  // column tid = 8 kk + kq
      for (int wq = 0; wq < DS_NW; ++wq)
        for (int e = 0; e < ES; ++e) {
          p += S.pacc[wq][kq][e * LPR + kk];
          dm += S.pdead[wq][kq][e * LPR + kk];
          const unsigned long long pk = S.pcnt[wq][kq][e * LPR + kk];
          np += pk & ((1ull << 40) - 1);
          nn += pk >> 40;
        }
      if (p != 0.0) atomicAdd(&ctl->pushed[buf][tid], p);
      if (dm != 0.0) atomicAdd(&ctl->dsum[buf][tid], dm);
      if (np) atomicAdd(&ctl->npush[buf][tid], np);
      if (nn) atomicAdd(&ctl->nnode[buf][tid], nn);
      if (np) atomicAdd(&ctl->et[buf][tid], np - S.nd[tid]);
    }
    grid_barrier2(&ctl->gbar, ++gen);
    if (tid < K) {
      const double pushed = __ldcg(&ctl->pushed[buf][tid]);
      const unsigned long long np = __ldcg(&ctl->npush[buf][tid]);
      S.dd[tid] = __ldcg(&ctl->dsum[buf][tid]);
      if (!S.done[tid]) {
        S.sweeps[tid] += 1;
        S.pushes[tid] += np;
        S.r_sum[tid] -= P.alpha * pushed;
        if (np == 0) S.epoch[tid] += 1;  // fixpoint: nothing active at this threshold
        else if (S.epoch[tid] == P.E - 1 && np < P.handoff_np) S.epoch[tid] += 1;  // refine tail
        while (S.epoch[tid] < P.E && !(S.r_sum[tid] > P.lam[S.epoch[tid]])) S.epoch[tid] += 1;
        if (S.epoch[tid] >= P.E) S.done[tid] = 1;
      }
    }
    if (blockIdx.x == 0 && tid == 0) {
      // B = 8(n+1) + 8 k n + 4 E_t + 24 P_t over the live columns
      unsigned long long pt = 0, et = 0;
      for (int c = 0; c < P.k_live; ++c) {
        pt += __ldcg(&ctl->nnode[buf][c]);
        const unsigned long long e = __ldcg(&ctl->et[buf][c]);
        et = e > et ? e : et;
      }
      ctl->alg_bytes += 8ull * (P.n + 1) + 8ull * P.k_live * P.n + 4ull * et + 24ull * pt;
      ctl->total_sweeps = sweep + 1;
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && tid < K) {
    ctl->out_rsum[tid] = S.r_sum[tid];
    ctl->out_D[tid] = 0.0;
    ctl->out_sweeps[tid] = S.sweeps[tid];
    ctl->out_done[tid] = S.done[tid];
    ctl->out_epoch[tid] = S.epoch[tid];
    ctl->out_pushes[tid] = S.pushes[tid];
  }
}

// After the delta sweeps: query-major outputs through a shared-memory
// transpose (32 rows x K columns per step, 256-byte output segments) and the
// exact residue sum per column (push.cpp:9-15) into fctl->pushed[0].
template <int K>
__global__ void __launch_bounds__(256) k_delta_final(const double* x, const double* r, uint64_t n,
                                                     int k_live, double alpha, double* out_reserve,
                                                     double* out_residue, SweepCtl* fctl) {
  __shared__ double tx[32][K + 1], tr[32][K + 1];
  __shared__ double csum[K];
  const int tid = threadIdx.x;
  if (tid < K) csum[tid] = 0.0;
  double loc = 0.0;  // column tid % K (256 % K == 0)
  for (uint64_t u0 = (uint64_t)blockIdx.x * 32; u0 < n; u0 += (uint64_t)gridDim.x * 32) {
    const uint32_t rows = n - u0 < 32 ? (uint32_t)(n - u0) : 32u;
    __syncthreads();
    for (uint32_t i = tid; i < rows * K; i += 256) {
      const double rv = __ldcs(r + u0 * K + i);
      tr[i / K][i % K] = rv;
      loc += rv;
      if (out_reserve) tx[i / K][i % K] = __ldcs(x + u0 * K + i);
    }
    __syncthreads();
    for (uint32_t i = tid; i < 32u * k_live; i += 256) {
      const uint32_t c = i / 32, rr = i % 32;
      if (rr < rows) {
        if (out_reserve) __stcs(out_reserve + (uint64_t)c * n + u0 + rr, alpha * tx[rr][c]);
        if (out_residue) __stcs(out_residue + (uint64_t)c * n + u0 + rr, tr[rr][c]);
      }
    }
  }
  __syncthreads();
  if (loc != 0.0) atomicAdd(&csum[tid % K], loc);
  __syncthreads();
  if (tid < K) {
    if (csum[tid] != 0.0) atomicAdd(&fctl->pushed[0][tid], csum[tid]);
    if (blockIdx.x == 0) fctl->out_scale[tid] = 1.0;
  }
}

}  // namespace pprg
