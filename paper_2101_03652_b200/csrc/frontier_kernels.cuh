// Device side of the frontier (push-form) levels: the local phase of PowerPush,
// refine and FIFO forward push, plus the small per-block helper kernels.
// Included by push.cu only (one translation unit).
#pragma once
#include "sweep_kernel.cuh"

namespace pprg {
// ---- local phase / refine / FIFO: frontier levels in push form ------------
// Entry = (node v, column c) of the interleaved state i = v*K + c. Frontier of
// one level: per column c a FIFO segment seg[c*seg_cap, c*seg_cap + q_c) of
// node ids, so an entry's position in its segment is the number of pops of
// column c before it. One warp per entry: claim r (the FIFO pop,
// push.cpp:38-41), x += r, scatter (1-a) r / deg_eff over the out-edges
// (push.cpp:44-56) and append each newly active (t, c) once per level (stamp).
struct HeavyEntry {  // a frontier node whose scatter is spread over the grid
  uint64_t begin;    // first out-edge
  uint32_t deg;
  uint32_t c;
  double share;
};
constexpr uint32_t HEAVY_DEG = 2048;
constexpr uint32_t HEAVY_CHUNK = 1024;

// Where a level's scatter lands: residues, the enqueue test's thresholds and
// stamps, and column c's next segment with its append counter. DET: residues
// are fixed-point integers (value * sc[c]) in the same 8-byte slots, so their
// sums are exact and independent of the order of the atomics.
template <bool DET>
struct ScatterCtx {
  double* res;
  const uint32_t* deg;
  const double* thr;              // [K] enqueue threshold per unit of deg_eff (DET: * sc)
  const double* sc;               // [K] DET: fixed-point scale 2^S_c
  unsigned* stamp;
  unsigned tag;
  uint32_t* next;
  uint64_t seg_cap;
  int K;
  unsigned long long* col_cnt;    // [K] appends (= next segment length)
  unsigned long long* col_deg;    // [K] DET with a queue limit: sum of the appended deg_eff, else null
};

// Append t to column c's next segment once per level when it becomes active
// (drain_queue's enqueue test, push.cpp:49-53); one atomic per ballot group.
template <bool DET>
__device__ __forceinline__ void maybe_append(const ScatterCtx<DET>& C, bool app, uint32_t t, int c,
                                             uint32_t td, unsigned mask) {
  // every lane of the warp is here; `mask` is this lane's group (one column)
  const unsigned bal = __ballot_sync(0xffffffffu, app) & mask;
  if (DET && C.col_deg && bal) {
    const unsigned dsum = __reduce_add_sync(mask, app ? (td ? td : 1u) : 0u);
    if ((threadIdx.x & 31) == __ffs(bal) - 1) atomicAdd(C.col_deg + c, (unsigned long long)dsum);
  }
  if (app) {
    const int lane = threadIdx.x & 31, leader = __ffs(bal) - 1;
    unsigned long long basepos = 0;
    if (lane == leader) basepos = atomicAdd(C.col_cnt + c, (unsigned long long)__popc(bal));
    basepos = __shfl_sync(bal, basepos, leader);
    C.next[(uint64_t)c * C.seg_cap + basepos + __popc(bal & ((1u << lane) - 1u))] = t;
  }
}

// share added to (t, c), then the enqueue test on the new value. The degree
// of t is loaded before the atomic (independent of it).
template <bool DET>
__device__ __forceinline__ void relax_scatter(const ScatterCtx<DET>& C, uint32_t t, int c, double share,
                                              bool ok, unsigned mask) {
  bool app = false;
  uint32_t td = 0;
  if (ok) {
    const uint64_t ti = (uint64_t)t * C.K + c;
    td = __ldg(C.deg + t);
    double nv;
    if constexpr (DET) {
      const long long q = __double2ll_rn(share * C.sc[c]);
      nv = (double)(long long)(atomicAdd(reinterpret_cast<unsigned long long*>(C.res + ti),
                                         (unsigned long long)q) + (unsigned long long)q);
    } else {
      nv = atomicAdd(C.res + ti, share) + share;
    }
    if (nv > (double)(td ? td : 1) * C.thr[c])
      app = atomicExch(C.stamp + ti, C.tag) != C.tag;
  }
  maybe_append(C, app, t, c, td, mask);
}

// Scatter `share` over the de out-edges starting at b of an entry by its
// group of GL lanes (every lane of the warp calls this; de = 0 for lanes
// without an entry), four neighbour ids per lane in flight. Dead ends scatter
// to the column's source.
template <int GL>
__device__ __forceinline__ unsigned group_mask() {
  if constexpr (GL == 32) return 0xffffffffu;
  else return ((1u << GL) - 1u) << ((threadIdx.x & 31) / GL * GL);
}
template <bool DET, int GL>
__device__ __forceinline__ void group_scatter(const ScatterCtx<DET>& C, const uint32_t* nbr, uint64_t b,
                                              uint32_t d, uint32_t src_c, int c, double share,
                                              uint64_t de) {
  const int sub = (threadIdx.x & 31) % GL;
  const unsigned gm = group_mask<GL>();
  const unsigned most = __reduce_max_sync(0xffffffffu, (unsigned)de);  // warp-uniform trip count
  for (uint64_t q0 = 0; q0 < most; q0 += 4 * GL) {
    uint32_t t[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t qq = q0 + sub + GL * k;
      t[k] = qq < de ? (d ? __ldg(nbr + b + qq) : src_c) : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) relax_scatter(C, t[k], c, share, t[k] != 0xFFFFFFFFu, gm);
  }
}

// The scatter of one HEAVY_CHUNK-edge chunk of a heavy entry by one block,
// four neighbour ids per thread loaded before the first atomic. Every lane of
// a chunk shares the entry's column, so appends group the whole warp.
template <bool DET>
__device__ __forceinline__ void heavy_chunk(const ScatterCtx<DET>& C, const uint32_t* nbr,
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

// ---- the drain: all levels of drain_queue (push.cpp:34-59) in one
// cooperative launch, or one level per launch for observed / traced calls.
// Per level:
//   entries (warp per entry; heavy entries queued) | grid barrier |
//   heavy entries (chunks of HEAVY_CHUNK edges, enumerated on the device from
//   a block-wide scan of their chunk counts) | grid barrier |
//   every block derives the next level from the reduced counters:
//   r_sum -= alpha * pushed, queue sizes, the stop tests.
// Level counters are triple-buffered (slot = level % 3); slot level+1 is
// cleared during `level` by block 0, two barriers after its last reader.
//
// Fast mode: the pop (atomicExch) races with the same level's scatters to the
// same entry, and the queue-limit test (push.cpp:38) runs before every pop
// against the out-degrees reserved by the pops so far.
// DET (PPRG_DETERMINISTIC): bitwise-reproducible. Every pop of a level
// happens before any of its scatters (pop phase | grid barrier | scatter
// phase), residues are fixed-point integers while the drain runs (exact,
// order-independent sums), the queue limit is tested at level boundaries,
// and the pushed mass is summed as integers. The set of entries of every
// level is then a function of the inputs; their order in a segment is not,
// and nothing depends on it.
struct DrainCtl {
  GridBarrier gbar;
  unsigned long long cnt[3][KMAX];   // appends per column (next queue size)
  unsigned long long np[3][KMAX];    // edge pushes
  unsigned long long nn[3][KMAX];    // node pushes
  unsigned long long resv[3][KMAX];  // out-degrees reserved by pops (queue-limit test)
  unsigned long long qdeg[3][KMAX];  // DET: sum of deg_eff over the appended entries
  double dr[3][KMAX];                // alpha * pushed residue (fast mode)
  unsigned long long dq[3][KMAX];    // pushed residue, fixed point (DET)
  unsigned stop[3][KMAX];            // queue outgrew the limit
  unsigned heavy_cnt[3];
  unsigned levels_run;
  double out_rsum[KMAX];
  unsigned long long out_np[KMAX];
  unsigned long long out_q[KMAX];
  unsigned long long out_qdeg[KMAX];
  unsigned out_levels[KMAX];
  unsigned long long out_live;
  unsigned long long scan_cnt[KMAX];  // initial frontier sizes of a scan start
  double out_exact[KMAX];             // recompute_r_sum (push.cpp:9-15) of every column at the end
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
  unsigned long long* popv;          // DET: popped value of segment slot [c*seg_cap + pos]
  unsigned long long limit;          // queue limit (~0: none)
  unsigned long long live0;          // columns draining
  double lam_stop;                   // r_sum stop (0: none)
  double alpha;
  uint64_t n;
  unsigned tag0;                     // level L stamps tag0 + L + 1 (no wrap: host-checked)
  unsigned max_levels;
  int K;
  uint32_t src[KMAX];
  double thr[KMAX];
  double r_sum0[KMAX];
  unsigned long long q0[KMAX];       // first level's queue sizes (start = 0)
  unsigned long long qdeg0[KMAX];    // DET: first level's sum of deg_eff (start = 0)
  int start;                         // 0: seg[0] holds the first level (q0); 1: seed_source
                                     // (push.cpp:61-66); 2: scan every active node in id order
                                     // (refine, push.cpp:212-218); both tested against thr
  int want_exact;                    // sum every column's residues at the end (out_exact)
  double* part;                      // DET exact sums: per-block partials [gridDim][KMAX]
  double sc[KMAX];                   // DET: fixed-point scale 2^S_c (all residues < 2^61 / sc)
};

constexpr int DRAIN_NT = 256;
constexpr unsigned DRAIN_HSH = 2048;  // heavy entries whose chunk prefix is kept in shared memory

template <bool DET, int GL>
__global__ void __launch_bounds__(DRAIN_NT) k_drain(const __grid_constant__ DrainParams D) {
  constexpr int NG = 32 / GL;  // entries per warp at a time
  __shared__ double s_rsum[KMAX], s_thr[KMAX], s_sc[KMAX];
  __shared__ uint32_t s_src[KMAX];
  __shared__ unsigned long long s_q[KMAX], s_pre[KMAX + 1], s_np[KMAX], s_qd[KMAX];
  __shared__ unsigned s_lv[KMAX];
  __shared__ unsigned long long s_live;
  __shared__ double sh_dr[KMAX];
  __shared__ unsigned long long sh_np[KMAX], sh_nn[KMAX], sh_dq[KMAX];
  __shared__ unsigned s_hpre[DRAIN_HSH + 1];
  using Scan = cub::BlockScan<unsigned, DRAIN_NT>;
  __shared__ typename Scan::TempStorage scan_tmp;
  const int tid = threadIdx.x, lane = tid & 31;
  const int gid = lane / GL, sub = lane % GL;  // entry group of this lane, lane in the group
  const int K = D.K;
  DrainCtl* ctl = D.ctl;
  if (tid < KMAX) {
    s_rsum[tid] = D.r_sum0[tid];
    s_sc[tid] = D.sc[tid];
    s_thr[tid] = DET ? D.thr[tid] * D.sc[tid] : D.thr[tid];
    s_src[tid] = D.src[tid];
    s_q[tid] = D.q0[tid];
    s_qd[tid] = D.qdeg0[tid];
    s_np[tid] = 0;
    s_lv[tid] = 0;
  }
  if (tid == 0) s_live = D.live0;
  __syncthreads();
  const uint64_t gtid = blockIdx.x * (uint64_t)DRAIN_NT + tid;
  const uint64_t gthreads = (uint64_t)gridDim.x * DRAIN_NT;
  const uint64_t nk = D.n * (uint64_t)K;
  unsigned long long gen = 0;
  // ---- the first level -----------------------------------------------------
  if (D.start == 1) {  // seed_source: the source alone if it is active
    if (tid < K && ((D.live0 >> tid) & 1ull)) {
      const uint32_t d = D.deg[s_src[tid]];
      const uint64_t de = d ? d : 1;
      const bool act = 1.0 > (double)de * D.thr[tid];
      s_q[tid] = act ? 1 : 0;
      s_qd[tid] = act ? de : 0;
      if (act && blockIdx.x == 0) D.seg[0][(uint64_t)tid * D.seg_cap] = s_src[tid];
    }
  } else if (D.start == 2) {  // every active (u, c) in id order; order within a
                              // segment follows warp-aggregated appends
    for (uint64_t i0 = blockIdx.x * (uint64_t)DRAIN_NT; i0 < nk; i0 += gthreads) {
      const uint64_t i = i0 + tid;
      const bool in = i < nk;
      const int c = in ? (int)(i % K) : -1;
      const uint32_t d = in ? D.deg[i / K] : 0;
      const bool act = in && ((D.live0 >> c) & 1ull) && D.res[i] > (double)(d ? d : 1) * D.thr[c];
      const unsigned grp = __match_any_sync(0xffffffffu, c);
      const unsigned bal = __ballot_sync(0xffffffffu, act) & grp;
      if (act) {
        D.stamp[i] = D.tag0;
        const int leader = __ffs(bal) - 1;
        unsigned long long b = 0;
        if (lane == leader) b = atomicAdd(ctl->scan_cnt + c, (unsigned long long)__popc(bal));
        b = __shfl_sync(bal, b, leader);
        D.seg[0][(uint64_t)c * D.seg_cap + b + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)(i / K);
      }
    }
    grid_barrier2(&ctl->gbar, ++gen);
    if (tid < K) s_q[tid] = __ldcg(&ctl->scan_cnt[tid]);
  }
  if (D.start) {  // the first loop test (drain_queue, push.cpp:38)
    __syncthreads();
    if (tid < K && ((D.live0 >> tid) & 1ull)) {
      const unsigned long long q = s_q[tid];
      const bool still = q > 0 && (DET && D.limit != ~0ull ? q + s_qd[tid] <= D.limit : q <= D.limit) &&
                         !(D.lam_stop > 0 && s_rsum[tid] <= D.lam_stop);
      if (!still) atomicAnd(&s_live, ~(1ull << tid));
    }
    __syncthreads();
  }
  if constexpr (DET) {  // residues of the draining columns to fixed point
    for (uint64_t i = gtid; i < nk; i += gthreads) {
      const int c = (int)(i % K);
      if ((D.live0 >> c) & 1ull)
        reinterpret_cast<long long*>(D.res)[i] = __double2ll_rn(D.res[i] * s_sc[c]);
    }
  }
  if (DET || D.start == 1) grid_barrier2(&ctl->gbar, ++gen);
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
    if (tid < KMAX) sh_dr[tid] = 0.0, sh_np[tid] = 0, sh_nn[tid] = 0, sh_dq[tid] = 0;
    __syncthreads();
    const unsigned long long total = s_pre[K];
    if (total == 0 || level >= D.max_levels) break;  // identical in every block
    if (blockIdx.x == 0 && tid < KMAX) {
      const int ns = (int)((level + 1) % 3);
      ctl->cnt[ns][tid] = 0;
      ctl->np[ns][tid] = 0;
      ctl->nn[ns][tid] = 0;
      ctl->resv[ns][tid] = 0;
      ctl->qdeg[ns][tid] = 0;
      ctl->dr[ns][tid] = 0.0;
      ctl->dq[ns][tid] = 0;
      ctl->stop[ns][tid] = 0;
      if (tid == 0) ctl->heavy_cnt[ns] = 0;
    }
    const ScatterCtx<DET> C{D.res, D.deg, s_thr, s_sc, D.stamp, D.tag0 + level + 1,
                            D.seg[(level + 1) & 1], D.seg_cap, K, ctl->cnt[slot],
                            DET && D.limit != ~0ull ? ctl->qdeg[slot] : nullptr};
    const uint32_t* cur = D.seg[level & 1];
    // entries are taken NG = 32/GL at a time per warp, GL lanes per entry:
    // the pop chain (claim, then scatter, then append) of NG entries is in
    // flight at once instead of one
    const uint64_t w0 = (gtid >> 5) * NG, nw = (gthreads >> 5) * NG;
    // ---- pops (fast mode: and their scatters) ------------------------------
    for (uint64_t w = w0; w < total; w += nw) {
      const uint64_t e = w + gid;
      const bool valid = e < total;
      int c = 0;
      uint64_t pos = 0, seg_i = 0, de = 1, b = 0, i = 0;
      uint32_t d = 0;
      if (valid) {
        while (e >= s_pre[c + 1]) ++c;
        pos = e - s_pre[c];
        seg_i = (uint64_t)c * D.seg_cap + pos;
        const uint32_t v = cur[seg_i];
        i = (uint64_t)v * K + c;
        d = D.deg[v];
        de = d ? d : 1;
        b = D.off[v];
      }
      double r = 0.0;
      unsigned long long rq = 0;
      if (valid && sub == 0) {
        if constexpr (DET) {
          rq = atomicExch(reinterpret_cast<unsigned long long*>(D.res) + i, 0ull);
          D.popv[seg_i] = rq;
          r = (double)(long long)rq / s_sc[c];
        } else {
          bool stop = false;
          if (D.limit != ~0ull) {
            stop = *(volatile unsigned*)(ctl->stop[slot] + c) != 0;
            if (!stop) {
              // appends of the pops before this one are bounded by their
              // out-degrees, reserved at pop time, so concurrent warps see the
              // queue growth at once
              const unsigned long long reserved = atomicAdd(ctl->resv[slot] + c, de);
              if (s_pre[c + 1] - s_pre[c] - pos + reserved > D.limit) {
                stop = true;
                ctl->stop[slot][c] = 1;
              }
            }
          }
          if (!stop)
            r = __longlong_as_double((long long)atomicExch((unsigned long long*)(D.res + i), 0ull));
        }
      }
      r = __shfl_sync(0xffffffffu, r, gid * GL);
      const bool ok = r > 0.0;
      const double share = (1.0 - D.alpha) * r / (double)de;
      if (ok && sub == 0) {
        D.x[i] += r;
        if constexpr (DET) atomicAdd(&sh_dq[c], rq);
        else atomicAdd(&sh_dr[c], D.alpha * r);
        atomicAdd(&sh_np[c], (unsigned long long)de);
        atomicAdd(&sh_nn[c], 1ull);
        if (de > HEAVY_DEG) D.heavy[atomicAdd(&ctl->heavy_cnt[slot], 1u)] = HeavyEntry{b, d, (uint32_t)c, share};
      }
      if constexpr (!DET)
        group_scatter<DET, GL>(C, D.nbr, b, d, s_src[c], c, share, ok && de <= HEAVY_DEG ? de : 0);
    }
    __syncthreads();
    if (tid < K) {
      if (sh_dr[tid] != 0.0) atomicAdd(&ctl->dr[slot][tid], sh_dr[tid]);
      if (sh_dq[tid]) atomicAdd(&ctl->dq[slot][tid], sh_dq[tid]);
      if (sh_np[tid]) atomicAdd(&ctl->np[slot][tid], sh_np[tid]);
      if (sh_nn[tid]) atomicAdd(&ctl->nn[slot][tid], sh_nn[tid]);
    }
    grid_barrier2(&ctl->gbar, ++gen);
    if constexpr (DET) {  // ---- scatters, after every pop of the level ----------
      for (uint64_t w = w0; w < total; w += nw) {
        const uint64_t e = w + gid;
        int c = 0;
        uint64_t de = 0, b = 0;
        uint32_t d = 0;
        double share = 0.0;
        if (e < total) {
          while (e >= s_pre[c + 1]) ++c;
          const uint64_t seg_i = (uint64_t)c * D.seg_cap + (e - s_pre[c]);
          const long long rq = (long long)__ldcg(D.popv + seg_i);
          if (rq > 0) {
            const uint32_t v = __ldcg(cur + seg_i);
            d = D.deg[v];
            const uint64_t dd = d ? d : 1;
            if (dd <= HEAVY_DEG) {
              de = dd;
              b = D.off[v];
              share = (1.0 - D.alpha) * ((double)rq / s_sc[c]) / (double)dd;
            }
          }
        }
        group_scatter<DET, GL>(C, D.nbr, b, d, s_src[c], c, share, de);
      }
    }
    const unsigned nh = __ldcg(&ctl->heavy_cnt[slot]);
    if (nh) {  // ---- heavy entries ------------------------------------------
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
    }
    if (DET || nh) grid_barrier2(&ctl->gbar, ++gen);
    // ---- the next level, identically in every block (drain_queue's loop test)
    if (tid < K && ((s_live >> tid) & 1ull)) {
      if constexpr (DET)
        s_rsum[tid] -= D.alpha * ((double)(long long)__ldcg(&ctl->dq[slot][tid]) / s_sc[tid]);
      else
        s_rsum[tid] -= __ldcg(&ctl->dr[slot][tid]);
      s_np[tid] += __ldcg(&ctl->np[slot][tid]);
      s_lv[tid] += 1;
      const unsigned long long q = __ldcg(&ctl->cnt[slot][tid]);
      s_q[tid] = q;
      // DET: a level runs only if no sequence of its pops can take the queue
      // past the limit (its entries' deg_eff bound their appends); the fast
      // mode stops mid-level at the first pop that could
      const unsigned long long qd = __ldcg(&ctl->qdeg[slot][tid]);
      s_qd[tid] = qd;
      const bool still = q > 0 && (DET && D.limit != ~0ull ? q + qd <= D.limit : q <= D.limit) &&
                         !(D.lam_stop > 0 && s_rsum[tid] <= D.lam_stop);
      if (__ldcg(&ctl->stop[slot][tid]) || !still) atomicAnd(&s_live, ~(1ull << tid));
    }
    __syncthreads();
  }
  if constexpr (DET) {  // back to doubles (every scatter completed before the last barrier)
    for (uint64_t i = gtid; i < nk; i += gthreads) {
      const int c = (int)(i % K);
      if ((D.live0 >> c) & 1ull)
        D.res[i] = (double)reinterpret_cast<const long long*>(D.res)[i] / s_sc[c];
    }
  }
  if (D.want_exact) {  // recompute_r_sum (push.cpp:9-15) of every column
    if (DET) grid_barrier2(&ctl->gbar, ++gen);
    // the grid stride is a multiple of K: each thread sums one column, in order
    double t = 0.0;
    for (uint64_t i = gtid; i < nk; i += gthreads) t += D.res[i];
    __shared__ double sh_col[DRAIN_NT];
    sh_col[tid] = t;
    __syncthreads();
    if (tid < K) {
      double bsum = 0.0;
      for (int g2 = 0; g2 < DRAIN_NT / K; ++g2) bsum += sh_col[g2 * K + tid];  // fixed order
      if constexpr (DET) D.part[(uint64_t)blockIdx.x * KMAX + tid] = bsum;
      else atomicAdd(&ctl->out_exact[tid], bsum);
    }
    if constexpr (DET) {
      grid_barrier2(&ctl->gbar, ++gen);
      if (blockIdx.x == 0 && tid < K) {
        double e = 0.0;
        for (unsigned b = 0; b < gridDim.x; ++b) e += __ldcg(D.part + (uint64_t)b * KMAX + tid);
        ctl->out_exact[tid] = e;
      }
    }
  }
  if (blockIdx.x == 0 && tid < KMAX) {
    ctl->out_rsum[tid] = s_rsum[tid];
    ctl->out_np[tid] = s_np[tid];
    ctl->out_q[tid] = s_q[tid];
    ctl->out_qdeg[tid] = s_qd[tid];
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

// Deterministic per-column sums (PPRG_DETERMINISTIC): out[c] = scale *
// sum over rows r of a[row(r)*K + c], row(r) = rows ? rows[r] : r. A fixed
// grid of DSUM_BLOCKS blocks; thread t of a block owns column t % K and a
// fixed stride of rows, summed in order; the block's row groups meet in a
// fixed order in shared memory, and k_dsum_final adds the blocks' partials in
// block order. Same bits on every run and every device.
constexpr int DSUM_BLOCKS = 296;
constexpr int DSUM_NT = 256;
__global__ void __launch_bounds__(DSUM_NT) k_dsum_part(const double* a, const uint32_t* rows,
                                                       uint64_t nrows, int K, double* part) {
  __shared__ double sh[DSUM_NT];
  const int tid = threadIdx.x;
  const int groups = DSUM_NT / K;  // K divides 256 (a power of two <= 64)
  const int c = tid % K, grp = tid / K;
  double s = 0.0;
  for (uint64_t r = (uint64_t)blockIdx.x * groups + grp; r < nrows; r += (uint64_t)gridDim.x * groups) {
    const uint64_t row = rows ? rows[r] : r;
    s += a[row * K + c];
  }
  sh[tid] = s;
  __syncthreads();
  if (tid < K) {
    double t = 0.0;
    for (int g2 = 0; g2 < groups; ++g2) t += sh[g2 * K + tid];
    part[(uint64_t)blockIdx.x * K + tid] = t;
  }
}
__global__ void k_dsum_final(const double* part, int nblocks, int K, double scale, double* out) {
  const int c = threadIdx.x;
  if (c >= K) return;
  double t = 0.0;
  for (int b = 0; b < nblocks; ++b) t += part[(uint64_t)b * K + c];
  out[c] = scale * t;
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
