// Design probe (not product code): which gather engine moves the 64-column
// pull sweep's 512-byte y rows fastest on B200? The real configs[2] transpose
// (R-MAT 22/16 seed 3, relabelled) is read from a file written by
// tools/microbench/dump_transpose.py. Every variant sums y over the in-edges of
// edge-balanced pieces of <= PL in-edges and writes one 64-column sum per
// piece (no decisions, no atomics), so the time is the gather engine alone:
//   reg   : G row loads (ld.global.v2.f64 per lane) in registers, then add
//   regpp : the same, software-pipelined: the next G loads are issued before
//           the current G are added (2G in flight)
//   lgs   : cp.async.cg 16 B per lane into a per-warp ring of D rows
//           (commit/wait_group), the warp streams edges across pieces
//   bulk  : cp.async.bulk of the 512-byte row into a per-warp ring of D rows,
//           one mbarrier per slot, issued by one lane per edge
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ge gather_engines.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <functional>
#include <cmath>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

constexpr int K = 64;

struct Piece {
  uint64_t e0;
  uint32_t ne, row;
};

__device__ __forceinline__ double2 ldg2(const double* p) {
  double2 v;
  asm volatile("ld.global.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// cp.async.bulk ring: lane (e % 32) issues edge e's 512-byte copy; slot mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* m, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(m)),
               "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint64_t* m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(m)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, unsigned parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(m);
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* m) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(m))
      : "memory");
}

// ---- reg: one warp per piece (grid-stride), G loads in flight -----------------
template <int G>
__global__ void __launch_bounds__(128, 8) k_reg(const Piece* pc, uint64_t npc, const uint32_t* nbr,
                                                const double* y, double* out) {
  const int lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t p = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; p < npc; p += nw) {
    const Piece d = pc[p];
    double ax = 0, ay = 0;
    for (uint32_t b = 0; b < d.ne; b += 32) {
      const uint32_t myid = b + lane < d.ne ? nbr[d.e0 + b + lane] : 0u;
      const int cnt = d.ne - b < 32 ? d.ne - b : 32;
      for (int j0 = 0; j0 < cnt; j0 += G) {
        double2 v[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int j = j0 + g;
          const uint32_t id = __shfl_sync(0xffffffffu, myid, j < cnt ? j : cnt - 1);
          v[g] = ldg2(y + (uint64_t)id * K + 2 * lane);
        }
#pragma unroll
        for (int g = 0; g < G; ++g)
          if (j0 + g < cnt) {
            ax += v[g].x;
            ay += v[g].y;
          }
      }
    }
    reinterpret_cast<double2*>(out + p * K)[lane] = make_double2(ax, ay);
  }
}

// ---- reg with per-gather L2 policy: bit 31 of an in-edge id marks a hot
// source (top out-degree): MODE 1 hot evict_last / cold evict_first,
// MODE 2 hot evict_last / cold normal, MODE 3 hot normal / cold evict_first;
// the id stream is evict_first in every mode.
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ldg2_pol(const double* p, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ldid_first(const uint32_t* p) {
  uint32_t v;
  asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol_first()));
  return v;
}
template <int G, int MODE>
__global__ void __launch_bounds__(128, 8) k_reg_hint(const Piece* pc, uint64_t npc, const uint32_t* nbr,
                                                     const double* y, double* out) {
  const int lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t pf = pol_first(), pl = pol_last();
  for (uint64_t p = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; p < npc; p += nw) {
    const Piece d = pc[p];
    double ax = 0, ay = 0;
    for (uint32_t b = 0; b < d.ne; b += 32) {
      const uint32_t myid = b + lane < d.ne ? ldid_first(nbr + d.e0 + b + lane) : 0u;
      const int cnt = d.ne - b < 32 ? d.ne - b : 32;
      for (int j0 = 0; j0 < cnt; j0 += G) {
        double2 v[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int j = j0 + g;
          const uint32_t raw = __shfl_sync(0xffffffffu, myid, j < cnt ? j : cnt - 1);
          const bool hot = raw >> 31;
          const double* src = y + (uint64_t)(raw & 0x7FFFFFFFu) * K + 2 * lane;
          if (MODE == 1) v[g] = ldg2_pol(src, hot ? pl : pf);
          else if (MODE == 2) v[g] = hot ? ldg2_pol(src, pl) : ldg2(src);
          else v[g] = hot ? ldg2(src) : ldg2_pol(src, pf);
        }
#pragma unroll
        for (int g = 0; g < G; ++g)
          if (j0 + g < cnt) {
            ax += v[g].x;
            ay += v[g].y;
          }
      }
    }
    reinterpret_cast<double2*>(out + p * K)[lane] = make_double2(ax, ay);
  }
}

// ---- stream: a warp walks a contiguous, piece-aligned edge range as one
// stream; bit 31 of an in-edge id marks the last edge of its piece, so the
// warp keeps G row loads in flight whatever the row lengths. PIPE = 1: groups
// of G double-buffered (the next group is issued before this one is added).
template <int G, int PIPE>
__global__ void __launch_bounds__(128, 8) k_stream(const Piece* pc, uint64_t npc, const uint32_t* nbr,
                                                   const double* y, double* out) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t m = pc[npc - 1].e0 + pc[npc - 1].ne;
  auto first_piece = [&](uint64_t edge) {
    uint64_t lo = 0, hi = npc;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (pc[mid].e0 < edge) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  const uint64_t p0 = first_piece(m * w / nw), p1 = first_piece(m * (w + 1) / nw);
  if (p0 >= p1) return;
  const uint64_t E0 = pc[p0].e0, E1 = p1 < npc ? pc[p1].e0 : m;
  uint64_t piece = p0;
  double ax = 0, ay = 0;
  uint32_t ids = E0 + lane < E1 ? __ldg(nbr + E0 + lane) : 0u;
  for (uint64_t c0 = E0; c0 < E1; c0 += 32) {
    const uint64_t cn = c0 + 32;
    const uint32_t ids_n = cn + lane < E1 ? __ldg(nbr + cn + lane) : 0u;  // next chunk, early
    const int cnt = E1 - c0 < 32 ? (int)(E1 - c0) : 32;
    if (PIPE == 0) {
      for (int j0 = 0; j0 < cnt; j0 += G) {
        double2 v[G];
        uint32_t ends = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int j = j0 + g < cnt ? j0 + g : cnt - 1;
          const uint32_t raw = __shfl_sync(0xffffffffu, ids, j);
          ends |= (raw >> 31) << g;
          v[g] = ldg2(y + (uint64_t)(raw & 0x7FFFFFFFu) * K + 2 * lane);
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          if (j0 + g >= cnt) break;
          ax += v[g].x;
          ay += v[g].y;
          if ((ends >> g) & 1u) {
            reinterpret_cast<double2*>(out + piece * K)[lane] = make_double2(ax, ay);
            ++piece;
            ax = ay = 0;
          }
        }
      }
    } else {
      double2 v[2][G];
      uint32_t ends[2] = {0, 0};
      auto issue = [&](int j0, int b) {
        ends[b] = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int j = j0 + g < cnt ? j0 + g : cnt - 1;
          const uint32_t raw = __shfl_sync(0xffffffffu, ids, j);
          ends[b] |= (raw >> 31) << g;
          v[b][g] = ldg2(y + (uint64_t)(raw & 0x7FFFFFFFu) * K + 2 * lane);
        }
      };
      issue(0, 0);
#pragma unroll
      for (int q = 0; q < 32 / G; ++q) {
        const int j0 = q * G;
        if (j0 >= cnt) break;
        if (j0 + G < cnt) issue(j0 + G, (q + 1) & 1);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          if (j0 + g >= cnt) break;
          ax += v[q & 1][g].x;
          ay += v[q & 1][g].y;
          if ((ends[q & 1] >> g) & 1u) {
            reinterpret_cast<double2*>(out + piece * K)[lane] = make_double2(ax, ay);
            ++piece;
            ax = ay = 0;
          }
        }
      }
    }
    ids = ids_n;
  }
}

// ---- stream + L2 prefetch: as k_stream<G,0>, and each lane bulk-prefetches
// into L2 the 512-byte row of its edge PF chunks (of 32 edges) ahead, so the
// register gathers mostly hit L2. PF = 0: no prefetch.
__device__ __forceinline__ void l2_prefetch_row(const double* p) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], 512;" ::"l"(p) : "memory");
}
template <int G, int PF>
__global__ void __launch_bounds__(128, 8) k_stream_pf(const Piece* pc, uint64_t npc, const uint32_t* nbr,
                                                      const double* y, double* out) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t m = pc[npc - 1].e0 + pc[npc - 1].ne;
  auto first_piece = [&](uint64_t edge) {
    uint64_t lo = 0, hi = npc;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (pc[mid].e0 < edge) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  const uint64_t p0 = first_piece(m * w / nw), p1 = first_piece(m * (w + 1) / nw);
  if (p0 >= p1) return;
  const uint64_t E0 = pc[p0].e0, E1 = p1 < npc ? pc[p1].e0 : m;
  uint64_t piece = p0;
  double ax = 0, ay = 0;
  auto ld_ids = [&](uint64_t c) -> uint32_t { return c + lane < E1 ? __ldg(nbr + c + lane) : 0xFFFFFFFFu; };
  auto pf = [&](uint32_t raw) {
    if (raw != 0xFFFFFFFFu) l2_prefetch_row(y + (uint64_t)(raw & 0x7FFFFFFFu) * K);
  };
  uint32_t ids = ld_ids(E0);
  uint32_t q1 = ld_ids(E0 + 32), q2 = PF >= 2 ? ld_ids(E0 + 64) : 0u;
  if (PF >= 1) pf(ids);
  if (PF >= 1) pf(q1);
  if (PF >= 2) pf(q2);
  for (uint64_t c0 = E0; c0 < E1; c0 += 32) {
    // ids of the chunk PF+1 ahead: loaded now, prefetched next round
    uint32_t qn = 0;
    if (PF >= 1) {
      qn = ld_ids(c0 + 32 * (PF + 1));
    }
    const int cnt = E1 - c0 < 32 ? (int)(E1 - c0) : 32;
    for (int j0 = 0; j0 < cnt; j0 += G) {
      double2 v[G];
      uint32_t ends = 0;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int j = j0 + g < cnt ? j0 + g : cnt - 1;
        const uint32_t raw = __shfl_sync(0xffffffffu, ids, j);
        ends |= (raw >> 31) << g;
        v[g] = ldg2(y + (uint64_t)(raw & 0x7FFFFFFFu) * K + 2 * lane);
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (j0 + g >= cnt) break;
        ax += v[g].x;
        ay += v[g].y;
        if ((ends >> g) & 1u) {
          reinterpret_cast<double2*>(out + piece * K)[lane] = make_double2(ax, ay);
          ++piece;
          ax = ay = 0;
        }
      }
    }
    if (PF == 0) {
      ids = q1;
      q1 = ld_ids(c0 + 64);
    } else if (PF == 1) {
      ids = q1;
      q1 = qn;
      pf(q1);
    } else {
      ids = q1;
      q1 = q2;
      q2 = qn;
      pf(q2);
    }
  }
}

// ---- TMA gather4: y as a 2D tensor map [n rows x 64 f64]; a warp streams
// its edge range in chunks of 32 edges = 8 gather4 ops (2 KB each) into a
// ring of R chunk buffers (16 KB each), one mbarrier per buffer.
__device__ __forceinline__ void tma_gather4(uint32_t dst, const void* tmap, uint32_t mbar, int r0,
                                            int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
      "l"(tmap), "r"(mbar), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}
template <int R, int WPB>
__global__ void __launch_bounds__(WPB * 32) k_tma(const __grid_constant__ CUtensorMap tmap, const Piece* pc,
                                                 uint64_t npc, const uint32_t* nbr, double* out) {
  extern __shared__ __align__(1024) double tma_ring[];
  __shared__ __align__(8) uint64_t tbar[WPB * R];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* ring = tma_ring + (size_t)warp * R * 32 * K;
  uint64_t* bars = tbar + warp * R;
  if (lane < R) mbar_init(bars + lane, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const uint64_t w = blockIdx.x * (uint64_t)WPB + warp;
  const uint64_t nw = (uint64_t)gridDim.x * WPB;
  const uint64_t m = pc[npc - 1].e0 + pc[npc - 1].ne;
  auto first_piece = [&](uint64_t edge) {
    uint64_t lo = 0, hi = npc;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (pc[mid].e0 < edge) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  const uint64_t p0 = first_piece(m * w / nw), p1 = first_piece(m * (w + 1) / nw);
  if (p0 >= p1) return;
  const uint64_t E0 = pc[p0].e0, E1 = p1 < npc ? pc[p1].e0 : m;
  const uint64_t nchunks = (E1 - E0 + 31) / 32;
  uint32_t idsbuf[R];
  auto issue = [&](uint64_t ch, int b) {  // chunk ch into buffer b; returns the chunk's ids
    const uint64_t e = E0 + ch * 32 + lane;
    const uint32_t raw = e < E1 ? __ldg(nbr + e) : 0u;
    const int row = (int)(raw & 0x7FFFFFFFu);
    const int r1 = __shfl_down_sync(0xffffffffu, row, 1);
    const int r2 = __shfl_down_sync(0xffffffffu, row, 2);
    const int r3 = __shfl_down_sync(0xffffffffu, row, 3);
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(bars + b);
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(bars + b, 32 * K * 8);
    }
    __syncwarp();
    if ((lane & 3) == 0)
      tma_gather4((uint32_t)__cvta_generic_to_shared(ring + ((size_t)b * 32 + lane) * K), &tmap, mb,
                  row, r1, r2, r3);
    return raw;
  };
  for (int b = 0; b < R; ++b) idsbuf[b] = (uint64_t)b < nchunks ? issue(b, b) : 0u;
  uint64_t piece = p0;
  double ax = 0, ay = 0;
  for (uint64_t ch = 0; ch < nchunks; ++ch) {
    const int b = (int)(ch % R);
    mbar_wait(bars + b, (unsigned)((ch / R) & 1));
    const uint32_t ids = idsbuf[0];
    const int cnt = E1 - (E0 + ch * 32) < 32 ? (int)(E1 - (E0 + ch * 32)) : 32;
    const double2* rows = reinterpret_cast<const double2*>(ring + (size_t)b * 32 * K);
    for (int j = 0; j < cnt; ++j) {
      const uint32_t raw = __shfl_sync(0xffffffffu, ids, j);
      const double2 v = rows[j * (K / 2) + lane];
      ax += v.x;
      ay += v.y;
      if (raw >> 31) {
        reinterpret_cast<double2*>(out + piece * K)[lane] = make_double2(ax, ay);
        ++piece;
        ax = ay = 0;
      }
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q + 1 < R; ++q) idsbuf[q] = idsbuf[q + 1];
    idsbuf[R - 1] = ch + R < nchunks ? issue(ch + R, b) : 0u;
  }
}

// ---- edge streams: a warp owns a contiguous run of pieces and walks their
// edges as one stream; `issue(e)` starts edge e's row, `row(e)` returns it.
struct WarpRun {
  uint64_t p0, p1;  // pieces
};
// edge-balanced: warp w starts at the first piece whose first edge is >= m*w/nw
__device__ __forceinline__ uint64_t first_piece_at(const Piece* pc, uint64_t npc, uint64_t edge) {
  uint64_t lo = 0, hi = npc;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (pc[mid].e0 < edge) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ WarpRun warp_run(const Piece* pc, uint64_t npc, int wpb) {
  const uint64_t w = blockIdx.x * (uint64_t)wpb + (threadIdx.x >> 5);
  const uint64_t nw = (uint64_t)gridDim.x * wpb;
  const uint64_t m = pc[npc - 1].e0 + pc[npc - 1].ne;
  return WarpRun{first_piece_at(pc, npc, m * w / nw), first_piece_at(pc, npc, m * (w + 1) / nw)};
}

// register pipeline: batches of G edges, next batch issued before this is added
template <int G>
__global__ void __launch_bounds__(128, 8) k_regpp(const Piece* pc, uint64_t npc, const uint32_t* nbr,
                                                  const double* y, double* out) {
  const int lane = threadIdx.x & 31;
  const WarpRun wr = warp_run(pc, npc, 4);
  if (wr.p0 >= wr.p1) return;
  const uint64_t E0 = pc[wr.p0].e0, E1 = pc[wr.p1 - 1].e0 + pc[wr.p1 - 1].ne;
  uint64_t cur_p = wr.p0;
  uint64_t cur_end = pc[cur_p].e0 + pc[cur_p].ne;
  double ax = 0, ay = 0;
  double2 v[2][G];
  uint32_t ids = 0;
  uint64_t idbase = E0;
  auto load_batch = [&](uint64_t e, double2* dst) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint64_t ee = e + g < E1 ? e + g : E1 - 1;
      const uint32_t id = __ldg(nbr + ee);  // broadcast load (same address in the warp)
      dst[g] = ldg2(y + (uint64_t)id * K + 2 * lane);
    }
  };
  (void)ids;
  (void)idbase;
  load_batch(E0, v[0]);
  int buf = 0;
  for (uint64_t e = E0; e < E1; e += G) {
    if (e + G < E1) load_batch(e + G, v[buf ^ 1]);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint64_t ee = e + g;
      if (ee >= E1) break;
      ax += v[buf][g].x;
      ay += v[buf][g].y;
      if (ee + 1 == cur_end) {
        reinterpret_cast<double2*>(out + cur_p * K)[lane] = make_double2(ax, ay);
        ax = ay = 0;
        ++cur_p;
        if (cur_p < wr.p1) cur_end = pc[cur_p].e0 + pc[cur_p].ne;
      }
    }
    buf ^= 1;
  }
}

// cp.async (LDGSTS) ring of D rows per warp
template <int D, int WPB>
__global__ void __launch_bounds__(WPB * 32) k_lgs(const Piece* pc, uint64_t npc, const uint32_t* nbr,
                                                 const double* y, double* out) {
  extern __shared__ __align__(16) double ring_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* ring = ring_all + (size_t)warp * D * K;
  const WarpRun wr = warp_run(pc, npc, WPB);
  if (wr.p0 >= wr.p1) return;
  const uint64_t E0 = pc[wr.p0].e0, E1 = pc[wr.p1 - 1].e0 + pc[wr.p1 - 1].ne;
  uint64_t cur_p = wr.p0;
  uint64_t cur_end = pc[cur_p].e0 + pc[cur_p].ne;
  uint32_t myid = 0;
  uint64_t idb = ~0ull;
  auto issue = [&](uint64_t e) {
    if (e < E1) {
      const uint64_t b = e & ~31ull;
      if (b != idb) {
        idb = b;
        myid = b + lane < E1 ? __ldg(nbr + b + lane) : 0u;
      }
      const uint32_t id = __shfl_sync(0xffffffffu, myid, (int)(e - b));
      const double* src = y + (uint64_t)id * K + 2 * lane;
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring + (e % D) * K + 2 * lane);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int i = 0; i < D - 1; ++i) issue(E0 + i);
  double ax = 0, ay = 0;
  for (uint64_t e = E0; e < E1; ++e) {
    issue(e + D - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
    const double2 v = reinterpret_cast<const double2*>(ring + (e % D) * K)[lane];
    ax += v.x;
    ay += v.y;
    if (e + 1 == cur_end) {
      reinterpret_cast<double2*>(out + cur_p * K)[lane] = make_double2(ax, ay);
      ax = ay = 0;
      ++cur_p;
      if (cur_p < wr.p1) cur_end = pc[cur_p].e0 + pc[cur_p].ne;
    }
  }
}

template <int D, int WPB>
__global__ void __launch_bounds__(WPB * 32) k_bulk(const Piece* pc, uint64_t npc, const uint32_t* nbr,
                                                  const double* y, double* out) {
  extern __shared__ __align__(128) double ring_bulk[];
  __shared__ __align__(8) uint64_t bars_all[WPB * D];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* ring = ring_bulk + (size_t)warp * D * K;
  uint64_t* bars = bars_all + warp * D;
  if (lane < D)
    for (int i = lane; i < D; i += 32) mbar_init(bars + i, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const WarpRun wr = warp_run(pc, npc, WPB);
  if (wr.p0 >= wr.p1) return;
  const uint64_t E0 = pc[wr.p0].e0, E1 = pc[wr.p1 - 1].e0 + pc[wr.p1 - 1].ne;
  uint64_t cur_p = wr.p0;
  uint64_t cur_end = pc[cur_p].e0 + pc[cur_p].ne;
  // issue in batches of 32 edges: lane j issues edge b + j into slot (b + j) % D
  // (D a multiple of 32 here would let whole batches be in flight; with D < 32
  // a batch is split: lanes whose slot is still being consumed wait)
  uint32_t myid = 0;
  uint64_t idb = ~0ull;
  auto issue = [&](uint64_t e) {  // called by every lane with the same e; lane (e%32) acts
    if (e >= E1) return;
    const uint64_t b = e & ~31ull;
    if (b != idb) {
      idb = b;
      myid = b + lane < E1 ? __ldg(nbr + b + lane) : 0u;
    }
    if ((int)(e & 31) == lane) {
      const uint64_t i = e - E0;
      uint64_t* m = bars + (i % D);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(m, K * 8);
      bulk_g2s(ring + (i % D) * K, y + (uint64_t)myid * K, K * 8, m);
    }
  };
  for (int i = 0; i < D - 1; ++i) issue(E0 + i);
  double ax = 0, ay = 0;
  for (uint64_t e = E0; e < E1; ++e) {
    issue(e + D - 1);
    const uint64_t i = e - E0;
    mbar_wait(bars + (i % D), (unsigned)((i / D) & 1));
    const double2 v = reinterpret_cast<const double2*>(ring + (i % D) * K)[lane];
    __syncwarp();  // the slot is reused by issue(e + D) next iteration
    ax += v.x;
    ay += v.y;
    if (e + 1 == cur_end) {
      reinterpret_cast<double2*>(out + cur_p * K)[lane] = make_double2(ax, ay);
      ax = ay = 0;
      ++cur_p;
      if (cur_p < wr.p1) cur_end = pc[cur_p].e0 + pc[cur_p].ne;
    }
  }
}

template <typename F>
float timeit(F f, int reps) {
  f();
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.0f / reps;
}

int main(int argc, char** argv) {
  const char* path = argc > 1 ? argv[1] : "/tmp/transpose.bin";
  const uint32_t PL = argc > 2 ? atoi(argv[2]) : 128;
  FILE* f = fopen(path, "rb");
  if (!f) {
    perror(path);
    return 1;
  }
  uint64_t n, m;
  if (fread(&n, 8, 1, f) != 1 || fread(&m, 8, 1, f) != 1) return 1;
  std::vector<uint64_t> off(n + 1);
  std::vector<uint32_t> nbr(m);
  if (fread(off.data(), 8, n + 1, f) != n + 1 || fread(nbr.data(), 4, m, f) != m) return 1;
  fclose(f);
  std::vector<Piece> pcs;
  for (uint64_t u = 0; u < n; ++u)
    for (uint64_t b = off[u]; b < off[u + 1]; b += PL)
      pcs.push_back(Piece{b, (uint32_t)(off[u + 1] - b < PL ? off[u + 1] - b : PL), (uint32_t)u});
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  printf("{\"n\":%lu,\"m\":%lu,\"pieces\":%zu,\"PL\":%u,\"sms\":%d}\n", n, m, pcs.size(), PL, sms);
  Piece* dpc;
  uint32_t* dnbr;
  double *y, *out;
  CK(cudaMalloc(&dpc, pcs.size() * sizeof(Piece)));
  CK(cudaMalloc(&dnbr, 4 * m));
  CK(cudaMalloc(&y, 8 * n * K));
  CK(cudaMalloc(&out, 8 * pcs.size() * K));
  CK(cudaMemcpy(dpc, pcs.data(), pcs.size() * sizeof(Piece), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dnbr, nbr.data(), 4 * m, cudaMemcpyHostToDevice));
  CK(cudaMemset(y, 0, 8 * n * K));
  const uint64_t npc = pcs.size();
  const double gb = (double)m * 512 / 1e9;
  auto rep = [&](const char* name, float us) {
    printf("%-28s %9.1f us/sweep  %7.2f TB/s (gathered rows)\n", name, us, gb / us * 1e3);
    fflush(stdout);
  };
  rep("reg G=8 (1184x128)", timeit([&] { k_reg<8><<<sms * 8, 128>>>(dpc, npc, dnbr, y, out); }, 5));
  rep("reg G=8 (4736x128)", timeit([&] { k_reg<8><<<sms * 32, 128>>>(dpc, npc, dnbr, y, out); }, 5));
  {  // row-end bits for the stream kernels
    std::vector<uint32_t> marked(nbr);
    for (const Piece& p : pcs) marked[p.e0 + p.ne - 1] |= 0x80000000u;
    uint32_t* dmk;
    CK(cudaMalloc(&dmk, 4 * m));
    CK(cudaMemcpy(dmk, marked.data(), 4 * m, cudaMemcpyHostToDevice));
    for (int bps : {4, 8}) {
      char name[64];
      snprintf(name, sizeof name, "stream G=8 bps=%d", bps);
      rep(name, timeit([&] { k_stream<8, 0><<<sms * bps, 128>>>(dpc, npc, dmk, y, out); }, 5));
      snprintf(name, sizeof name, "stream G=4 pipe bps=%d", bps);
      rep(name, timeit([&] { k_stream<4, 1><<<sms * bps, 128>>>(dpc, npc, dmk, y, out); }, 5));
      snprintf(name, sizeof name, "stream G=8 pipe bps=%d", bps);
      rep(name, timeit([&] { k_stream<8, 1><<<sms * bps, 128>>>(dpc, npc, dmk, y, out); }, 5));
    }
    for (int bps : {8}) {
      char name[64];
      snprintf(name, sizeof name, "stream_pf G=8 PF=0");
      rep(name, timeit([&] { k_stream_pf<8, 0><<<sms * bps, 128>>>(dpc, npc, dmk, y, out); }, 5));
      snprintf(name, sizeof name, "stream_pf G=8 PF=1");
      rep(name, timeit([&] { k_stream_pf<8, 1><<<sms * bps, 128>>>(dpc, npc, dmk, y, out); }, 5));
      snprintf(name, sizeof name, "stream_pf G=8 PF=2");
      rep(name, timeit([&] { k_stream_pf<8, 2><<<sms * bps, 128>>>(dpc, npc, dmk, y, out); }, 5));
      snprintf(name, sizeof name, "stream_pf G=4 PF=1");
      rep(name, timeit([&] { k_stream_pf<4, 1><<<sms * bps, 128>>>(dpc, npc, dmk, y, out); }, 5));
    }
    CUtensorMap tmap;
    {
      cuuint64_t gdim[2] = {(cuuint64_t)K, (cuuint64_t)n};
      cuuint64_t gstride[1] = {(cuuint64_t)K * 8};
      cuuint32_t box[2] = {(cuuint32_t)K, 1};
      cuuint32_t estr[2] = {1, 1};
      CUresult r = cuTensorMapEncodeTiled(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)y, gdim,
                                          gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      printf("tensor map: %d\n", (int)r);
    }
#define TMA(R, WPB, BPS)                                                                           \
  {                                                                                                \
    const size_t sm = (size_t)R * 32 * K * 8 * WPB;                                                \
    CK(cudaFuncSetAttribute(k_tma<R, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));  \
    rep("tma R=" #R " wpb=" #WPB " bps=" #BPS,                                                      \
        timeit([&] { k_tma<R, WPB><<<sms * BPS, WPB * 32, sm>>>(tmap, dpc, npc, dmk, out); }, 5));  \
    CK(cudaGetLastError());                                                                        \
  }
    TMA(2, 2, 3)
    TMA(2, 4, 1)
    TMA(3, 1, 4)
    TMA(4, 1, 3)
    TMA(2, 1, 6)
    TMA(3, 2, 2)
#define LGS(D, WPB, BPS)                                                                           \
  {                                                                                                \
    const size_t sm = (size_t)D * K * 8 * WPB;                                                     \
    CK(cudaFuncSetAttribute(k_lgs<D, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));  \
    rep("lgs D=" #D " wpb=" #WPB " bps=" #BPS,                                                      \
        timeit([&] { k_lgs<D, WPB><<<sms * BPS, WPB * 32, sm>>>(dpc, npc, dnbr, y, out); }, 5));    \
    CK(cudaGetLastError());                                                                        \
  }
#define BULK(D, WPB, BPS)                                                                          \
  {                                                                                                \
    const size_t sm = (size_t)D * K * 8 * WPB;                                                     \
    CK(cudaFuncSetAttribute(k_bulk<D, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    rep("bulk D=" #D " wpb=" #WPB " bps=" #BPS,                                                     \
        timeit([&] { k_bulk<D, WPB><<<sms * BPS, WPB * 32, sm>>>(dpc, npc, dnbr, y, out); }, 5));   \
    CK(cudaGetLastError());                                                                        \
  }
    LGS(8, 4, 8)
    LGS(16, 4, 6)
    LGS(16, 8, 3)
    LGS(24, 4, 4)
    LGS(32, 4, 3)
    LGS(32, 2, 6)
    BULK(8, 4, 8)
    BULK(16, 4, 6)
    BULK(16, 8, 3)
    BULK(32, 4, 3)
    BULK(32, 2, 6)
    rep("regpp G=4", timeit([&] { k_regpp<4><<<sms * 8, 128>>>(dpc, npc, dnbr, y, out); }, 5));
    rep("regpp G=8", timeit([&] { k_regpp<8><<<sms * 8, 128>>>(dpc, npc, dnbr, y, out); }, 5));
    // correctness: stream and reg must give the same sums
    std::vector<double> a(npc * K), b(npc * K);
    CK(cudaMemset(y, 0, 8 * n * K));
    std::vector<double> hy(n * K);
    for (uint64_t i = 0; i < n * K; ++i) hy[i] = (double)((i * 2654435761u) % 1000) / 1000.0;
    CK(cudaMemcpy(y, hy.data(), 8 * n * K, cudaMemcpyHostToDevice));
    k_reg<8><<<sms * 8, 128>>>(dpc, npc, dnbr, y, out);
    CK(cudaMemcpy(a.data(), out, 8 * npc * K, cudaMemcpyDeviceToHost));
    k_stream<4, 1><<<sms * 8, 128>>>(dpc, npc, dmk, y, out);
    CK(cudaMemcpy(b.data(), out, 8 * npc * K, cudaMemcpyDeviceToHost));
    double md = 0;
    for (uint64_t i = 0; i < npc * K; ++i) md = std::max(md, std::abs(a[i] - b[i]));
    printf("stream vs reg max |diff| = %g\n", md);
    k_stream<8, 0><<<sms * 8, 128>>>(dpc, npc, dmk, y, out);
    CK(cudaMemcpy(b.data(), out, 8 * npc * K, cudaMemcpyDeviceToHost));
    md = 0;
    for (uint64_t i = 0; i < npc * K; ++i) md = std::max(md, std::abs(a[i] - b[i]));
    printf("stream8 vs reg max |diff| = %g\n", md);
    k_stream_pf<8, 2><<<sms * 8, 128>>>(dpc, npc, dmk, y, out);
    CK(cudaMemcpy(b.data(), out, 8 * npc * K, cudaMemcpyDeviceToHost));
    md = 0;
    for (uint64_t i = 0; i < npc * K; ++i) md = std::max(md, std::abs(a[i] - b[i]));
    printf("stream_pf vs reg max |diff| = %g\n", md);
    {
      const size_t sm = (size_t)2 * 32 * K * 8 * 2;
      k_tma<2, 2><<<sms * 3, 64, sm>>>(tmap, dpc, npc, dmk, out);
      CK(cudaGetLastError());
      CK(cudaMemcpy(b.data(), out, 8 * npc * K, cudaMemcpyDeviceToHost));
      md = 0;
      for (uint64_t i = 0; i < npc * K; ++i) md = std::max(md, std::abs(a[i] - b[i]));
      printf("tma vs reg max |diff| = %g\n", md);
    }
    {
      const size_t sm = (size_t)16 * K * 8 * 4;
      k_lgs<16, 4><<<sms * 6, 128, sm>>>(dpc, npc, dnbr, y, out);
      CK(cudaGetLastError());
      CK(cudaMemcpy(b.data(), out, 8 * npc * K, cudaMemcpyDeviceToHost));
      md = 0;
      for (uint64_t i = 0; i < npc * K; ++i) md = std::max(md, std::abs(a[i] - b[i]));
      printf("lgs vs reg max |diff| = %g\n", md);
      k_bulk<16, 4><<<sms * 6, 128, sm>>>(dpc, npc, dnbr, y, out);
      CK(cudaGetLastError());
      CK(cudaMemcpy(b.data(), out, 8 * npc * K, cudaMemcpyDeviceToHost));
      md = 0;
      for (uint64_t i = 0; i < npc * K; ++i) md = std::max(md, std::abs(a[i] - b[i]));
      printf("bulk vs reg max |diff| = %g\n", md);
    }
    CK(cudaMemset(y, 0, 8 * n * K));
  }
  return 0;
  // hot sources: the top H by out-degree (occurrences in the in-edge ids)
  std::vector<uint32_t> outdeg(n, 0);
  for (uint32_t v : nbr) ++outdeg[v];
  std::vector<uint32_t> sorted(outdeg);
  std::sort(sorted.begin(), sorted.end(), std::greater<uint32_t>());
  uint32_t* dnbr_h;
  CK(cudaMalloc(&dnbr_h, 4 * m));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  printf("{\"persistingL2CacheMaxSize\":%d,\"l2\":%d}\n", prop.persistingL2CacheMaxSize, prop.l2CacheSize);
  for (uint64_t H : {100000ull, 150000ull, 200000ull, 300000ull}) {
    const uint32_t thr = sorted[H - 1];
    std::vector<uint32_t> tagged(nbr);
    uint64_t hot_edges = 0;
    for (auto& v : tagged)
      if (outdeg[v] >= thr) {
        v |= 0x80000000u;
        ++hot_edges;
      }
    CK(cudaMemcpy(dnbr_h, tagged.data(), 4 * m, cudaMemcpyHostToDevice));
    char name[96];
    for (int persist : {0, 1}) {
      CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize,
                            persist ? (size_t)prop.persistingL2CacheMaxSize : 0));
      snprintf(name, sizeof name, "H=%lu(%.0f%%e) p=%d last/first", H, 100.0 * hot_edges / m, persist);
      rep(name, timeit([&] { k_reg_hint<8, 1><<<sms * 32, 128>>>(dpc, npc, dnbr_h, y, out); }, 5));
      snprintf(name, sizeof name, "H=%lu p=%d last/normal", H, persist);
      rep(name, timeit([&] { k_reg_hint<8, 2><<<sms * 32, 128>>>(dpc, npc, dnbr_h, y, out); }, 5));
      snprintf(name, sizeof name, "H=%lu p=%d normal/first", H, persist);
      rep(name, timeit([&] { k_reg_hint<8, 3><<<sms * 32, 128>>>(dpc, npc, dnbr_h, y, out); }, 5));
    }
  }
  CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0));
  return 0;
}
