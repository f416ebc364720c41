// Shared device/host helpers for the PPR engine (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace pprg {

// ---- errors (mapped to PPRG_* codes at the C ABI) --------------------------
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
enum { OK = 0, EINVAL_ = 1, EDATA = 2, EINTERNAL = 3, ECUDA = 4, ENCCL = 5 };

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

#define PPRG_CUDA(call)                                                              \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      ::pprg::fail(::pprg::ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// in destructors: errors are ignored (a failed call already reported its own)
#define PPRG_CUDA_NOTHROW(call) ((void)(call))

// ---- Philox4x32-10 (Salmon et al. SC'11) -----------------------------------
struct U4 {
  uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
#if defined(__CUDA_ARCH__)
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
#else
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
    const uint32_t lo0 = (uint32_t)p0, hi0 = (uint32_t)(p0 >> 32);
    const uint32_t lo1 = (uint32_t)p1, hi1 = (uint32_t)(p1 >> 32);
#endif
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
  }
  return c;
}

__host__ __device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// Walk-step randomness, the product's definition:
// step t of walk (k, v) under tag (source id, or kIndexTag for the index)
// is Philox(key = seed, ctr = (k, v, tag, t)). Word pair (x,y) gives the
// 53-bit stop uniform (rng.hpp:21 semantics), (z,w) the 64-bit neighbour
// draw, bounded by Lemire multiply-high with rejection (rng.hpp:24-35
// semantics); rejected draws re-key word 3 as t + (retry << 24).
constexpr uint32_t kIndexTag = 0xFFFFFFFFu;

__host__ __device__ __forceinline__ uint64_t walk_below(uint64_t first, uint64_t bound, uint32_t k,
                                                        uint32_t v, uint32_t tag, uint32_t t,
                                                        uint32_t k0, uint32_t k1) {
  uint64_t hi = mulhi64(first, bound), low = first * bound;
  if (low < bound) {
    const uint64_t threshold = (0 - bound) % bound;
    uint32_t retry = 1;
    while (low < threshold) {
      const U4 o = philox4x32_10(U4{k, v, tag, t + (retry++ << 24)}, k0, k1);
      const uint64_t r = ((uint64_t)o.w << 32) | o.z;
      hi = mulhi64(r, bound);
      low = r * bound;
    }
  }
  return hi;
}

// Full alpha-random walk from `start` (walk_index.cpp:10-17 semantics).
__host__ __device__ __forceinline__ uint32_t philox_walk(const uint64_t* off, const uint32_t* nbr,
                                                         uint32_t start, uint32_t source,
                                                         double alpha, uint64_t seed, uint32_t k,
                                                         uint32_t v, uint32_t tag) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  uint32_t cur = start;
  for (uint32_t t = 0;; ++t) {
    const U4 o = philox4x32_10(U4{k, v, tag, t}, k0, k1);
    const double u = (double)((((uint64_t)o.y << 32) | o.x) >> 11) * 0x1.0p-53;
    if (!(u >= alpha)) return cur;
    const uint64_t b = off[cur], d = off[cur + 1] - b;
    if (d == 0) {
      cur = source;
    } else {
      cur = nbr[b + walk_below(((uint64_t)o.w << 32) | o.z, d, k, v, tag, t, k0, k1)];
    }
  }
}

// ---- device memory helpers -------------------------------------------------
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) PPRG_CUDA(cudaMalloc(&p, count * sizeof(T)));
  }
  void ensure(size_t count) {
    if (count > n) alloc(count);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
};

#if defined(__CUDACC__)
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

// L2 eviction-priority hints for the sweep streams. Per sweep the in-edge ids,
// row data and the state x are touched once (streams, > L2), while the gathered
// operand y is re-read once per out-edge of its node; marking the streams
// evict-first keeps L2 for y. PPRG_HINTS: 0 = none, 1 = streams evict-first,
// 2 = 1 + y gathers evict-last.
#ifndef PPRG_HINTS
#define PPRG_HINTS 0
#endif
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) {
#if PPRG_HINTS >= 1
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(l2_evict_first()));
  return v;
#else
  return __ldg(p);
#endif
}
__device__ __forceinline__ double ld_state(const double* p) {  // coherent (L2), streamed
#if PPRG_HINTS >= 1
  double v;
  asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(l2_evict_first()));
  return v;
#else
  return __ldcg(p);
#endif
}
__device__ __forceinline__ double2 ld_state2(const double* p) {  // two adjacent columns
  double2 v;
  asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_state(double* p, double v) {
#if PPRG_HINTS >= 1
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" :: "l"(p), "d"(v), "l"(l2_evict_first()) : "memory");
#else
  *p = v;
#endif
}
// four adjacent columns in one 32-byte access (LDG.E.ENL2.256, sm_100)
struct dbl4 {
  double v[4];
};
__device__ __forceinline__ dbl4 ld_state4(const double* p) {
  dbl4 r;
  asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3]) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_state4(double* p, const dbl4& r) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};"
               :: "l"(p), "d"(r.v[0]), "d"(r.v[1]), "d"(r.v[2]), "d"(r.v[3]) : "memory");
}
__device__ __forceinline__ dbl4 ld_gather4(const double* p) {
  dbl4 r;
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3]) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_gather2(const double* p) {
#if PPRG_HINTS == 3
  double2 v;
  asm volatile("ld.global.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
#elif PPRG_HINTS >= 2
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(l2_evict_last()));
  return v;
#else
  return *reinterpret_cast<const double2*>(p);
#endif
}
__device__ __forceinline__ double ld_gather(const double* p) {
#if PPRG_HINTS == 3
  double v;
  asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
#elif PPRG_HINTS >= 2
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(l2_evict_last()));
  return v;
#else
  return *p;
#endif
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Sense-free grid barrier over a monotonically increasing counter; `target`
// = (barrier generation + 1) * gridDim.x. Requires a cooperative launch (all
// blocks co-resident). The gpu-scope fence also invalidates the SM's L1, so
// every sweep starts from values at least as new as the previous sweep's.
// Two-level grid barrier: blocks arrive on one of up to 32 group counters
// (separate 128-byte lines), the last of each group on the top counter, and
// the very last block publishes the generation that everyone polls. The
// serialised atomics per barrier drop from gridDim.x to ~gridDim.x/32 + 32.
struct GridBarrier {
  unsigned long long grp[32][16];
  unsigned long long top[16];
  unsigned long long flag[16];
};

// The barrier's release (before arriving) and acquire (after the flag) fences:
// acq_rel at gpu scope is what the arrival/flag chain needs (PPRG_BAR_SC=1:
// the sequentially consistent __threadfence instead).
#ifndef PPRG_BAR_SC
#define PPRG_BAR_SC 0
#endif
__device__ __forceinline__ void bar_fence() {
#if PPRG_BAR_SC
  __threadfence();
#else
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
}

__device__ __forceinline__ void grid_barrier2(GridBarrier* gb, unsigned long long gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned ng = gridDim.x < 32 ? gridDim.x : 32;
    const unsigned g = blockIdx.x % ng;
    const unsigned long long gsize = gridDim.x / ng + (g < gridDim.x % ng ? 1 : 0);
    bar_fence();
    const unsigned long long old = atomicAdd(&gb->grp[g][0], 1ull);
    if (old + 1 == gsize * gen) {
      bar_fence();
      const unsigned long long o2 = atomicAdd(&gb->top[0], 1ull);
      if (o2 + 1 == (unsigned long long)ng * gen) {
        bar_fence();
        atomicExch(&gb->flag[0], gen);
      }
    }
    while (ld_acquire(&gb->flag[0]) < gen) __nanosleep(20);
    bar_fence();
  }
  __syncthreads();
}

__device__ __forceinline__ void grid_barrier(unsigned long long* counter,
                                             unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(counter, 1ull);
    while (ld_acquire(counter) < target) __nanosleep(20);
    __threadfence();
  }
  __syncthreads();
}
#endif

}  // namespace pprg
