// Design probe (not product code): on a directed R-MAT graph, how fast is one
// Jacobi r.P sweep done as (a) push with fp64 RED atomics over the out-CSR vs
// (b) pull with fp64 gathers over the in-CSR, at k = 1 and k = 4 columns.
// Also raw random RED / gather rates into an L2-resident vector and the plain
// CSR streaming rate. Output: one line per variant with us/sweep and rates.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sg scatter_vs_gather.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <thrust/device_vector.h>
#include <thrust/sort.h>
#include <thrust/unique.h>
#include <thrust/remove.h>
#include <thrust/scan.h>
#include <thrust/sequence.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void rmat_kernel(uint64_t seed, int S, uint64_t count, uint64_t* keys) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  uint32_t u = 0, v = 0;
  for (int l = 0; l < S; ++l) {
    double p = (splitmix(seed * 0x100000001b3ull + i * 64 + l) >> 11) * 0x1.0p-53;
    uint32_t bu = 0, bv = 0;
    if (p < 0.57) {} else if (p < 0.76) { bv = 1; } else if (p < 0.95) { bu = 1; } else { bu = 1; bv = 1; }
    u = (u << 1) | bu; v = (v << 1) | bv;
  }
  keys[i] = ((uint64_t)u << 32) | v;
}

struct IsLoop { __device__ bool operator()(uint64_t k) const { return (k >> 32) == (k & 0xffffffffu); } };

__global__ void count_rows(const uint64_t* keys, uint64_t m, uint64_t* deg) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < m) atomicAdd((unsigned long long*)&deg[keys[i] >> 32], 1ull);
}
__global__ void low_ids(const uint64_t* keys, uint64_t m, uint32_t* nb) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < m) nb[i] = (uint32_t)keys[i];
}
__global__ void swap_key(uint64_t* keys, uint64_t m) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < m) { uint64_t k = keys[i]; keys[i] = (k << 32) | (k >> 32); }
}

// ---- sweeps -----------------------------------------------------------------
__global__ void push_warp(const uint64_t* __restrict__ off, const uint32_t* __restrict__ nb,
                          const double* __restrict__ cur, double* next, uint32_t n, uint32_t s) {
  const int lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
    const double r = cur[v];
    if (r == 0.0) continue;
    const uint64_t b = off[v], e = off[v + 1];
    if (b == e) { if (lane == 0) atomicAdd(next + s, 0.8 * r); continue; }
    const double share = 0.8 * r / (double)(e - b);
    for (uint64_t j = b + lane; j < e; j += 32) atomicAdd(next + nb[j], share);
  }
}
__global__ void push_thread(const uint64_t* __restrict__ off, const uint32_t* __restrict__ nb,
                            const double* __restrict__ cur, double* next, uint32_t n, uint32_t s) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const double r = cur[v];
    if (r == 0.0) continue;
    const uint64_t b = off[v], e = off[v + 1];
    if (b == e) { atomicAdd(next + s, 0.8 * r); continue; }
    const double share = 0.8 * r / (double)(e - b);
    for (uint64_t j = b; j < e; ++j) atomicAdd(next + nb[j], share);
  }
}
__global__ void make_y(const uint64_t* __restrict__ off, const double* __restrict__ cur, double* y, uint32_t n) {
  uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) { uint64_t d = off[v + 1] - off[v]; y[v] = 0.8 * cur[v] / (double)(d ? d : 1); }
}
__global__ void pull_warp(const uint64_t* __restrict__ ioff, const uint32_t* __restrict__ inb,
                          const double* __restrict__ y, double* next, uint32_t n) {
  const int lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
    const uint64_t b = ioff[u], e = ioff[u + 1];
    double acc = 0.0;
    for (uint64_t j = b + lane; j < e; j += 32) acc += y[inb[j]];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) next[u] = acc;
  }
}
__global__ void pull_thread(const uint64_t* __restrict__ ioff, const uint32_t* __restrict__ inb,
                            const double* __restrict__ y, double* next, uint32_t n) {
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
    const uint64_t b = ioff[u], e = ioff[u + 1];
    double acc = 0.0;
    for (uint64_t j = b; j < e; ++j) acc += y[inb[j]];
    next[u] = acc;
  }
}
// k = 4 interleaved columns: 8 edges per warp step, 4 lanes per edge
__global__ void push_warp_k4(const uint64_t* __restrict__ off, const uint32_t* __restrict__ nb,
                             const double* __restrict__ cur, double* next, uint32_t n, uint32_t s) {
  const int lane = threadIdx.x & 31, c = lane & 3, sub = lane >> 2;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
    const double r = cur[4 * (uint64_t)v + c];
    const uint64_t b = off[v], e = off[v + 1];
    if (b == e) { if (sub == 0) atomicAdd(next + 4 * (uint64_t)s + c, 0.8 * r); continue; }
    const double share = 0.8 * r / (double)(e - b);
    for (uint64_t j = b + sub; j < e; j += 8) atomicAdd(next + 4 * (uint64_t)nb[j] + c, share);
  }
}
__global__ void make_y4(const uint64_t* __restrict__ off, const double* __restrict__ cur, double* y, uint32_t n) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < 4ull * n) { uint32_t v = i >> 2; uint64_t d = off[v + 1] - off[v]; y[i] = 0.8 * cur[i] / (double)(d ? d : 1); }
}
__global__ void pull_warp_k4(const uint64_t* __restrict__ ioff, const uint32_t* __restrict__ inb,
                             const double* __restrict__ y, double* next, uint32_t n) {
  const int lane = threadIdx.x & 31, c = lane & 3, sub = lane >> 2;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
    const uint64_t b = ioff[u], e = ioff[u + 1];
    double acc = 0.0;
    for (uint64_t j = b + sub; j < e; j += 8) acc += y[4 * (uint64_t)inb[j] + c];
    acc += __shfl_xor_sync(0xffffffffu, acc, 16);
    acc += __shfl_xor_sync(0xffffffffu, acc, 8);
    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
    if (sub == 0) next[4 * (uint64_t)u + c] = acc;
  }
}

// ---- K = 64 interleaved columns: the bench's block shape --------------------
// One warp per destination row, lanes = 32 x 16 B of one in-edge's 512-byte y
// row; in-edge ids loaded 32 at a time (coalesced) and broadcast by shuffle,
// G row gathers issued before any add. Writes the 64 sums (x row). `mask`
// folds source ids into a small table (L2-resident variant) when nonzero.
template <int G>
__global__ void __launch_bounds__(128, 8) pull_k64(const uint64_t* __restrict__ ioff, const uint32_t* __restrict__ inb,
                         const double* __restrict__ y, double* next, uint32_t n, uint32_t mask) {
  const int lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  const double* yb = y + 2 * lane;
  for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < n; u += warps) {
    const uint64_t b = ioff[u], e = ioff[u + 1];
    double a0 = 0.0, a1 = 0.0;
    for (uint64_t p0 = b; p0 < e; p0 += 32) {
      uint32_t myid = p0 + lane < e ? inb[p0 + lane] : 0u;
      if (mask) myid &= mask;
      const int cnt = e - p0 < 32 ? (int)(e - p0) : 32;
      for (int j0 = 0; j0 < cnt; j0 += G) {
        double2 v[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int j = j0 + g;
          const uint32_t id = __shfl_sync(0xffffffffu, myid, j < cnt ? j : cnt - 1);
          v[g] = *reinterpret_cast<const double2*>(yb + (uint64_t)id * 64);
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const bool ok = j0 + g < cnt;
          a0 += ok ? v[g].x : 0.0;
          a1 += ok ? v[g].y : 0.0;
        }
      }
    }
    *reinterpret_cast<double2*>(next + (uint64_t)u * 64 + 2 * lane) = make_double2(a0, a1);
  }
}
// Same, rows taken from a global atomic counter in chunks of 32 (dynamic balance).
template <int G>
__global__ void __launch_bounds__(128, 8) pull_k64_dyn(const uint64_t* __restrict__ ioff, const uint32_t* __restrict__ inb,
                         const double* __restrict__ y, double* next, uint32_t n, unsigned* ctr) {
  const int lane = threadIdx.x & 31;
  const double* yb = y + 2 * lane;
  for (;;) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(ctr, 8u);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= n) break;
    for (uint32_t u = base; u < base + 8 && u < n; ++u) {
      const uint64_t b = ioff[u], e = ioff[u + 1];
      double a0 = 0.0, a1 = 0.0;
      for (uint64_t p0 = b; p0 < e; p0 += 32) {
        const uint32_t myid = p0 + lane < e ? inb[p0 + lane] : 0u;
        const int cnt = e - p0 < 32 ? (int)(e - p0) : 32;
        for (int j0 = 0; j0 < cnt; j0 += G) {
          double2 v[G];
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const int j = j0 + g;
            const uint32_t id = __shfl_sync(0xffffffffu, myid, j < cnt ? j : cnt - 1);
            v[g] = *reinterpret_cast<const double2*>(yb + (uint64_t)id * 64);
          }
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const bool ok = j0 + g < cnt;
            a0 += ok ? v[g].x : 0.0;
            a1 += ok ? v[g].y : 0.0;
          }
        }
      }
      *reinterpret_cast<double2*>(next + (uint64_t)u * 64 + 2 * lane) = make_double2(a0, a1);
    }
  }
}

// Edge-balanced variant: rows longer than PL in-edges are cut into pieces of PL
// edges (host-built list), pieces of split rows add their partial sums with
// fp64 RED; warps take pieces in grid-stride order.
struct Piece { uint32_t row; uint32_t len; uint64_t b; uint32_t split; uint32_t pad; };
template <int G>
__global__ void __launch_bounds__(128, 8) pull_k64_pieces(const Piece* __restrict__ pc, uint64_t npc,
                         const uint32_t* __restrict__ inb, const double* __restrict__ y, double* next, uint32_t mask,
                         double* ystate = nullptr) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (gridDim.x * blockDim.x) >> 5;
  const double* yb = y + 2 * lane;
  for (uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; w < npc; w += warps) {
    const Piece P = pc[w];
    const uint64_t b = P.b, e = P.b + P.len;
    double a0 = 0.0, a1 = 0.0;
    for (uint64_t p0 = b; p0 < e; p0 += 32) {
      uint32_t myid = p0 + lane < e ? inb[p0 + lane] : 0u;
      if (mask) myid &= mask;
      const int cnt = e - p0 < 32 ? (int)(e - p0) : 32;
      for (int j0 = 0; j0 < cnt; j0 += G) {
        double2 v[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int j = j0 + g;
          const uint32_t id = __shfl_sync(0xffffffffu, myid, j < cnt ? j : cnt - 1);
          v[g] = *reinterpret_cast<const double2*>(yb + (uint64_t)id * 64);
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const bool ok = j0 + g < cnt;
          a0 += ok ? v[g].x : 0.0;
          a1 += ok ? v[g].y : 0.0;
        }
      }
    }
    double* dst = next + (uint64_t)P.row * 64 + 2 * lane;
    if (P.split) { atomicAdd(dst, a0); atomicAdd(dst + 1, a1); }
    else if (ystate) {  // PowerPush state traffic: read x row, push -> write x and y rows
      const double2 xo = __ldcg(reinterpret_cast<const double2*>(dst));
      if (a0 + 1.0 != xo.x || a1 + 1.0 != xo.y) {  // always: an upper bound (80% push in practice)
        *reinterpret_cast<double2*>(dst) = make_double2(a0, a1);
        *reinterpret_cast<double2*>(ystate + (uint64_t)P.row * 64 + 2 * lane) = make_double2(0.8 * a0, 0.8 * a1);
      }
    } else *reinterpret_cast<double2*>(dst) = make_double2(a0, a1);
  }
}

// 128-column rows (1 KB): lanes load 32 B each (two 16-byte loads)
template <int G>
__global__ void __launch_bounds__(128, 8) pull_k128_pieces(const Piece* __restrict__ pc, uint64_t npc,
                         const uint32_t* __restrict__ inb, const double* __restrict__ y, double* next) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (gridDim.x * blockDim.x) >> 5;
  const double* yb = y + 4 * lane;
  for (uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; w < npc; w += warps) {
    const Piece P = pc[w];
    const uint64_t b = P.b, e = P.b + P.len;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (uint64_t p0 = b; p0 < e; p0 += 32) {
      const uint32_t myid = p0 + lane < e ? inb[p0 + lane] : 0u;
      const int cnt = e - p0 < 32 ? (int)(e - p0) : 32;
      for (int j0 = 0; j0 < cnt; j0 += G) {
        double2 v[G][2];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int j = j0 + g;
          const uint32_t id = __shfl_sync(0xffffffffu, myid, j < cnt ? j : cnt - 1);
          const double2* src = reinterpret_cast<const double2*>(yb + (uint64_t)id * 128);
          v[g][0] = src[0];
          v[g][1] = src[1];
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const bool ok = j0 + g < cnt;
          a0 += ok ? v[g][0].x : 0.0; a1 += ok ? v[g][0].y : 0.0;
          a2 += ok ? v[g][1].x : 0.0; a3 += ok ? v[g][1].y : 0.0;
        }
      }
    }
    double* dst = next + (uint64_t)P.row * 128 + 4 * lane;
    if (P.split) { atomicAdd(dst, a0); atomicAdd(dst + 1, a1); atomicAdd(dst + 2, a2); atomicAdd(dst + 3, a3); }
    else { reinterpret_cast<double2*>(dst)[0] = make_double2(a0, a1); reinterpret_cast<double2*>(dst)[1] = make_double2(a2, a3); }
  }
}
// raw rates
__global__ void rand_red(const uint32_t* __restrict__ idx, uint64_t cnt, double* vec) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(vec + idx[i], 1e-9);
}
__global__ void rand_gather(const uint32_t* __restrict__ idx, uint64_t cnt, const double* __restrict__ vec, double* out) {
  double acc = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * blockDim.x)
    acc += vec[idx[i]];
  if (acc == 123.456) out[0] = acc;
}
__global__ void stream_read(const uint4* __restrict__ p, uint64_t cnt, uint32_t* out) {
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 x = p[i]; acc ^= x.x ^ x.y ^ x.z ^ x.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}
__global__ void hash_idx(uint32_t* idx, uint64_t cnt, uint32_t n, uint64_t seed) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < cnt) idx[i] = (uint32_t)(splitmix(seed + i) % n);
}

template <typename F>
float timeit(F f, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b); CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  CK(cudaGetLastError());
  return ms * 1000.f / reps;
}

int main(int argc, char** argv) {
  const int S = argc > 1 ? atoi(argv[1]) : 22;
  const int ef = argc > 2 ? atoi(argv[2]) : 16;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  const uint32_t n = 1u << S;
  const uint64_t draws = (uint64_t)ef << S;
  thrust::device_vector<uint64_t> keys(draws);
  rmat_kernel<<<(draws + 255) / 256, 256>>>(3, S, draws, thrust::raw_pointer_cast(keys.data()));
  thrust::sort(keys.begin(), keys.end());
  keys.erase(thrust::unique(keys.begin(), keys.end()), keys.end());
  keys.erase(thrust::remove_if(keys.begin(), keys.end(), IsLoop()), keys.end());
  const uint64_t m = keys.size();
  thrust::device_vector<uint64_t> off(n + 1, 0), ioff(n + 1, 0);
  thrust::device_vector<uint32_t> nb(m), inb(m);
  const int TB = 256; const uint64_t gb = (m + TB - 1) / TB;
  count_rows<<<gb, TB>>>(thrust::raw_pointer_cast(keys.data()), m, thrust::raw_pointer_cast(off.data()) + 1);
  thrust::inclusive_scan(off.begin(), off.end(), off.begin());
  low_ids<<<gb, TB>>>(thrust::raw_pointer_cast(keys.data()), m, thrust::raw_pointer_cast(nb.data()));
  swap_key<<<gb, TB>>>(thrust::raw_pointer_cast(keys.data()), m);
  thrust::sort(keys.begin(), keys.end());
  count_rows<<<gb, TB>>>(thrust::raw_pointer_cast(keys.data()), m, thrust::raw_pointer_cast(ioff.data()) + 1);
  thrust::inclusive_scan(ioff.begin(), ioff.end(), ioff.begin());
  low_ids<<<gb, TB>>>(thrust::raw_pointer_cast(keys.data()), m, thrust::raw_pointer_cast(inb.data()));
  CK(cudaDeviceSynchronize());
  keys.clear(); keys.shrink_to_fit();
  printf("{\"S\":%d,\"ef\":%d,\"n\":%u,\"m\":%llu,\"sms\":%d,\"l2\":%d}\n", S, ef, n, (unsigned long long)m, sms, l2);

  const uint64_t* o = thrust::raw_pointer_cast(off.data());
  const uint64_t* io = thrust::raw_pointer_cast(ioff.data());
  const uint32_t* nbp = thrust::raw_pointer_cast(nb.data());
  const uint32_t* inbp = thrust::raw_pointer_cast(inb.data());
  double *cur, *next, *y;
  CK(cudaMalloc(&cur, 8ull * 4 * n)); CK(cudaMalloc(&next, 8ull * 4 * n)); CK(cudaMalloc(&y, 8ull * 4 * n));
  {  // dense-ish residue: every node nonzero (global phase is ~80% active)
    std::vector<double> h(4ull * n, 1.0 / n);
    CK(cudaMemcpy(cur, h.data(), 8ull * 4 * n, cudaMemcpyHostToDevice));
  }
  const int G = sms * 8;  // 8 x 256 threads per SM resident
  float t;
  auto rep = [&](const char* name, float us, double bytes, double ops) {
    printf("%-16s %9.1f us  %7.1f GB/s(alg)  %7.1f Gops/s\n", name, us, bytes / us / 1e3, ops / us / 1e3);
  };

  if (argc > 3 && atoi(argv[3]) == 64) {  // K = 64 ceiling probe
    double *y64, *x64; unsigned* ctr;
    CK(cudaMalloc(&y64, 8ull * 64 * n)); CK(cudaMalloc(&x64, 8ull * 64 * n)); CK(cudaMalloc(&ctr, 4));
    CK(cudaMemset(y64, 0, 8ull * 64 * n));
    const double b64 = 4.0 * m + 512.0 * m + 512.0 * n;  // ids + gathered rows + x rows written
    for (int blocks : {sms * 8, sms * 16, sms * 32}) {
      t = timeit([&] { pull_k64<8><<<blocks, 128>>>(io, inbp, y64, x64, n, 0); }, 5);
      printf("pull_k64_G8 grid=%d", blocks); rep("", t, b64, (double)m);
    }
    t = timeit([&] { pull_k64<4><<<sms * 8, 128>>>(io, inbp, y64, x64, n, 0); }, 5); rep("pull_k64_G4", t, b64, (double)m);
    t = timeit([&] { pull_k64<16><<<sms * 8, 128>>>(io, inbp, y64, x64, n, 0); }, 5); rep("pull_k64_G16", t, b64, (double)m);
    t = timeit([&] { cudaMemsetAsync(ctr, 0, 4); pull_k64_dyn<8><<<sms * 8, 128>>>(io, inbp, y64, x64, n, ctr); }, 5);
    rep("pull_k64_dyn_G8", t, b64, (double)m);
    // source ids folded into 2^17 rows (64 MB of y): the gathers hit L2
    t = timeit([&] { pull_k64<8><<<sms * 8, 128>>>(io, inbp, y64, x64, n, (1u << 17) - 1); }, 5);
    rep("pull_k64_L2res", t, b64, (double)m);
    t = timeit([&] { pull_k64<8><<<sms * 8, 128>>>(io, inbp, y64, x64, n, (1u << 14) - 1); }, 5);
    rep("pull_k64_L2small", t, b64, (double)m);

    for (uint32_t PL : {128u, 512u, 2048u}) {
      std::vector<uint64_t> h(n + 1);
      CK(cudaMemcpy(h.data(), io, 8ull * (n + 1), cudaMemcpyDeviceToHost));
      std::vector<Piece> pcs;
      for (uint32_t u = 0; u < n; ++u) {
        const uint64_t len = h[u + 1] - h[u];
        if (!len) continue;
        const uint32_t split = len > PL;
        for (uint64_t q = 0; q < len; q += PL)
          pcs.push_back(Piece{u, (uint32_t)(len - q < PL ? len - q : PL), h[u] + q, split, 0});
      }
      Piece* dpc; CK(cudaMalloc(&dpc, sizeof(Piece) * pcs.size()));
      CK(cudaMemcpy(dpc, pcs.data(), sizeof(Piece) * pcs.size(), cudaMemcpyHostToDevice));
      for (int blocks : {sms * 8, sms * 32}) {
        t = timeit([&] { pull_k64_pieces<8><<<blocks, 128>>>(dpc, pcs.size(), inbp, y64, x64, 0); }, 5);
        printf("pieces PL=%u grid=%d npc=%zu", PL, blocks, pcs.size()); rep("", t, b64, (double)m);
      }
      {  // + the PowerPush per-row state traffic (x row read, x and y rows written); y2 = y64 copy target
        double* y2; CK(cudaMalloc(&y2, 8ull * 64 * n)); CK(cudaMemset(x64, 0, 8ull * 64 * n));
        t = timeit([&] { pull_k64_pieces<8><<<sms * 32, 128>>>(dpc, pcs.size(), inbp, y64, x64, 0, y2); }, 5);
        printf("pieces PL=%u +state", PL); rep("", t, b64, (double)m);
        cudaFree(y2);
      }
      if (PL == 128) {  // 128 columns: per-query cost vs 64
        double *y128, *x128;
        CK(cudaMalloc(&y128, 8ull * 128 * n)); CK(cudaMalloc(&x128, 8ull * 128 * n));
        CK(cudaMemset(y128, 0, 8ull * 128 * n));
        for (int G2 : {4, 8}) {
          t = G2 == 4 ? timeit([&] { pull_k128_pieces<4><<<sms * 32, 128>>>(dpc, pcs.size(), inbp, y128, x128); }, 5)
                      : timeit([&] { pull_k128_pieces<8><<<sms * 32, 128>>>(dpc, pcs.size(), inbp, y128, x128); }, 5);
          printf("pieces PL=128 K=128 G=%d (per 64 columns: %.1f us)", G2, t / 2); rep("", t, 2 * b64, (double)m);
        }
        cudaFree(y128); cudaFree(x128);
      }
      t = timeit([&] { pull_k64_pieces<8><<<sms * 32, 128>>>(dpc, pcs.size(), inbp, y64, x64, (1u << 17) - 1); }, 5);
      printf("pieces PL=%u L2res", PL); rep("", t, b64, (double)m);
      cudaFree(dpc);
    }
    return 0;
  }
  const double b1 = 8.0 * (n + 1) + 4.0 * m + 32.0 * n;
  t = timeit([&] { cudaMemsetAsync(next, 0, 8ull * n); push_warp<<<G, 256>>>(o, nbp, cur, next, n, 0); }, 10);
  rep("push_warp_k1", t, b1, (double)m);
  t = timeit([&] { cudaMemsetAsync(next, 0, 8ull * n); push_thread<<<G, 256>>>(o, nbp, cur, next, n, 0); }, 10);
  rep("push_thread_k1", t, b1, (double)m);
  t = timeit([&] { make_y<<<(n + 255) / 256, 256>>>(o, cur, y, n); pull_warp<<<G, 256>>>(io, inbp, y, next, n); }, 10);
  rep("pull_warp_k1", t, b1, (double)m);
  t = timeit([&] { make_y<<<(n + 255) / 256, 256>>>(o, cur, y, n); pull_thread<<<G, 256>>>(io, inbp, y, next, n); }, 10);
  rep("pull_thread_k1", t, b1, (double)m);
  const double b4 = 8.0 * (n + 1) + 4.0 * m + 32.0 * 4 * n;
  t = timeit([&] { cudaMemsetAsync(next, 0, 32ull * n); push_warp_k4<<<G, 256>>>(o, nbp, cur, next, n, 0); }, 10);
  rep("push_warp_k4", t, b4, 4.0 * m);
  t = timeit([&] { make_y4<<<(4ull * n + 255) / 256, 256>>>(o, cur, y, n); pull_warp_k4<<<G, 256>>>(io, inbp, y, next, n); }, 10);
  rep("pull_warp_k4", t, b4, 4.0 * m);
  // raw rates over an n-double vector
  uint32_t* idx; CK(cudaMalloc(&idx, 4ull * m));
  hash_idx<<<gb, TB>>>(idx, m, n, 77);
  t = timeit([&] { rand_red<<<G, 256>>>(idx, m, next); }, 10);
  rep("rand_red", t, 4.0 * m, (double)m);
  t = timeit([&] { rand_gather<<<G, 256>>>(idx, m, cur, y); }, 10);
  rep("rand_gather", t, 4.0 * m, (double)m);
  t = timeit([&] { rand_red<<<G, 256>>>(inbp, m, next); }, 10);
  rep("rmat_red(src)", t, 4.0 * m, (double)m);
  t = timeit([&] { rand_red<<<G, 256>>>(nbp, m, next); }, 10);
  rep("rmat_red(dst)", t, 4.0 * m, (double)m);
  t = timeit([&] { rand_gather<<<G, 256>>>(inbp, m, cur, y); }, 10);
  rep("rmat_gather(src)", t, 4.0 * m, (double)m);
  t = timeit([&] { stream_read<<<G, 256>>>((const uint4*)inbp, m / 4, (uint32_t*)y); }, 10);
  rep("stream_nbrs", t, 4.0 * m, (double)m);
  return 0;
}
