// Design probe (not product code): how fast can a pull sweep gather y when a
// query block has K < 64 columns, so that y (n x K f64) is small enough to stay
// in the 126 MB L2? Same input as gather_engines.cu (the configs[2] transpose,
// R-MAT 22/16 seed 3). Every variant sums y over the in-edges of pieces of
// <= PL in-edges and writes one K-column sum per piece (no decisions), so the
// time is the gather alone. Reported per sweep and per 64 columns (64/K
// sweeps), the unit the 64-column engine is measured in.
//   regk<K,G,W>: W bytes per lane (16 or 32), LPR = 8K/W lanes per row,
//                EPI = 32/LPR in-edges per warp load instruction, G loads in
//                flight; at the piece end the EPI lane groups are reduced by
//                xor shuffles.
//   hint=1: in-edge ids streamed with L2::evict_first, y gathers evict_last.
//   win=1 : y under a persisting L2 access-policy window.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nk narrow_k.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) {                                                                    \
      fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);        \
      exit(1);                                                                                  \
    }                                                                                           \
  } while (0)

struct Piece {
  uint64_t e0;
  uint32_t ne, row;
};

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

template <int W, int HINT>
struct Vec;
template <int HINT>
struct Vec<16, HINT> {
  double a[2];
  __device__ __forceinline__ void load(const double* p, uint64_t pol) {
    if (HINT)
      asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                   : "=d"(a[0]), "=d"(a[1]) : "l"(p), "l"(pol));
    else
      asm volatile("ld.global.v2.f64 {%0,%1}, [%2];" : "=d"(a[0]), "=d"(a[1]) : "l"(p));
  }
};
template <int HINT>
struct Vec<32, HINT> {
  double a[4];
  __device__ __forceinline__ void load(const double* p, uint64_t pol) {
    if (HINT)
      asm volatile("ld.global.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
                   : "=d"(a[0]), "=d"(a[1]), "=d"(a[2]), "=d"(a[3]) : "l"(p), "l"(pol));
    else
      asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(a[0]), "=d"(a[1]), "=d"(a[2]), "=d"(a[3]) : "l"(p));
  }
};

template <int HINT>
__device__ __forceinline__ uint32_t ld_id(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  if (HINT)
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  else
    v = __ldg(p);
  return v;
}

template <int K, int G, int W, int HINT>
__global__ void __launch_bounds__(128, 8) k_regk(const Piece* pc, uint64_t npc, const uint32_t* nbr,
                                                 const double* y, double* out) {
  constexpr int NV = W / 8;          // doubles per lane
  constexpr int LPR = K / NV;        // lanes per row
  constexpr int EPI = 32 / LPR;      // in-edges per load instruction
  const int lane = threadIdx.x & 31;
  const int grp = lane / LPR, sub = lane % LPR;
  const uint64_t pf = pol_first(), pl = pol_last();
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t p = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; p < npc; p += nw) {
    const Piece d = pc[p];
    double acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = 0;
    for (uint32_t b = 0; b < d.ne; b += 32) {
      const uint32_t myid = b + lane < d.ne ? ld_id<HINT>(nbr + d.e0 + b + lane, pf) : 0u;
      const int cnt = d.ne - b < 32 ? d.ne - b : 32;
      for (int j0 = 0; j0 < cnt; j0 += EPI * G) {
        Vec<W, HINT> v[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int j = j0 + g * EPI + grp;
          const uint32_t id = __shfl_sync(0xffffffffu, myid, j < cnt ? j : cnt - 1);
          v[g].load(y + (uint64_t)id * K + NV * sub, pl);
        }
#pragma unroll
        for (int g = 0; g < G; ++g)
          if (j0 + g * EPI + grp < cnt) {
#pragma unroll
            for (int i = 0; i < NV; ++i) acc[i] += v[g].a[i];
          }
      }
    }
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
      for (int i = 0; i < NV; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
    if (grp == 0)
#pragma unroll
      for (int i = 0; i < NV; ++i) out[p * K + NV * sub + i] = acc[i];
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
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  printf("{\"n\":%lu,\"m\":%lu,\"sms\":%d,\"l2\":%d,\"persist_max\":%d}\n", n, m, sms, prop.l2CacheSize,
         prop.persistingL2CacheMaxSize);
  uint32_t* dnbr;
  double *y, *out;
  CK(cudaMalloc(&dnbr, 4 * m));
  CK(cudaMalloc(&y, 8 * n * 64));
  CK(cudaMemcpy(dnbr, nbr.data(), 4 * m, cudaMemcpyHostToDevice));
  CK(cudaMemset(y, 0, 8 * n * 64));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  const bool quick = argc > 2;  // ncu: one launch of a few variants
  if (quick) {
    const uint32_t PL = 128;
    std::vector<Piece> pcs;
    for (uint64_t u = 0; u < n; ++u)
      for (uint64_t b = off[u]; b < off[u + 1]; b += PL)
        pcs.push_back(Piece{b, (uint32_t)(off[u + 1] - b < PL ? off[u + 1] - b : PL), (uint32_t)u});
    const uint64_t npc = pcs.size();
    Piece* dpc;
    CK(cudaMalloc(&dpc, npc * sizeof(Piece)));
    CK(cudaMalloc(&out, 8 * npc * 64));
    CK(cudaMemcpy(dpc, pcs.data(), npc * sizeof(Piece), cudaMemcpyHostToDevice));
    k_regk<64, 8, 16, 0><<<sms * 8, 128, 0, st>>>(dpc, npc, dnbr, y, out);
    k_regk<32, 8, 16, 0><<<sms * 8, 128, 0, st>>>(dpc, npc, dnbr, y, out);
    k_regk<16, 8, 32, 0><<<sms * 8, 128, 0, st>>>(dpc, npc, dnbr, y, out);
    k_regk<16, 8, 16, 0><<<sms * 8, 128, 0, st>>>(dpc, npc, dnbr, y, out);
    k_regk<8, 8, 16, 0><<<sms * 8, 128, 0, st>>>(dpc, npc, dnbr, y, out);
    k_regk<4, 4, 16, 0><<<sms * 8, 128, 0, st>>>(dpc, npc, dnbr, y, out);
    CK(cudaDeviceSynchronize());
    return 0;
  }
  for (uint32_t PL : {128u, 512u}) {
    std::vector<Piece> pcs;
    for (uint64_t u = 0; u < n; ++u)
      for (uint64_t b = off[u]; b < off[u + 1]; b += PL)
        pcs.push_back(Piece{b, (uint32_t)(off[u + 1] - b < PL ? off[u + 1] - b : PL), (uint32_t)u});
    const uint64_t npc = pcs.size();
    Piece* dpc;
    CK(cudaMalloc(&dpc, npc * sizeof(Piece)));
    CK(cudaMalloc(&out, 8 * npc * 64));
    CK(cudaMemcpy(dpc, pcs.data(), npc * sizeof(Piece), cudaMemcpyHostToDevice));
    printf("PL=%u pieces=%lu\n", PL, npc);
    auto rep = [&](const char* name, int K, float us) {
      printf("%-34s K=%2d %9.1f us/sweep %9.1f us/64col  %6.2f TB/s gathered\n", name, K, us, us * 64 / K,
             (double)m * 8 * K / us / 1e6);
      fflush(stdout);
    };
    for (int win : {0, 1}) {
#define RUN(K, G, W, H, BPS)                                                                         \
  {                                                                                                  \
    if (win) {                                                                                       \
      cudaStreamAttrValue a = {};                                                                    \
      const size_t bytes = (size_t)8 * n * K;                                                        \
      CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)prop.persistingL2CacheMaxSize)); \
      a.accessPolicyWindow.base_ptr = y;                                                             \
      a.accessPolicyWindow.num_bytes = bytes < (size_t)prop.accessPolicyMaxWindowSize                \
                                           ? bytes : (size_t)prop.accessPolicyMaxWindowSize;         \
      a.accessPolicyWindow.hitRatio =                                                                \
          std::min(1.0f, (float)prop.persistingL2CacheMaxSize / (float)a.accessPolicyWindow.num_bytes); \
      a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;                                   \
      a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;                                   \
      CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a));                     \
    }                                                                                                \
    char name[96];                                                                                   \
    snprintf(name, sizeof name, "G=%d W=%d hint=%d win=%d bps=%d", G, W, H, win, BPS);               \
    rep(name, K, timeit([&] { k_regk<K, G, W, H><<<sms * BPS, 128, 0, st>>>(dpc, npc, dnbr, y, out); }, 5)); \
    CK(cudaGetLastError());                                                                          \
    if (win) {                                                                                       \
      cudaStreamAttrValue a = {};                                                                    \
      a.accessPolicyWindow.num_bytes = 0;                                                            \
      CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &a));                     \
      CK(cudaCtxResetPersistingL2Cache());                                                           \
      CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0));                                     \
    }                                                                                                \
  }
      if (win == 0) {
        RUN(64, 8, 16, 0, 8)
        RUN(64, 4, 32, 0, 8)
        RUN(64, 6, 32, 0, 8)
        RUN(64, 8, 16, 0, 12)
        RUN(64, 4, 32, 0, 12)
        RUN(32, 8, 16, 0, 8)
        RUN(32, 4, 32, 0, 8)
      }
      RUN(16, 8, 16, 0, 8)
      RUN(16, 8, 16, 1, 8)
      RUN(16, 4, 32, 0, 8)
      RUN(16, 8, 32, 0, 8)
      RUN(8, 8, 16, 0, 8)
      RUN(8, 4, 16, 0, 8)
      RUN(8, 8, 16, 1, 8)
      RUN(8, 4, 32, 0, 8)
      RUN(8, 8, 32, 0, 8)
      RUN(8, 8, 32, 1, 8)
      RUN(4, 4, 16, 0, 8)
      RUN(4, 8, 16, 0, 8)
      RUN(4, 8, 16, 1, 8)
      RUN(4, 4, 32, 0, 8)
      RUN(4, 8, 32, 0, 8)
      RUN(4, 8, 32, 1, 8)
      RUN(2, 8, 16, 0, 8)
      RUN(2, 8, 16, 1, 8)
    }
    CK(cudaFree(dpc));
    CK(cudaFree(out));
  }
  return 0;
}
