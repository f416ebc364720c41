// Design probe (not product code): one-column (K = 1) pull-sweep gathers over
// a large transpose, with the gathered ids as generated and with the nodes
// relabelled by descending out-degree. A K = 1 gather reads 8 bytes out of a
// 32-byte sector; relabelling packs the hot (high out-degree) nodes' y values
// into shared sectors, so the hot set's L2 footprint shrinks up to 4x.
// Input: tools/microbench/dump_transpose.py <file> <scale> <ef> <seed>.
// Every variant sums y over the in-edges of <= PL-edge pieces (warp per piece,
// each lane 8 gathers in flight) and writes one sum per piece.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o k1r k1_relabel.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numeric>
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

template <int G>
__global__ void __launch_bounds__(128, 8) k_k1(const Piece* pc, uint64_t npc, const uint32_t* nbr,
                                               const double* y, double* out) {
  const int lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t p = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; p < npc; p += nw) {
    const Piece d = pc[p];
    double acc = 0.0;
    for (uint32_t b = 0; b < d.ne; b += 32 * G) {
      uint32_t id[G];
      double v[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const uint32_t e = b + 32 * g + lane;
        id[g] = e < d.ne ? __ldg(nbr + d.e0 + e) : 0xFFFFFFFFu;
      }
#pragma unroll
      for (int g = 0; g < G; ++g) v[g] = id[g] != 0xFFFFFFFFu ? y[id[g]] : 0.0;
#pragma unroll
      for (int g = 0; g < G; ++g) acc += v[g];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[p] = acc;
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
  const char* path = argc > 1 ? argv[1] : "/tmp/transpose25.bin";
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
  const uint32_t PL = 256;
  std::vector<Piece> pcs;
  for (uint64_t u = 0; u < n; ++u)
    for (uint64_t b = off[u]; b < off[u + 1]; b += PL)
      pcs.push_back(Piece{b, (uint32_t)(off[u + 1] - b < PL ? off[u + 1] - b : PL), (uint32_t)u});
  const uint64_t npc = pcs.size();
  // out-degree of v = its occurrences among the in-edge ids
  std::vector<uint32_t> outdeg(n, 0);
  for (uint32_t v : nbr) ++outdeg[v];
  std::vector<uint32_t> order(n);
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return outdeg[a] > outdeg[b]; });
  std::vector<uint32_t> perm(n);
  for (uint64_t i = 0; i < n; ++i) perm[order[i]] = (uint32_t)i;
  std::vector<uint32_t> rel(m);
  for (uint64_t e = 0; e < m; ++e) rel[e] = perm[nbr[e]];
  // coverage of the hottest y sectors
  {
    uint64_t acc = 0, hot = 0;
    const uint64_t l2_vals = 126ull * 1024 * 1024 / 8;  // y values that fit in L2 if packed
    for (uint64_t i = 0; i < n && i < l2_vals; ++i) hot += outdeg[order[i]];
    for (uint64_t i = 0; i < n; ++i) acc += outdeg[i];
    printf("{\"n\":%lu,\"m\":%lu,\"pieces\":%lu,\"edges_to_hottest_126MB_of_y\":%.3f}\n", n, m, npc,
           (double)hot / (double)acc);
  }
  Piece* dpc;
  uint32_t *dnbr, *drel;
  double *y, *out;
  CK(cudaMalloc(&dpc, npc * sizeof(Piece)));
  CK(cudaMalloc(&dnbr, 4 * m));
  CK(cudaMalloc(&drel, 4 * m));
  CK(cudaMalloc(&y, 8 * n));
  CK(cudaMalloc(&out, 8 * npc));
  CK(cudaMemcpy(dpc, pcs.data(), npc * sizeof(Piece), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dnbr, nbr.data(), 4 * m, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(drel, rel.data(), 4 * m, cudaMemcpyHostToDevice));
  CK(cudaMemset(y, 0, 8 * n));
  for (int bps : {8, 16}) {
    const float a = timeit([&] { k_k1<8><<<sms * bps, 128>>>(dpc, npc, dnbr, y, out); }, 5);
    const float b = timeit([&] { k_k1<8><<<sms * bps, 128>>>(dpc, npc, drel, y, out); }, 5);
    printf("bps=%d  natural ids %9.1f us/sweep   degree-relabelled %9.1f us/sweep   (%.2fx)\n", bps, a, b, a / b);
    fflush(stdout);
  }
  return 0;
}
