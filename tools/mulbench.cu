// Microbenchmark: throughput of the bit-sliced multiply (GF::mul_acc_n2,
// warp-uniform factors) against resident warps per SM; W = lane-words per
// thread (W = 2 shares each factor's branches between two words, as
// mul_acc2_n2 does).  Experiments only: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a tools/mulbench.cu -o tools/mulbench
#include <cstdint>
#include <cstdio>
#include "../paper_1404_3458_b200/csrc/lch_device.cuh"
using F = lch::GF<16, 0x1100Bu>;

template <int W>
__global__ void __launch_bounds__(256) k(const uint32_t *fac, uint32_t *out, int iters) {
  uint32_t v[W][16], u[W][16];
  for (int w = 0; w < W; ++w)
    for (int b = 0; b < 16; ++b) { v[w][b] = threadIdx.x * 977u + b * 131u + w; u[w][b] = b; }
  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0);
  for (int it = 0; it < iters; ++it) {
    const uint32_t f = fac[(blockIdx.x * 8 + warp + it * 7) & 4095];
    if (W == 1) {
      F::mul_acc_n2(u[0], v[0], f);
      for (int b = 0; b < 16; ++b) v[0][b] ^= u[0][b];
    } else {
      F::mul_acc2_n2(u[0], v[0], u[W - 1], v[W - 1], f);
      for (int b = 0; b < 16; ++b) { v[0][b] ^= u[0][b]; v[W-1][b] ^= u[W-1][b]; }
    }
  }
  uint32_t x = 0;
  for (int w = 0; w < W; ++w) for (int b = 0; b < 16; ++b) x ^= u[w][b] ^ v[w][b];
  out[blockIdx.x * 256 + threadIdx.x] = x;
}

int main() {
  uint32_t *fac, *out;
  cudaMalloc(&fac, 4096 * 4);
  cudaMalloc(&out, 148 * 8 * 256 * 4);
  uint32_t h[4096];
  for (int i = 0; i < 4096; ++i) h[i] = (i * 2654435761u) >> 16;
  cudaMemcpy(fac, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 2000;
  for (int W = 1; W <= 2; ++W)
    for (int ctas_per_sm = 1; ctas_per_sm <= 8; ctas_per_sm *= 2) {
      const int grid = 148 * ctas_per_sm;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (W == 1) k<1><<<grid, 256>>>(fac, out, iters); else k<2><<<grid, 256>>>(fac, out, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double muls = double(grid) * 256 * iters * 32 * W;
      printf("W=%d warps/SM=%d: %.3f ms  %.2f T symbol-muls/s (%s)\n", W, ctas_per_sm * 8, ms,
             muls / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
