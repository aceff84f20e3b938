// Microbenchmark (experiments only): bit-sliced GF(2^16) multiply-accumulate
// variants inside a register-resident radix-4 "round" (4 positions x 16
// planes per thread, as in pass_kernel), warp-uniform factors.
//   V=0: mul_acc_n2 (nested 2-bit digits, two uniform branches per digit)
//   V=1: 2-bit digits through a 4-way switch
//   V=2: 3-bit windows (p, x p, x^2 p live) through an 8-way switch
//   V=3: 1-bit digits, predicated XORs (no branches)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/mulbench2.cu -o tools/mulbench2_bin
#include <cstdint>
#include <cstdio>
#include "../paper_1404_3458_b200/csrc/lch_device.cuh"
using F = lch::GF<16, 0x1100Bu>;
constexpr int R = 16;

__device__ __forceinline__ void adv(const uint32_t (&p)[R], uint32_t (&q)[R]) {
#pragma unroll
  for (int b = 0; b < R; ++b) q[b] = F::xor_set(p, F::s1(b));
}

__device__ __forceinline__ void mul_sw2(uint32_t (&u)[R], const uint32_t (&v)[R], uint32_t f) {
  uint32_t p[R];
#pragma unroll
  for (int b = 0; b < R; ++b) p[b] = v[b];
#pragma unroll
  for (int t = 0; t < R; t += 2) {
    uint32_t q[R];
    adv(p, q);
    switch ((f >> t) & 3u) {
      case 1:
#pragma unroll
        for (int b = 0; b < R; ++b) u[b] ^= p[b];
        break;
      case 2:
#pragma unroll
        for (int b = 0; b < R; ++b) u[b] ^= q[b];
        break;
      case 3:
#pragma unroll
        for (int b = 0; b < R; ++b) u[b] = F::lop3_xor(u[b], p[b], q[b]);
        break;
      default:
        break;
    }
    if (t + 2 < R) adv(q, p);
  }
}

__device__ __forceinline__ void mul_w3(uint32_t (&u)[R], const uint32_t (&v)[R], uint32_t f) {
  uint32_t p[R];
#pragma unroll
  for (int b = 0; b < R; ++b) p[b] = v[b];
#pragma unroll
  for (int t = 0; t < R; t += 3) {
    uint32_t q[R], r[R];
    adv(p, q);
    if (t + 2 < R) adv(q, r);
    const uint32_t d = (f >> t) & (t + 2 < R ? 7u : 1u);
    switch (d) {
      case 1:
#pragma unroll
        for (int b = 0; b < R; ++b) u[b] ^= p[b];
        break;
      case 2:
#pragma unroll
        for (int b = 0; b < R; ++b) u[b] ^= q[b];
        break;
      case 3:
#pragma unroll
        for (int b = 0; b < R; ++b) u[b] = F::lop3_xor(u[b], p[b], q[b]);
        break;
      case 4:
#pragma unroll
        for (int b = 0; b < R; ++b) u[b] ^= r[b];
        break;
      case 5:
#pragma unroll
        for (int b = 0; b < R; ++b) u[b] = F::lop3_xor(u[b], p[b], r[b]);
        break;
      case 6:
#pragma unroll
        for (int b = 0; b < R; ++b) u[b] = F::lop3_xor(u[b], q[b], r[b]);
        break;
      case 7:
#pragma unroll
        for (int b = 0; b < R; ++b) u[b] = F::lop3_xor(u[b], p[b], q[b]) ^ r[b];
        break;
      default:
        break;
    }
    if (t + 3 < R) adv(r, p);
  }
}


// predicated accumulation: u ^= p under a (warp-uniform) predicate, 16 planes
// in one asm block so the predicate is set once (no branches at all)
__device__ __forceinline__ void pxor16(uint32_t (&u)[R], const uint32_t (&p)[R], uint32_t cond) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %32, 0;\n"
      "@q xor.b32 %0, %0, %16;\n @q xor.b32 %1, %1, %17;\n @q xor.b32 %2, %2, %18;\n @q xor.b32 %3, %3, %19;\n"
      "@q xor.b32 %4, %4, %20;\n @q xor.b32 %5, %5, %21;\n @q xor.b32 %6, %6, %22;\n @q xor.b32 %7, %7, %23;\n"
      "@q xor.b32 %8, %8, %24;\n @q xor.b32 %9, %9, %25;\n @q xor.b32 %10, %10, %26;\n @q xor.b32 %11, %11, %27;\n"
      "@q xor.b32 %12, %12, %28;\n @q xor.b32 %13, %13, %29;\n @q xor.b32 %14, %14, %30;\n @q xor.b32 %15, %15, %31;\n}"
      : "+r"(u[0]), "+r"(u[1]), "+r"(u[2]), "+r"(u[3]), "+r"(u[4]), "+r"(u[5]), "+r"(u[6]), "+r"(u[7]),
        "+r"(u[8]), "+r"(u[9]), "+r"(u[10]), "+r"(u[11]), "+r"(u[12]), "+r"(u[13]), "+r"(u[14]), "+r"(u[15])
      : "r"(p[0]), "r"(p[1]), "r"(p[2]), "r"(p[3]), "r"(p[4]), "r"(p[5]), "r"(p[6]), "r"(p[7]),
        "r"(p[8]), "r"(p[9]), "r"(p[10]), "r"(p[11]), "r"(p[12]), "r"(p[13]), "r"(p[14]), "r"(p[15]), "r"(cond));
}

__device__ __forceinline__ void mul_pred(uint32_t (&u)[R], const uint32_t (&v)[R], uint32_t f) {
  uint32_t p[R];
#pragma unroll
  for (int b = 0; b < R; ++b) p[b] = v[b];
#pragma unroll
  for (int t = 0; t < R; ++t) {
    pxor16(u, p, (f >> t) & 1u);
    if (t + 1 < R) {
      uint32_t q[R];
      adv(p, q);
#pragma unroll
      for (int b = 0; b < R; ++b) p[b] = q[b];
    }
  }
}

template <int V>
__device__ __forceinline__ void mac(uint32_t (&u)[R], const uint32_t (&v)[R], uint32_t f) {
  if (V == 0) F::mul_acc_n2(u, v, f);
  else if (V == 1) mul_sw2(u, v, f);
  else if (V == 2) mul_w3(u, v, f);
  else mul_pred(u, v, f);
}

template <int V>
__device__ __forceinline__ void bfly(uint32_t (&u)[R], uint32_t (&v)[R], uint32_t f) {
#pragma unroll
  for (int b = 0; b < R; ++b) v[b] ^= u[b];  // inverse butterfly: v' = u + v, u' = u + f v'
  if (f) mac<V>(u, v, f);
}

template <int V>
__global__ void __launch_bounds__(256, 2) k(const uint32_t *fac, uint32_t *out, int iters) {
  uint32_t a0[R], a1[R], a2[R], a3[R];
  for (int b = 0; b < R; ++b) {
    a0[b] = threadIdx.x * 977u + b * 131u;
    a1[b] = a0[b] * 3u;
    a2[b] = a0[b] * 5u;
    a3[b] = a0[b] * 7u;
  }
  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0);
  for (int it = 0; it < iters; ++it) {
    const uint32_t *fp = fac + ((blockIdx.x * 8 + warp + it * 7) & 1023) * 4;
    const uint32_t f0 = __shfl_sync(~0u, fp[0], 0), f1 = __shfl_sync(~0u, fp[1], 0),
                   f2 = __shfl_sync(~0u, fp[2], 0), f3 = __shfl_sync(~0u, fp[3], 0);
    bfly<V>(a0, a1, f0);
    bfly<V>(a2, a3, f1);
    bfly<V>(a0, a2, f2);
    bfly<V>(a1, a3, f3);
  }
  uint32_t x = 0;
  for (int b = 0; b < R; ++b) x ^= a0[b] ^ a1[b] ^ a2[b] ^ a3[b];
  out[blockIdx.x * 256 + threadIdx.x] = x;
}

int main() {
  uint32_t *fac, *out;
  cudaMalloc(&fac, 4096 * 4);
  cudaMalloc(&out, 148 * 8 * 256 * 4);
  uint32_t h[4096];
  for (int i = 0; i < 4096; ++i) h[i] = ((i + 1) * 2654435761u) >> 16;
  cudaMemcpy(fac, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 1000;
  uint32_t ref[4] = {0, 0, 0, 0};
  for (int V = 0; V < 4; ++V) {
    const int grid = 148 * 2;
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (V == 0) k<0><<<grid, 256>>>(fac, out, iters);
      else if (V == 1) k<1><<<grid, 256>>>(fac, out, iters);
      else if (V == 2) k<2><<<grid, 256>>>(fac, out, iters);
      else k<3><<<grid, 256>>>(fac, out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    uint32_t hv[64];
    cudaMemcpy(hv, out, sizeof(hv), cudaMemcpyDeviceToHost);
    ref[V] = hv[0] ^ hv[37];
    const double bf = double(grid) * 256 * iters * 4 * 32;  // symbol-butterflies
    printf("V=%d 16 warps/SM: %.3f ms  %.3f T symbol-butterflies/s  check %08x (%s)\n", V, ms, bf / ms / 1e9,
           ref[V], cudaGetErrorString(cudaGetLastError()));
  }
  printf(ref[0] == ref[1] && ref[1] == ref[2] && ref[2] == ref[3] ? "variants agree\n" : "VARIANTS DIFFER\n");
  return 0;
}
