// Probe for the tensor-core dequant-GEMV design: does
// mma.sync.m16n8k16 f32.f16.f16.f32 on sm_100a take fp16 SUBNORMAL A operands
// exactly (a masked b-bit code read as an fp16 bit pattern is c * 2^(p-24)),
// and what is its issue throughput next to LOP3?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_probe tools/mma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_fp16.h>
#include <vector>

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4],
                                         const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// exactness: one warp, A[16][16] fp16 bit patterns, B[16][8] fp16, D = A B (one MMA)
__global__ void k_exact(const uint16_t* A, const uint16_t* B, float* D) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  auto ah = [&](int r, int c) { return (uint32_t)A[r * 16 + c]; };
  auto bh = [&](int k, int n) { return (uint32_t)B[k * 8 + n]; };
  uint32_t a[4] = {ah(g, 2 * t) | ah(g, 2 * t + 1) << 16, ah(g + 8, 2 * t) | ah(g + 8, 2 * t + 1) << 16,
                   ah(g, 2 * t + 8) | ah(g, 2 * t + 9) << 16,
                   ah(g + 8, 2 * t + 8) | ah(g + 8, 2 * t + 9) << 16};
  uint32_t b[2] = {bh(2 * t, g) | bh(2 * t + 1, g) << 16, bh(2 * t + 8, g) | bh(2 * t + 9, g) << 16};
  float d[4] = {0, 0, 0, 0};
  mma16816(d, a, b);
  D[g * 8 + 2 * t] = d[0];
  D[g * 8 + 2 * t + 1] = d[1];
  D[(g + 8) * 8 + 2 * t] = d[2];
  D[(g + 8) * 8 + 2 * t + 1] = d[3];
}

// throughput: each warp issues `iters` x 8 independent MMAs (+ optional LOP3s)
template <int LOPS>
__global__ void k_rate(int iters, float* out, uint32_t seed) {
  uint32_t a[4] = {seed, seed * 3u, seed * 5u, seed * 7u};
  uint32_t b[2] = {seed ^ 0x3c003c00u, seed ^ 0x3c003c00u};
  float d[8][4] = {};
  uint32_t w = seed + threadIdx.x, acc = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      mma16816(d[j], a, b);
#pragma unroll
      for (int l = 0; l < LOPS; ++l) {
        acc ^= (w & (0x00070007u << l)) | acc;
        w += 0x9E3779B9u;
      }
    }
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  if (s == 1.2345f || acc == 0x12345) out[0] = s + acc;
}

int main() {
  // ---- exactness
  std::vector<uint16_t> A(256), B(128);
  srand(1);
  for (int i = 0; i < 256; ++i) {
    const int c = rand() & 7, p = 3 * (rand() % 3);  // 3-bit code at field 0/3/6
    A[i] = (uint16_t)(c << p);                       // subnormal: c * 2^(p-24)
  }
  for (int i = 0; i < 128; ++i) {
    const float v = ((rand() / (float)RAND_MAX) - 0.5f) * 60000.f;
    B[i] = __half_as_ushort(__float2half_rn(v));
  }
  uint16_t *dA, *dB;
  float* dD;
  cudaMalloc(&dA, 512);
  cudaMalloc(&dB, 256);
  cudaMalloc(&dD, 512);
  cudaMemcpy(dA, A.data(), 512, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), 256, cudaMemcpyHostToDevice);
  k_exact<<<1, 32>>>(dA, dB, dD);
  std::vector<float> D(128);
  cudaMemcpy(D.data(), dD, 512, cudaMemcpyDeviceToHost);
  double maxrel = 0;
  int zeros = 0;
  for (int m = 0; m < 16; ++m)
    for (int n = 0; n < 8; ++n) {
      double ref = 0, mag = 0;
      for (int k = 0; k < 16; ++k) {
        const double a = (double)A[m * 16 + k] * ldexp(1.0, -24);
        const double b = __half2float(__ushort_as_half(B[k * 8 + n]));
        ref += a * b;
        mag += fabs(a * b);
      }
      const double e = fabs(D[m * 8 + n] - ref) / (mag > 0 ? mag : 1);
      if (D[m * 8 + n] == 0 && ref != 0) ++zeros;
      maxrel = e > maxrel ? e : maxrel;
    }
  printf("exact: max |D - AB| / sum|a b| = %.3g (2^-23 = %.3g), flushed-to-zero outputs %d\n",
         maxrel, ldexp(1.0, -23), zeros);

  // ---- throughput
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* dout;
  cudaMalloc(&dout, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    for (int lops = 0; lops < 3; ++lops) {
      auto run = [&]() {
        if (lops == 0) k_rate<0><<<sms, warps * 32>>>(iters, dout, 7);
        if (lops == 1) k_rate<4><<<sms, warps * 32>>>(iters, dout, 7);
        if (lops == 2) k_rate<8><<<sms, warps * 32>>>(iters, dout, 7);
      };
      run();
      cudaEventRecord(e0);
      run();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double mmas = (double)sms * warps * iters * 8;
      int clk = 0;
      cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      const double cyc = ms * 1e-3 * clk * 1e3;
      printf("warps/SM %2d LOP3 per MMA %d: %.3f MMA/clk/SM (%.1f TFLOP/s dense-equivalent)\n",
             warps, lops * 4, mmas / sms / cyc, mmas * 4096 * 2 / (ms * 1e-3) / 1e12);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
