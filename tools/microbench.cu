// Microbenchmarks that validate the design assumptions of the expert GEMV and
// the copy engine on the B200 before the real kernels are written:
//   1. fp32 FFMA / FFMA2 with subnormal operands (the "code bits as a subnormal
//      float" dequant trick) are exact and full-rate;
//   2. a prototype 2-bit dequant-GEMV reaches a useful fraction of HBM;
//   3. pinned H2D bandwidth for expert-sized copies (58-72 MB), 1 and 2 streams;
//   4. cuStreamWriteValue32 works (slot-ready flags set by the copy stream).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o mb microbench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

// ---------------------------------------------------------------- subnormal FMA
__global__ void k_subnormal(const uint32_t* codes, const float* xs, float* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float m = __uint_as_float(codes[i]);
  float2 a = make_float2(xs[i], xs[i]);
  float2 b = make_float2(m, m);
  float2 c = make_float2(0.f, 1.f);
  float2 r = __ffma2_rn(a, b, c);
  out[2 * i] = r.x;
  out[2 * i + 1] = fmaf(xs[i], m, 0.f);
}

// ---------------------------------------------------------------- zero-copy pull
// GPU-initiated H2D: CTAs read a mapped pinned host buffer over PCIe and store
// into HBM (the alternative to DMA copies issued by a host thread).
template <int UNR>
__global__ void k_pull(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (UNR - 1) * stride < n; i += UNR * stride) {
    uint4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) v[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < UNR; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < n; i += stride) dst[i] = src[i];
}

// ---------------------------------------------------------------- proto GEMV
// Matrix K x N, 2-bit codes, groups of 16 along N.  Device layout:
//   codes uint4 [cb][quad][lane]   (cb = 32-chunk column block, chunk = 16 outputs)
//   zeros uint32 [cb][quad][lane]  (4 zero codes, one per row of the quad)
//   scales uint2 [cb][quad][sg4]   (4 fp16 scales, one per row, sg = 8 chunks)
//   zmeta  half2 [row][N/2048]     (zscale, zoffset per run of 128 groups)
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
k_gemv2(const uint4* __restrict__ codes, const uint32_t* __restrict__ zeros,
        const uint2* __restrict__ scales, const __half2* __restrict__ zmeta,
        const float* __restrict__ x, float* __restrict__ partial,
        int K, int N, int quads_per_split) {
  __shared__ float xs_sh[4096];
  __shared__ float red[WARPS][32 * 17];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cb = blockIdx.x, split = blockIdx.y;
  const int nquads = K / 4;
  const int q0 = split * quads_per_split;
  const int r0 = q0 * 4, nrows = quads_per_split * 4;
  for (int i = threadIdx.x; i < nrows; i += blockDim.x) xs_sh[i] = x[r0 + i] * 0x1p100f;
  __syncthreads();
  const int runs_per_row = N / 2048;
  const int run_col = (cb * 32) / 128;
  float acc[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = 0.f;
  float zacc = 0.f;
  const int qpw = quads_per_split / WARPS;
  const size_t base = (size_t)cb * nquads;
  for (int qq = 0; qq < qpw; ++qq) {
    const int q = q0 + warp * qpw + qq;
    const uint4 w4 = __ldg(codes + (base + q) * 32 + lane);
    const uint32_t z4 = __ldg(zeros + (base + q) * 32 + lane);
    const uint2 s4 = __ldg(scales + (base + q) * 4 + (lane >> 3));
    const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
    const uint32_t sv[4] = {s4.x & 0xffff, s4.x >> 16, s4.y & 0xffff, s4.y >> 16};
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int row = q * 4 + r;
      const float xr = xs_sh[row - r0];
      const float s = __half2float(__ushort_as_half((unsigned short)sv[r]));
      const float xsv = xr * s;
      const __half2 zm = __ldg(zmeta + row * runs_per_row + run_col);
      const float zc = (float)((z4 >> (8 * r)) & 0xff);
      const float zh = fmaf(zc, __low2float(zm), __high2float(zm));
      zacc = fmaf(xr, zh, zacc);
      const uint32_t w = wv[r];
      const uint32_t wh = w >> 16;
      float m[16];
#pragma unroll
      for (int k = 0; k < 12; ++k) m[k] = __uint_as_float(w & (3u << (2 * k)));
#pragma unroll
      for (int k = 12; k < 16; ++k) m[k] = __uint_as_float(wh & (3u << (2 * k - 16)));
#pragma unroll
      for (int k = 0; k < 16; k += 2) {
        float2 r2 = __ffma2_rn(make_float2(xsv, xsv), make_float2(m[k], m[k + 1]),
                               make_float2(acc[k], acc[k + 1]));
        acc[k] = r2.x; acc[k + 1] = r2.y;
      }
    }
  }
  // un-scale: code k sits at bit 2k (k<12) or 2k-16 (k>=12); x was scaled by 2^100
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int pos = k < 12 ? 2 * k : 2 * k - 16;
    float v = acc[k] * exp2f((float)(149 - 100 - pos)) + zacc * 0x1p-100f;
    red[warp][lane * 17 + k] = v;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 32 * 16; t += blockDim.x) {
    const int l = t / 16, k = t % 16;
    float s = 0.f;
    for (int w = 0; w < WARPS; ++w) s += red[w][l * 17 + k];
    partial[(size_t)split * N + (cb * 32 + l) * 16 + k] = s;
  }
}

static float h2f(uint16_t h) { __half hh = *reinterpret_cast<__half*>(&h); return __half2float(hh); }

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("device %s SMs %d smemPerBlockOptin %zu L2 %d clock %d kHz memclk %d kHz bus %d\n", p.name,
         p.multiProcessorCount, p.sharedMemPerBlockOptin, p.l2CacheSize, p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  // ---- 1. subnormal FMA exactness
  {
    const int n = 1 << 16;
    std::vector<uint32_t> c(n); std::vector<float> xs(n);
    srand(1);
    for (int i = 0; i < n; ++i) { int k = rand() % 12; c[i] = (uint32_t)(rand() & 3) << (2 * k); xs[i] = (rand() / (float)RAND_MAX - 0.5f) * 0x1p100f; }
    uint32_t* dc; float *dx, *dout; CK(cudaMalloc(&dc, n * 4)); CK(cudaMalloc(&dx, n * 4)); CK(cudaMalloc(&dout, n * 8));
    CK(cudaMemcpy(dc, c.data(), n * 4, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dx, xs.data(), n * 4, cudaMemcpyHostToDevice));
    k_subnormal<<<n / 256, 256>>>(dc, dx, dout, n); CK(cudaDeviceSynchronize());
    std::vector<float> out(2 * n); CK(cudaMemcpy(out.data(), dout, n * 8, cudaMemcpyDeviceToHost));
    int bad2 = 0, bad1 = 0;
    for (int i = 0; i < n; ++i) {
      double exact = (double)xs[i] * (double)c[i] * std::ldexp(1.0, -149);
      float e0 = (float)exact;  // fma(a,b,0)
      float e1 = (float)(exact + 1.0);
      if (out[2 * i] != e0 && !(out[2*i]==0 && e0==0)) ++bad2;
      if (out[2 * i + 1] != e0) ++bad1;
      (void)e1;
    }
    printf("subnormal FFMA2 mismatches %d / %d ; FFMA mismatches %d / %d\n", bad2, n, bad1, n);
  }
  // ---- 2. proto GEMV 2-bit, K=4096 N=14336 (W1-like), plus timing
  {
    const int K = 4096, N = 14336;
    const int nchunks = N / 16, ncb = nchunks / 32, nquads = K / 4;
    size_t ncode = (size_t)ncb * nquads * 32;  // uint4 count
    std::vector<uint32_t> hcodes(ncode * 4), hzeros(ncode);
    std::vector<uint16_t> hscales((size_t)ncb * nquads * 16);
    std::vector<uint32_t> hzm((size_t)K * (N / 2048));
    std::vector<float> hx(K);
    srand(7);
    for (auto& v : hcodes) v = ((uint32_t)rand() << 16) ^ (uint32_t)rand();
    for (auto& v : hzeros) v = ((uint32_t)rand() << 16) ^ (uint32_t)rand();
    for (auto& v : hscales) { __half h = __float2half(0.005f + 0.02f * rand() / (float)RAND_MAX); v = *reinterpret_cast<uint16_t*>(&h); }
    for (auto& v : hzm) { __half a = __float2half(0.0003f * (1 + rand() % 10)); __half b = __float2half(-0.05f * rand() / (float)RAND_MAX);
      v = (uint32_t)*reinterpret_cast<uint16_t*>(&a) | ((uint32_t)*reinterpret_cast<uint16_t*>(&b) << 16); }
    for (auto& v : hx) v = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
    // host reference (double)
    std::vector<double> ref(N, 0.0);
    for (int cb = 0; cb < ncb; ++cb) for (int q = 0; q < nquads; ++q) for (int lane = 0; lane < 32; ++lane) {
      size_t idx = ((size_t)cb * nquads + q) * 32 + lane;
      int chunk = cb * 32 + lane;
      for (int r = 0; r < 4; ++r) {
        int row = q * 4 + r;
        uint32_t w = hcodes[idx * 4 + r];
        uint16_t sh = hscales[((size_t)cb * nquads + q) * 16 + (lane >> 3) * 4 + r];
        double s = h2f(sh);
        uint32_t zm = hzm[(size_t)row * (N / 2048) + chunk / 128];
        float zc = (float)((hzeros[idx] >> (8 * r)) & 0xff);
        float zh = fmaf(zc, h2f(zm & 0xffff), h2f(zm >> 16));
        for (int k = 0; k < 16; ++k) {
          int c = (w >> (2 * k)) & 3;
          ref[chunk * 16 + k] += (double)hx[row] * ((double)c * s + (double)zh);
        }
      }
    }
    uint4* dcodes; uint32_t* dzeros; uint2* dscales; __half2* dzm; float *dx, *dpart;
    CK(cudaMalloc(&dcodes, ncode * 16)); CK(cudaMalloc(&dzeros, ncode * 4)); CK(cudaMalloc(&dscales, hscales.size() * 2));
    CK(cudaMalloc(&dzm, hzm.size() * 4)); CK(cudaMalloc(&dx, K * 4));
    CK(cudaMemcpy(dcodes, hcodes.data(), ncode * 16, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dzeros, hzeros.data(), ncode * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dscales, hscales.data(), hscales.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dzm, hzm.data(), hzm.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dx, hx.data(), K * 4, cudaMemcpyHostToDevice));
    const int WARPS = 8;
    for (int splits : {16, 32, 64}) {
      int qps = nquads / splits;
      CK(cudaMalloc(&dpart, (size_t)splits * N * 4));
      dim3 grid(ncb, splits);
      k_gemv2<WARPS><<<grid, WARPS * 32>>>(dcodes, dzeros, dscales, dzm, dx, dpart, K, N, qps);
      CK(cudaDeviceSynchronize());
      std::vector<float> part((size_t)splits * N); CK(cudaMemcpy(part.data(), dpart, part.size() * 4, cudaMemcpyDeviceToHost));
      double maxrel = 0, maxabs = 0;
      for (int j = 0; j < N; ++j) { double s = 0; for (int sp = 0; sp < splits; ++sp) s += part[(size_t)sp * N + j];
        maxabs = std::max(maxabs, std::fabs(s - ref[j])); maxrel = std::max(maxrel, std::fabs(s - ref[j]) / (std::fabs(ref[j]) + 1e-3)); }
      // timing: 3 different matrices would exceed L2; here one matrix of 19.4 MB (fits L2!) so flush with a big memset
      size_t flushb = 512ull << 20; void* flush; CK(cudaMalloc(&flush, flushb));
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      float best = 1e9, tot = 0; int reps = 20;
      for (int it = 0; it < reps; ++it) {
        CK(cudaMemsetAsync(flush, it, flushb));
        cudaEventRecord(e0);
        k_gemv2<WARPS><<<grid, WARPS * 32>>>(dcodes, dzeros, dscales, dzm, dx, dpart, K, N, qps);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms); tot += ms;
      }
      double bytes = ncode * 16.0 + ncode * 4.0 + hscales.size() * 2.0 + hzm.size() * 4.0;  // code+zero+scale+zmeta
      printf("gemv2 splits=%d grid=%d CTAs: maxabs %.3g maxrel %.3g | best %.1f us avg %.1f us | %.0f GB/s (best) %.0f GB/s (avg)\n",
             splits, ncb * splits, maxabs, maxrel, best * 1e3, tot / reps * 1e3, bytes / best / 1e6, bytes / (tot / reps) / 1e6);
      cudaFree(flush); cudaFree(dpart);
    }
  }
  // ---- 3. H2D bandwidth
  {
    size_t sz = 71651328;  // 3-bit expert bytes
    int nbuf = 8;
    char* host; CK(cudaHostAlloc(&host, sz * nbuf, cudaHostAllocDefault));
    for (size_t i = 0; i < sz * nbuf; i += 4096) host[i] = (char)i;
    char* dev; CK(cudaMalloc(&dev, sz * nbuf));
    cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int it = 0; it < 2; ++it) CK(cudaMemcpyAsync(dev, host, sz, cudaMemcpyHostToDevice, s1));
    CK(cudaStreamSynchronize(s1));
    float best = 1e9;
    for (int it = 0; it < 10; ++it) {
      cudaEventRecord(e0, s1);
      CK(cudaMemcpyAsync(dev + (it % nbuf) * sz, host + (it % nbuf) * sz, sz, cudaMemcpyHostToDevice, s1));
      cudaEventRecord(e1, s1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    printf("H2D 1 stream single copy %.1f MB: best %.3f ms = %.1f GB/s\n", sz / 1e6, best, sz / best / 1e6);
    // 8 back-to-back copies on one stream
    cudaEventRecord(e0, s1);
    for (int i = 0; i < nbuf; ++i) CK(cudaMemcpyAsync(dev + i * sz, host + i * sz, sz, cudaMemcpyHostToDevice, s1));
    cudaEventRecord(e1, s1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("H2D 1 stream %d copies back-to-back: %.3f ms = %.1f GB/s\n", nbuf, ms, nbuf * sz / ms / 1e6);
    // 2 streams
    cudaEventRecord(e0, s1);
    cudaStreamWaitEvent(s2, e0, 0);
    for (int i = 0; i < nbuf; ++i) CK(cudaMemcpyAsync(dev + i * sz, host + i * sz, sz, cudaMemcpyHostToDevice, (i & 1) ? s2 : s1));
    cudaEvent_t e2; cudaEventCreate(&e2); cudaEventRecord(e2, s2); cudaStreamWaitEvent(s1, e2, 0);
    cudaEventRecord(e1, s1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("H2D 2 streams %d copies: %.3f ms = %.1f GB/s\n", nbuf, ms, nbuf * sz / ms / 1e6);
    // chunked 4 MB pieces
    cudaEventRecord(e0, s1);
    size_t chunk = 4 << 20;
    for (int i = 0; i < nbuf; ++i) for (size_t off = 0; off < sz; off += chunk)
      CK(cudaMemcpyAsync(dev + i * sz + off, host + i * sz + off, std::min(chunk, sz - off), cudaMemcpyHostToDevice, s1));
    cudaEventRecord(e1, s1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("H2D 1 stream 4MB chunks: %.3f ms = %.1f GB/s\n", ms, nbuf * sz / ms / 1e6);
    // D2D for reference
    cudaEventRecord(e0, s1);
    CK(cudaMemcpyAsync(dev, dev + 4 * sz, 4 * sz, cudaMemcpyDeviceToDevice, s1));
    cudaEventRecord(e1, s1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("D2D copy %.1f MB: %.3f ms = %.1f GB/s (r+w)\n", 4 * sz / 1e6, ms, 2 * 4 * sz / ms / 1e6);
    // zero-copy pull kernel from mapped pinned memory
    {
      char* hm; CK(cudaHostAlloc(&hm, sz, cudaHostAllocMapped));
      memset(hm, 1, sz);
      char* hd; CK(cudaHostGetDevicePointer((void**)&hd, hm, 0));
      for (int nb : {2, 4, 8, 16, 32, 64, 148, 296}) {
        for (int thr : {256, 1024}) {
          float bestp = 1e9;
          for (int it = 0; it < 5; ++it) {
            cudaEventRecord(e0, s1);
            k_pull<8><<<nb, thr, 0, s1>>>((const uint4*)hd, (uint4*)dev, sz / 16);
            cudaEventRecord(e1, s1); CK(cudaEventSynchronize(e1));
            float m2; cudaEventElapsedTime(&m2, e0, e1); bestp = std::min(bestp, m2);
          }
          printf("zero-copy pull %3d CTAs x %4d thr: %.3f ms = %.1f GB/s\n", nb, thr, bestp, sz / bestp / 1e6);
        }
      }
      // DMA copy concurrent with a pull on another stream (two engines on one link)
      cudaEventRecord(e0, s1);
      cudaStreamWaitEvent(s2, e0, 0);
      CK(cudaMemcpyAsync(dev + sz, host, sz, cudaMemcpyHostToDevice, s2));
      k_pull<8><<<16, 1024, 0, s1>>>((const uint4*)hd, (uint4*)dev, sz / 16);
      cudaEvent_t e3; cudaEventCreate(&e3); cudaEventRecord(e3, s2); cudaStreamWaitEvent(s1, e3, 0);
      cudaEventRecord(e1, s1); CK(cudaEventSynchronize(e1));
      float m3; cudaEventElapsedTime(&m3, e0, e1);
      printf("DMA + pull concurrently (2 x %.1f MB): %.3f ms = %.1f GB/s\n", sz / 1e6, m3, 2 * sz / m3 / 1e6);
      cudaFreeHost(hm);
    }
    // ---- 4. stream write value
    CUdeviceptr flag; cuMemAlloc(&flag, 4); cuMemsetD32(flag, 0, 1);
    CUresult r = cuStreamWriteValue32((CUstream)s1, flag, 42, CU_STREAM_WRITE_VALUE_DEFAULT);
    cudaStreamSynchronize(s1);
    uint32_t v = 0; cuMemcpyDtoH(&v, flag, 4);
    int attr = 0; cuDeviceGetAttribute(&attr, CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_MEM_OPS_V1, 0);
    printf("cuStreamWriteValue32 result %d value %u (memops attr %d)\n", (int)r, v, attr);
    cudaFreeHost(host); cudaFree(dev);
  }
  return 0;
}
