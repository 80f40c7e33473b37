// Shared device helpers and the device-side data layout of the engine.
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#define MOE_DEV __device__ __forceinline__

// ---------------------------------------------------------------- loads
MOE_DEV uint4 ld_nc_v4(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
MOE_DEV uint32_t ld_nc_u32(const uint32_t* p) {
  uint32_t r;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
MOE_DEV uint2 ld_nc_v2(const uint2* p) {
  uint2 r;
  asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
MOE_DEV uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t r;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}
MOE_DEV float h2f_bits(uint32_t h16) { return __half2float(__ushort_as_half((unsigned short)h16)); }

// ---------------------------------------------------------------- reductions
MOE_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
MOE_DEV double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
MOE_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide double sum; `sh` needs >= 32 doubles.  All threads get the result.
MOE_DEV double block_sum_d(double v, double* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum_d(v);
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < nw; ++i) t += sh[i];  // fixed order -> deterministic
  return t;
}

// ---------------------------------------------------------------- layout
// Tiled device layout of one K x N matrix (x[K] @ W[K,N]).  A "chunk" is WC
// consecutive outputs of one row; a "quad" is 4 consecutive rows; 32 chunks form
// a column block (cb).  Record (quad, chunk) = the chunk's bytes for the 4 rows,
// R bytes = 16*NV uint4; records are stored [cb][quad][v][lane] so each warp
// load instruction is one contiguous 512 B segment.
//   quant (bits 2/3/4): the record bytes are the reference bitstream bytes of
//     the chunk (quant.py:105-113 packing), zeros [quad][G] u32 (4 rows' u8
//     zero codes), scales [quad][S] uint2 (4 rows' f16), zmeta [run] half2.
//   dense f16 / f32: the record holds the raw row values.
struct MatDev {
  const uint4* rec;
  const uint32_t* zeros;
  const uint2* scales;
  const __half2* zmeta;
  int K, N;      // rows (reduction dim), cols (outputs)
  int G, S;      // zero groups / scale groups per row
  int g_log2;    // zero group size (weights)
  int sg_log2;   // scale group size (weights) = zmeta run length (groups)
  int bits;      // 2,3,4 quant; 16, 32 dense
};

template <int BITS> struct Fmt;
template <> struct Fmt<2>  { static constexpr int WC = 16, NV = 1; };
template <> struct Fmt<3>  { static constexpr int WC = 32, NV = 3; };
template <> struct Fmt<4>  { static constexpr int WC = 8,  NV = 1; };
template <> struct Fmt<16> { static constexpr int WC = 8,  NV = 4; };
template <> struct Fmt<32> { static constexpr int WC = 4,  NV = 4; };

__host__ __device__ inline int fmt_wc(int bits) {
  return bits == 2 ? 16 : bits == 3 ? 32 : bits == 4 ? 8 : bits == 16 ? 8 : 4;
}
__host__ __device__ inline int fmt_nv(int bits) { return bits == 3 ? 3 : (bits >= 16 ? 4 : 1); }

// record (cb, quad, v, lane) -> uint4 index
__host__ __device__ inline int64_t rec_index(int cb, int quad, int v, int lane, int nquads,
                                             int nchunks, int nv) {
  const int wcb = min(32, nchunks - cb * 32);
  return (int64_t)cb * 32 * nquads * nv + ((int64_t)quad * nv + v) * wcb + lane;
}
