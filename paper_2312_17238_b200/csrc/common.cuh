// Shared device helpers and the device-side data layout of the engine.
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "mma_layout.cuh"

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
// Tiled device layout of one K x N matrix (x[K] @ W[K,N]), built for a
// bulk-copy (cp.async.bulk) pipeline through shared memory.
//   chunk  = WC consecutive outputs of one row (one lane's outputs)
//   quad   = 4 consecutive rows
//   column block (cb) = 32 chunks (the 32 lanes of a warp); the last cb of a
//            matrix may be narrower (wcb < 32 chunks)
// Record (cb, quad) holds everything one warp needs for 4 rows of its cb,
// contiguously:
//   codes   [NV][wcb] uint4   the chunk's bytes for the 4 rows: reference
//                             bitstream bytes (quant.py:105-113) for bits
//                             2/3/4, raw row values for dense f16 / f32
//   zeros   [ZPR] u32         4 rows' u8 zero codes per zero group (quant only)
//   scales  [SPR] uint2       4 rows' f16 scales per scale group (quant only)
// ZPR = wcb*WC/g zero groups and SPR = wcb*WC/sg scale groups per row of the
// cb.  Records are stored [cb][quad], so the records of one cb over a range
// of quads are one contiguous byte range = one bulk copy.  The zero-point
// metadata (one (zscale, zoffset) f16 pair per run of sg groups, flat over
// the whole matrix, quant.py:147-178) follows all records.  For the 2/3-bit
// presets at Mixtral shape the layout is a pure byte permutation of the
// reference block: total bytes == payload_nbytes (quant.py:332-343), so an
// expert buffer is exactly expert_bytes.
struct MatDev {
  const uint8_t* base;   // records (absolute, or byte offset when relative)
  const __half2* zmeta;  // [nruns] (absolute, or byte offset when relative)
  int K, N;              // rows (reduction dim), cols (outputs)
  int nquads, nchunks, ncb;
  int nqp;               // quads per cb in storage: nquads rounded up to a multiple
                         // of 8 (padding records are zero; only when K % 32 != 0)
  int rb_full;           // record bytes of a full (32-chunk) cb
  int G;                 // zero groups per row (N / g)
  int g_log2;            // zero group size (weights)
  int sg_log2;           // scale group size (weights) = zmeta run length (groups)
  int bits;              // 2,3,4 quant; 16, 32 dense
  int runs_uniform;      // 1: in every row the groups of a cb share one zero run
  // tensor-core tile layout (mma_layout.cuh; quant formats with N % 128 == 0,
  // K % 16 == 0, preset grouping): a "quad" is then a 16-row k-step, a cb is
  // 1024 outputs, nchunks counts 128-output slices, and the f16 scales live in
  // their own section [cb][row][1024/sg] at `scl` (absolute, or a byte offset
  // when the matrix is relative like zmeta)
  int mma;
  const __half* scl;
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

// bytes of one (cb, quad) record for a cb of `wcb` chunks, rounded up to 16 so
// every record (uint4 code loads) and every bulk copy stays 16-byte aligned.
// No padding for the 2/3-bit presets with full column blocks (672 / 1664 B);
// 4-bit records carry 8 pad bytes (536 -> 544).
__host__ __device__ inline int rec_bytes(int bits, int wcb, int g_log2, int sg_log2) {
  int b = 16 * fmt_nv(bits) * wcb;
  if (bits <= 4) {
    const int outs = wcb * fmt_wc(bits);
    b += 4 * (outs >> g_log2) + 8 * (outs >> sg_log2);
  }
  return (b + 15) & ~15;
}
__host__ __device__ inline int64_t cb_offset(const MatDev& M, int cb) {
  return (int64_t)cb * M.nqp * M.rb_full;
}
// tensor-core layout: record bytes of column block cb (slices it holds), and
// its first slice / row rows of the scale section
__host__ __device__ inline int mma_slices(const MatDev& M, int cb) {
  return M.nchunks - cb * mt::CBS < mt::CBS ? M.nchunks - cb * mt::CBS : mt::CBS;
}
__host__ __device__ inline int mma_rec_bytes(const MatDev& M, int cb) {
  return mma_slices(M, cb) * mt::slice_bytes(M.bits, 1 << M.g_log2);
}
// scales per row of cb (1024 / sg for a full cb)
__host__ __device__ inline int mma_nsc(const MatDev& M, int cb) {
  return (mma_slices(M, cb) * mt::SO) >> M.sg_log2;
}
__host__ __device__ inline int64_t mma_scl_offset(const MatDev& M, int cb) {  // in halves
  return (int64_t)cb * M.K * (mt::CBO >> M.sg_log2);
}
