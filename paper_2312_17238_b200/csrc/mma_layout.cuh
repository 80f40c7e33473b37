// Tensor-core tile layout of a 2/3/4-bit group-quantized matrix and the
// register maps shared by the tiler (tile.cu) and the dequant-GEMV
// (mma_gemv.cuh, mgemv_kernel.cuh).
//
// Idea: the b-bit codes are the u8 A operand of the integer
// tensor-core MMA (mma.sync m16n8k32 .u8 x .s8 -> .s32).  A code masked in
// place inside its byte is code * 2^p (p = 0, 2, 3, 4 or 6; at most 240), so
// one LOP3 yields FOUR ready A elements and the tile's accumulator carries
// the 2^p.  The input vector enters as the B operand: b = x * s (x times the
// row's f16 scale, one fp32 rounding as in the reference's fp32 GEMV) as a
// per-CTA fixed-point integer (|b| < 2^30) split into four signed bytes --
// the n = 0..3 columns of the n8 tile.  The MMA then accumulates exactly in
// int32; the only roundings are x * s, b's fixed point (2^-31 of the CTA's
// largest |x * s|) and one int64 -> fp32 conversion per output.
//
// Geometry (rows = reduction dim i, outputs j; x[K] @ W[K,N]):
//   k-step   = 32 consecutive rows (the MMA K)
//   slice    = 128 consecutive outputs of one k-step = 8 m16 tiles, one warp
//   cb       = 8 slices = 1024 outputs (the last cb of a matrix may be narrower)
//   record   = one (cb, k-step): its slices in order, each slice
//              [codes 512*b bytes: uint4 planes [b][lane]]
//              [zero codes: [32 rows][128/g groups] u8]
//   records are stored [cb][k-step]; then the scale section [cb][row][1024/sg]
//   (f16), then the zero-point runs (zmeta) as in the CUDA-core layout.
// Total bytes = codes + zeros + scales + zmeta = quant.payload_nbytes: a byte
// permutation of the reference block (quant.py:76-102, 332-343), so an expert
// buffer stays exactly expert_bytes and the pinned arena holds this layout.
//
// Lane (g = lane/4, t = lane%4) of a slice holds, per k-step, the A fragments
// of the 8 tiles: tile i, register r (0..3), byte e (0..3) = output row
// 16 i + g + 8 (r & 1), reduction row k = 4 t + 16 (r >> 1) + e.  Its 128
// codes are 4b words (word v = 4 * plane + component of the uint4).
#pragma once
#include <stdint.h>

namespace mt {

constexpr int KS = 32;          // rows per k-step
constexpr int SO = 128;         // outputs per slice (warp)
constexpr int CBS = 8;          // slices per column block
constexpr int CBO = SO * CBS;   // outputs per column block

__host__ __device__ constexpr int words(int b) { return 4 * b; }  // per lane per k-step
__host__ __device__ constexpr int code_bytes(int b) { return 512 * b; }
__host__ __device__ constexpr int zero_bytes(int g) { return KS * (SO / g); }
__host__ __device__ constexpr int slice_bytes(int b, int g) { return code_bytes(b) + zero_bytes(g); }

// log2 of the power of two tile i's codes carry in their bytes
__host__ __device__ constexpr int tile_shift(int b, int i) {
  return b == 4 ? (i < 4 ? 0 : 4) : b == 2 ? 2 * (i >> 1) : (i < 4 ? 0 : 3);
}

// lane-local coordinates of (tile i, register r, byte e)
__host__ __device__ constexpr int out_of(int i, int r, int g) { return 16 * i + g + 8 * (r & 1); }
__host__ __device__ constexpr int k_of(int r, int e, int t) { return 4 * t + 16 * (r >> 1) + e; }

// where code bit kb (0..b-1) of (tile i, register r, byte e) lives: word and
// bit position inside the lane's 4b words
__host__ __device__ inline void code_bit(int b, int i, int r, int e, int kb, int* word, int* bit) {
  if (b == 4) {
    *word = 4 * (i & 3) + r;
    *bit = 8 * e + (i < 4 ? 0 : 4) + kb;
  } else if (b == 2) {
    *word = 4 * (i & 1) + r;
    *bit = 8 * e + 2 * (i >> 1) + kb;
  } else {  // 3-bit: groups of three words, byte bits 6..7 carry the r = 3 codes
    const int G = i & 3, hi = i >= 4;
    if (r < 3) {
      *word = 3 * G + r;
      *bit = 8 * e + 3 * hi + kb;
    } else {  // t-byte bit tb = 3 hi + kb: bits (0,1) <- word 3G, (2,3) <- 3G+1, (4,5) <- 3G+2
      const int tb = 3 * hi + kb;
      *word = 3 * G + (tb >> 1);
      *bit = 8 * e + 6 + (tb & 1);
    }
  }
}

// zero codes of a slice: [row][group] bytes
__host__ __device__ constexpr int zero_off(int g, int row, int grp) { return row * (SO / g) + grp; }

// B-operand table of one (k-step, slice): [digit n 0..3][t 0..3][8 bytes:
// rows 4t..4t+3, 4t+16..4t+19]; lane (g < 4, t) loads the uint2 at (4g + t)
constexpr int BTAB = 128;  // bytes per (k-step, slice)
__host__ __device__ constexpr int btab_byte(int k, int n) {
  return n * 32 + ((k & 15) >> 2) * 8 + (k & 3) + 4 * (k >> 4);
}

}  // namespace mt
