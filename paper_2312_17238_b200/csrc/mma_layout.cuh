// Tensor-core tile layout of a 2/3/4-bit group-quantized matrix and the
// register maps shared by the tiler (tile.cu) and the dequant-GEMV (gemv).
//
// Idea: a b-bit code c masked in place at bit q (q + b <= 10)
// of a 16-bit lane is, read as an IEEE fp16, the subnormal c * 2^(q-24) --
// exact, and exactly what mma.sync.m16n8k16 (fp16 in, fp32 accumulate)
// multiplies.  One LOP3 therefore yields TWO ready A-operand elements (the low
// and high halves of a 32-bit word), and the multiply-adds go to the tensor
// pipe instead of the FMA pipe: ~0.55 ALU instructions per weight instead of
// the CUDA-core kernel's ~1.7 (one LOP3 + half an FFMA2 + shifts per weight).
// The input vector enters as the B operand, x * scale split into three fp16
// pieces (n = 0, 1, 2 of the n8 tile), so the products are exact and the
// only rounding is the fp32 accumulation -- as in the reference's fp32 GEMV.
//
// Geometry (rows = reduction dim i, outputs j; x[K] @ W[K,N]):
//   k-step   = 16 consecutive rows (the MMA K)
//   slice    = 128 consecutive outputs of one k-step = 8 m16 tiles, one warp
//   cb       = 8 slices = 1024 outputs (the last cb of a matrix may be narrower)
//   record   = one (cb, k-step): its slices in order, each slice
//              [codes 256*b bytes][zero codes 16*128/g bytes]
//   records are stored [cb][k-step]; then the scale section [cb][row][1024/sg]
//   (f16), then the zero-point runs (zmeta) as in the CUDA-core layout.
// Total bytes = codes + zeros + scales + zmeta = quant.payload_nbytes: a byte
// permutation of the reference block (quant.py:76-102, 332-343), so an expert
// buffer stays exactly expert_bytes and the pinned arena holds this layout.
//
// Lane (g = lane/4, t = lane%4) of a slice owns, per k-step, the A fragments
// of the 8 tiles: tile i, slot s in {a01, a23, a45, a67} = rows (16i + g +
// 8*(s&1)) of the output dim, k = 2t + 8*(s>>1) and k + 1 (low/high half).
// Its 64 codes are 2b words, stored as uint2 planes [plane][lane].  Register
// r (0..31) of the lane comes from word v, field f; registers pair up (same
// q) into (tile, row class): pair p -> tile p/2, row class p%2 (rows g or
// g+8), elements e = 0/1 -> k-halves (2t, 2t+8).
#pragma once
#include <stdint.h>

namespace mt {

constexpr int KS = 16;          // rows per k-step
constexpr int SO = 128;         // outputs per slice (warp)
constexpr int CBS = 8;          // slices per column block
constexpr int CBO = SO * CBS;   // outputs per column block

__host__ __device__ constexpr int words(int b) { return 2 * b; }      // per lane per k-step
__host__ __device__ constexpr int code_bytes(int b) { return 256 * b; }
__host__ __device__ constexpr int zero_bytes(int g) { return 16 * (SO / g); }
__host__ __device__ constexpr int slice_bytes(int b, int g) { return code_bytes(b) + zero_bytes(g); }

// ---- register r -> pair (tile, row class) and element
__host__ __device__ constexpr int pair_reg(int b, int p, int e) {
  return b == 4 ? 4 * (p >> 1) + (p & 1) + 2 * e
       : b == 2 ? (p < 12 ? 8 * (p / 3) + p % 3 + 5 * e
                  : p == 12 ? 3 + 8 * e : p == 13 ? 19 + 8 * e : p == 14 ? 4 + 8 * e : 20 + 8 * e)
                : (p < 6 ? 5 * p + 3 * e
                  : p < 12 ? 5 * (p - 6) + 1 + 3 * e
                  : p == 12 ? 2 + 5 * e : p == 13 ? 12 + 5 * e : p == 14 ? 22 + 5 * e : 30 + e);
}
// mantissa bit q of the pair's fields: element value = code * 2^(q - 24)
__host__ __device__ constexpr int pair_q(int b, int p) {
  return b == 4 ? 4 * (p & 1) : b == 2 ? (p < 12 ? 2 * (p % 3) : p < 14 ? 6 : 8)
                                       : (p < 6 ? 0 : p < 12 ? 3 : 6);
}

// ---- register r -> source word and original bit offset in each 16-bit half
// (assembled registers, 3-bit r = 30/31: the code's bit k sits in bit 15 of
// word 3*(r-30) + k; -1 returned)
__host__ __device__ constexpr int reg_word(int b, int r) {
  return b == 4 ? r / 4 : b == 2 ? r / 8 : (r < 30 ? r / 5 : -1);
}
__host__ __device__ constexpr int reg_off(int b, int r) {
  return b == 4 ? 4 * (r % 4) : b == 2 ? 2 * (r % 8) : (r < 30 ? 3 * (r % 5) : -1);
}

// ---- lane-local code coordinates of (tile i, pair row class c, element e)
__host__ __device__ constexpr int out_of(int i, int c, int g) { return 16 * i + g + 8 * c; }
__host__ __device__ constexpr int k_of(int e, int t) { return 2 * t + 8 * e; }

// ---- zero codes of a slice: byte index -> (group within slice, row in k-step)
__host__ __device__ inline void zero_pos(int g, int byte, int* grp, int* row) {
  if (g == 64) {  // 2 groups x 16 rows: lane l reads byte l
    *grp = byte >> 4;
    *row = byte & 15;
  } else {        // g == 16: 8 groups x 16 rows: lane l reads the u32 at 4l
    const int l = byte >> 2, j = byte & 3;
    *grp = l & 7;
    *row = 4 * (l >> 3) + j;
  }
}

// B-operand table entry of (k-step, slice): [piece n 0..2][t 0..3][4 halves
// k = 2t, 2t+1, 2t+8, 2t+9] = 96 bytes; lane (g, t) loads the uint2 at
// (min(g,2)*4 + t)
constexpr int BTAB = 48;  // halves per (k-step, slice)
__host__ __device__ constexpr int btab_half(int k, int n) {
  return n * 16 + ((k & 7) >> 1) * 4 + (k & 1) + 2 * (k >> 3);
}

}  // namespace mt
