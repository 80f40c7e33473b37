// Integer tensor-core dequant-GEMV core for the tile layout of mma_layout.cuh
// (2/3/4-bit reference presets).  Replaces the reference's
// ``x @ quant.dequantize(block)`` (quant.py:267-304, model.py:223-226,
// 290-300) like gemv.cuh, with the multiply-adds on mma.sync (IMMA) instead
// of FFMA2:
//
//   y_j = sum_i x_i (c_ij s_i,j/sg + zhat_i,j/g)
//       = 2^-E sum_n 256^n sum_i c_ij d_n,i,jb  +  sum_i x_i zhat_i,j/g
//   A = c_ij 2^p as u8 (one LOP3 per four codes; the tile's 2^p is undone at
//       the end), B = d_n = the signed byte digits of b_i = rint(x_i s_i 2^E),
//   D = s32 accumulators: exact.
// The zero-point term keeps the CUDA-core form (one FFMA per (row, group)).
#pragma once
#include "common.cuh"
#include "gemv.cuh"
#include "mma_layout.cuh"

namespace mg {

MOE_DEV void imma(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                  uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

using gemv::shr_fma;

// One k-step of one slice for this lane: the 4B code words, the B fragment,
// the zero codes of its row (row = lane) and that row's x * zscale * 2^100.
template <int B>
struct Unit {
  uint32_t w[4 * B];
  uint2 bf;
  uint2 z;  // 3/4-bit: 2 groups (bytes 0, 1 of z.x); 2-bit: 8 groups
  float x;
};

template <int B>
MOE_DEV void unit_load(Unit<B>& U, const uint8_t* slice, uint2 bf, const float* xz, int lane) {
  const uint4* cp = reinterpret_cast<const uint4*>(slice);
#pragma unroll
  for (int pl = 0; pl < B; ++pl) {
    const uint4 v = cp[pl * 32 + lane];
    U.w[4 * pl] = v.x;
    U.w[4 * pl + 1] = v.y;
    U.w[4 * pl + 2] = v.z;
    U.w[4 * pl + 3] = v.w;
  }
  U.bf = bf;
  const uint8_t* zc = slice + mt::code_bytes(B);
  if constexpr (B == 2) {
    U.z = reinterpret_cast<const uint2*>(zc)[lane];
  } else {
    U.z.x = reinterpret_cast<const uint16_t*>(zc)[lane];
    U.z.y = 0;
  }
  U.x = xz[lane];
}

// the 8 tiles' MMAs, registers produced tile by tile (few live at a time)
template <int B>
MOE_DEV void unit_math(int (&D)[8][4], float (&zacc)[8], const Unit<B>& U) {
  const uint32_t b0 = U.bf.x, b1 = U.bf.y;
  if constexpr (B == 4) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t m = i < 4 ? 0x0F0F0F0Fu : 0xF0F0F0F0u;
      const int v = 4 * (i & 3);
      imma(D[i], U.w[v] & m, U.w[v + 1] & m, U.w[v + 2] & m, U.w[v + 3] & m, b0, b1);
    }
  } else if constexpr (B == 2) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t m = 0x03030303u << (2 * (i >> 1));
      const int v = 4 * (i & 1);
      imma(D[i], U.w[v] & m, U.w[v + 1] & m, U.w[v + 2] & m, U.w[v + 3] & m, b0, b1);
    }
  } else {
#pragma unroll
    for (int G = 0; G < 4; ++G) {
      const uint32_t w0 = U.w[3 * G], w1 = U.w[3 * G + 1], w2 = U.w[3 * G + 2];
      // byte bits 6..7 of the three words: the codes of register 3
      const uint32_t t = (shr_fma(w0, 6) & 0x03030303u) | (shr_fma(w1, 4) & 0x0C0C0C0Cu) |
                         (shr_fma(w2, 2) & 0x30303030u);
      imma(D[G], w0 & 0x07070707u, w1 & 0x07070707u, w2 & 0x07070707u, t & 0x07070707u, b0, b1);
      imma(D[G + 4], w0 & 0x38383838u, w1 & 0x38383838u, w2 & 0x38383838u, t & 0x38383838u,
           b0, b1);
    }
  }
  // zero codes as subnormal / first-binade floats (linear while the byte sits
  // at bits 0..23): byte j of a word -> zacc scale 2^(8j - 149)
  if constexpr (B == 2) {
    zacc[0] = fmaf(gemv::fbits(U.z.x & 0xffu), U.x, zacc[0]);
    zacc[1] = fmaf(gemv::fbits(U.z.x & 0xff00u), U.x, zacc[1]);
    zacc[2] = fmaf(gemv::fbits(U.z.x & 0xff0000u), U.x, zacc[2]);
    zacc[3] = fmaf(gemv::fbits(shr_fma(U.z.x, 24)), U.x, zacc[3]);
    zacc[4] = fmaf(gemv::fbits(U.z.y & 0xffu), U.x, zacc[4]);
    zacc[5] = fmaf(gemv::fbits(U.z.y & 0xff00u), U.x, zacc[5]);
    zacc[6] = fmaf(gemv::fbits(U.z.y & 0xff0000u), U.x, zacc[6]);
    zacc[7] = fmaf(gemv::fbits(shr_fma(U.z.y, 24)), U.x, zacc[7]);
  } else {
    zacc[0] = fmaf(gemv::fbits(U.z.x & 0xffu), U.x, zacc[0]);
    zacc[1] = fmaf(gemv::fbits(U.z.x & 0xff00u), U.x, zacc[1]);
  }
}

// zacc scale exponent of zero group j (see unit_math): 2^(149 - 8 (j % 4)),
// byte 3 shifted down; times 2^-100 for the x prescale
MOE_DEV constexpr int zexp(int j) { return (j & 3) == 3 ? 49 : 49 - 8 * (j & 3); }

// The slice's 128 outputs (without the per-CTA zoffset sum): exact integer
// digit sums -> one fp32 rounding, tile shift and 2^-E undone, plus the
// zero-point total of each output's group.  Lanes t == 0 write ys[o].
template <int B>
MOE_DEV void finish(const int (&D)[8][4], const float (&zacc)[8], int E, int lane, float* ys) {
  const int g = lane >> 2, t = lane & 3;
  constexpr int NG = B == 2 ? 8 : 2;  // zero groups per slice
  float zt[NG];
#pragma unroll
  for (int j = 0; j < NG; ++j) {  // rows are lanes: sum over the warp
    float z = zacc[j] * __uint_as_float(gemv::pow2_bits(zexp(j)));
#pragma unroll
    for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    zt[j] = z;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float sc = __uint_as_float(gemv::pow2_bits(-E - mt::tile_shift(B, i)));
    const float z = B == 2 ? zt[i] : zt[i >> 2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {  // row g (c = 0) and g + 8
      // digits: t = 0 holds columns 0, 1 (256^0, 256^1), t = 1 columns 2, 3
      long long v = t == 0 ? (long long)D[i][2 * c] + ((long long)D[i][2 * c + 1] << 8)
                  : t == 1 ? ((long long)D[i][2 * c] << 16) + ((long long)D[i][2 * c + 1] << 24)
                           : 0ll;
      v += __shfl_down_sync(0xffffffffu, v, 1);
      if (t == 0) ys[16 * i + g + 8 * c] = fmaf(__ll2float_rn(v), sc, z);
    }
  }
}

// b = rint(xe * s) as four signed byte digits into a (k-step, slice) B table
// (xe = x * 2^E)
MOE_DEV void put_digits(uint8_t* tab, int k, float xe, float s) {
  int b = __float2int_rn(__fmul_rn(xe, s));
  const int d0 = (int)(int8_t)(b & 0xff);
  b = (b - d0) >> 8;
  const int d1 = (int)(int8_t)(b & 0xff);
  b = (b - d1) >> 8;
  const int d2 = (int)(int8_t)(b & 0xff);
  const int d3 = (b - d2) >> 8;
  tab[mt::btab_byte(k, 0)] = (uint8_t)d0;
  tab[mt::btab_byte(k, 1)] = (uint8_t)d1;
  tab[mt::btab_byte(k, 2)] = (uint8_t)d2;
  tab[mt::btab_byte(k, 3)] = (uint8_t)d3;
}

}  // namespace mg
