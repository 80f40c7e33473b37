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

// One k-step of one slice for this lane: the 4B code words, the zero codes of
// its row (row = lane) and that row's x * zscale * 2^100 for each of the NC
// input columns.
template <int B, int NC>
struct Unit {
  uint32_t w[4 * B];
  uint2 z;  // 3/4-bit: 2 groups (bytes 0, 1 of z.x); 2-bit: 8 groups
  float x[NC];
};

// xz: [NC][xstride] rows of x * zscale * 2^100, this k-step's rows at xz[.. + lane]
template <int B, int NC>
MOE_DEV void unit_load(Unit<B, NC>& U, const uint8_t* slice, const float* xz, int xstride,
                       int lane) {
  const uint4* cp = reinterpret_cast<const uint4*>(slice);
#pragma unroll
  for (int pl = 0; pl < B; ++pl) {
    const uint4 v = cp[pl * 32 + lane];
    U.w[4 * pl] = v.x;
    U.w[4 * pl + 1] = v.y;
    U.w[4 * pl + 2] = v.z;
    U.w[4 * pl + 3] = v.w;
  }
  const uint8_t* zc = slice + mt::code_bytes(B);
  if constexpr (B == 2) {
    U.z = reinterpret_cast<const uint2*>(zc)[lane];
  } else {
    U.z.x = reinterpret_cast<const uint16_t*>(zc)[lane];
    U.z.y = 0;
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) U.x[c] = xz[c * xstride + lane];
}

// the 8 tiles' MMAs, A registers produced tile by tile (few live at a time)
// and reused by the NM column groups' B fragments
template <int NM>
MOE_DEV void imma_n(int (&D)[NM][8][4], int i, uint32_t a0, uint32_t a1, uint32_t a2,
                    uint32_t a3, const uint2 (&bf)[NM]) {
#pragma unroll
  for (int m = 0; m < NM; ++m) imma(D[m][i], a0, a1, a2, a3, bf[m].x, bf[m].y);
}

template <int B, int NM, int NC>
MOE_DEV void unit_math(int (&D)[NM][8][4], float (&zacc)[NC][8], const Unit<B, NC>& U,
                       const uint2 (&bf)[NM]) {
  if constexpr (B == 4) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t m = i < 4 ? 0x0F0F0F0Fu : 0xF0F0F0F0u;
      const int v = 4 * (i & 3);
      imma_n<NM>(D, i, U.w[v] & m, U.w[v + 1] & m, U.w[v + 2] & m, U.w[v + 3] & m, bf);
    }
  } else if constexpr (B == 2) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t m = 0x03030303u << (2 * (i >> 1));
      const int v = 4 * (i & 1);
      imma_n<NM>(D, i, U.w[v] & m, U.w[v + 1] & m, U.w[v + 2] & m, U.w[v + 3] & m, bf);
    }
  } else {
#pragma unroll
    for (int G = 0; G < 4; ++G) {
      const uint32_t w0 = U.w[3 * G], w1 = U.w[3 * G + 1], w2 = U.w[3 * G + 2];
      // byte bits 6..7 of the three words: the codes of register 3
      const uint32_t t = (shr_fma(w0, 6) & 0x03030303u) | (shr_fma(w1, 4) & 0x0C0C0C0Cu) |
                         (shr_fma(w2, 2) & 0x30303030u);
      imma_n<NM>(D, G, w0 & 0x07070707u, w1 & 0x07070707u, w2 & 0x07070707u, t & 0x07070707u,
                 bf);
      imma_n<NM>(D, G + 4, w0 & 0x38383838u, w1 & 0x38383838u, w2 & 0x38383838u,
                 t & 0x38383838u, bf);
    }
  }
  // zero codes as subnormal / first-binade floats (linear while the byte sits
  // at bits 0..23): byte j of a word -> zacc scale 2^(8j - 149)
  float zf[8];
  if constexpr (B == 2) {
    zf[0] = gemv::fbits(U.z.x & 0xffu);
    zf[1] = gemv::fbits(U.z.x & 0xff00u);
    zf[2] = gemv::fbits(U.z.x & 0xff0000u);
    zf[3] = gemv::fbits(shr_fma(U.z.x, 24));
    zf[4] = gemv::fbits(U.z.y & 0xffu);
    zf[5] = gemv::fbits(U.z.y & 0xff00u);
    zf[6] = gemv::fbits(U.z.y & 0xff0000u);
    zf[7] = gemv::fbits(shr_fma(U.z.y, 24));
  } else {
    zf[0] = gemv::fbits(U.z.x & 0xffu);
    zf[1] = gemv::fbits(U.z.x & 0xff00u);
  }
  constexpr int NG = B == 2 ? 8 : 2;
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int j = 0; j < NG; ++j) zacc[c][j] = fmaf(zf[j], U.x[c], zacc[c][j]);
}

// zacc scale exponent of zero group j (see unit_math): 2^(149 - 8 (j % 4)),
// byte 3 shifted down; times 2^-100 for the x prescale
MOE_DEV constexpr int zexp(int j) { return (j & 3) == 3 ? 49 : 49 - 8 * (j & 3); }

// The slice's 128 outputs of every column (without the per-CTA zoffset sum):
// exact integer digit sums -> one fp32 rounding, tile shift and 2^-E undone,
// plus the zero-point total of each output's group.  Column group m holds
// CPG columns: the accumulator columns n = 4 c' + digit of column 2m + c'
// (lane t = 2 c' + digit / 2).  ys[col * ystride + o].
template <int B, int NM, int CPG>
MOE_DEV void finish(const int (&D)[NM][8][4], const float (&zacc)[NM * CPG][8],
                    const int (&E)[NM * CPG], int lane, float* ys, int ystride) {
  constexpr int NC = NM * CPG;
  const int g = lane >> 2, t = lane & 3;
  constexpr int NG = B == 2 ? 8 : 2;  // zero groups per slice
  float zt[NC][NG];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int j = 0; j < NG; ++j) {  // rows are lanes: sum over the warp
      float z = zacc[c][j] * __uint_as_float(gemv::pow2_bits(zexp(j)));
#pragma unroll
      for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
      zt[c][j] = z;
    }
#pragma unroll
  for (int m = 0; m < NM; ++m) {
    // this lane's column of group m (CPG 1: lanes t >= 2 hold zero columns)
    const int cl = CPG == 2 ? (t >> 1) : 0;
    const int col = m * CPG + cl;
    const int Ec = (CPG == 2 && cl) ? E[m * CPG + 1 < NC ? m * CPG + 1 : 0] : E[m * CPG];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float sc = __uint_as_float(gemv::pow2_bits(-Ec - mt::tile_shift(B, i)));
      float z;
      if constexpr (CPG == 2) {
        const float za = B == 2 ? zt[m * 2][i] : zt[m * 2][i >> 2];
        const float zb = B == 2 ? zt[m * 2 + 1][i] : zt[m * 2 + 1][i >> 2];
        z = cl ? zb : za;
      } else {
        z = B == 2 ? zt[m][i] : zt[m][i >> 2];
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) {  // row g (c = 0) and g + 8
        // digits: even t holds accumulator columns (256^0, 256^1), odd t (256^2, 256^3)
        long long v = (t & 1) == 0
                          ? (long long)D[m][i][2 * c] + ((long long)D[m][i][2 * c + 1] << 8)
                          : ((long long)D[m][i][2 * c] << 16) +
                                ((long long)D[m][i][2 * c + 1] << 24);
        if (CPG == 1 && t >= 2) v = 0;
        v += __shfl_down_sync(0xffffffffu, v, 1);
        if ((t & 1) == 0 && (CPG == 2 || t == 0))
          ys[col * ystride + 16 * i + g + 8 * c] = fmaf(__ll2float_rn(v), sc, z);
      }
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
