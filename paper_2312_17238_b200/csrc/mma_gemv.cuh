// Tensor-core dequant-GEMV core for the tile layout of mma_layout.cuh
// (2/3/4-bit reference presets).  Replaces the reference's
// ``x @ quant.dequantize(block)`` (quant.py:267-304, model.py:223-226,
// 290-300) like gemv.cuh, with the multiply-adds on mma.sync instead of FFMA2:
//
//   y_j = sum_i x_i (c_ij s_i,j/sg + zhat_i,j/g)
//       = sum_i c_ij b_i,jb  +  sum_i x_i zhat_i,j/g
//   A = c_ij as fp16 subnormals c * 2^(q-24) (one LOP3 per two codes),
//   B = b_i,jb = x_i * s_i,jb * 2^E split into three fp16 pieces (columns
//       n = 0, 1, 2 of the n8 tile; exact to 2^-25 of max |b| ~ 2^14),
//   D = fp32 accumulators in registers, rescaled by 2^(24-q-E) at the end.
// The zero-point term keeps the CUDA-core form (one FFMA per (row, group)).
// Every step is exact except the fp32 accumulation (tensor core) and the one
// fp32 rounding of x * s -- the same roundings class as the reference's fp32
// sgemv over the dequantized matrix.
#pragma once
#include "common.cuh"
#include "gemv.cuh"

namespace mg {

MOE_DEV void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                      uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

using gemv::shr_fma;

// the lane's 32 A-fragment registers of one k-step from its 2B code words
template <int B>
MOE_DEV void extract(const uint32_t (&w)[2 * B], uint32_t (&R)[32]) {
  if constexpr (B == 3) {
    uint32_t s[6];
#pragma unroll
    for (int v = 0; v < 6; ++v) {
      s[v] = shr_fma(w[v], 9);
      R[5 * v + 0] = w[v] & 0x00070007u;
      R[5 * v + 1] = w[v] & 0x00380038u;
      R[5 * v + 2] = w[v] & 0x01C001C0u;
      R[5 * v + 3] = s[v] & 0x00070007u;
      R[5 * v + 4] = s[v] & 0x00380038u;
    }
#pragma unroll
    for (int j = 0; j < 2; ++j)  // bit 15 / 31 of three words -> field [6, 9)
      R[30 + j] = (s[3 * j] & 0x00400040u) | (shr_fma(w[3 * j + 1], 8) & 0x00800080u) |
                  (shr_fma(w[3 * j + 2], 7) & 0x01000100u);
  } else if constexpr (B == 2) {
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const uint32_t s = shr_fma(w[v], 10);
#pragma unroll
      for (int f = 0; f < 5; ++f) R[8 * v + f] = w[v] & (0x00030003u << (2 * f));
#pragma unroll
      for (int f = 0; f < 3; ++f) R[8 * v + 5 + f] = s & (0x00030003u << (2 * f));
    }
  } else {
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const uint32_t s = shr_fma(w[v], 8);
      R[4 * v + 0] = w[v] & 0x000F000Fu;
      R[4 * v + 1] = w[v] & 0x00F000F0u;
      R[4 * v + 2] = s & 0x000F000Fu;
      R[4 * v + 3] = s & 0x00F000F0u;
    }
  }
}

// One k-step of one slice: 8 MMAs (the slice's 8 tiles) and the zero-point
// terms of its (row, group) pairs.
//   slice: the slice in smem (codes planes, then zero codes)
//   bf:    this lane's B fragment of (k-step, slice)
//   xz:    x * zscale * 2^100 of the k-step's 16 rows (16-byte aligned)
template <int B>
MOE_DEV void step(float (&D)[8][4], float (&zacc)[4], const uint8_t* slice, uint2 bf,
                  const float* xz, int lane) {
  const uint2* cp = reinterpret_cast<const uint2*>(slice);
  uint32_t w[2 * B];
#pragma unroll
  for (int pl = 0; pl < B; ++pl) {
    const uint2 v = cp[pl * 32 + lane];
    w[2 * pl] = v.x;
    w[2 * pl + 1] = v.y;
  }
  uint32_t R[32];
  extract<B>(w, R);
#pragma unroll
  for (int i = 0; i < 8; ++i)
    mma16816(D[i], R[mt::pair_reg(B, 2 * i, 0)], R[mt::pair_reg(B, 2 * i + 1, 0)],
             R[mt::pair_reg(B, 2 * i, 1)], R[mt::pair_reg(B, 2 * i + 1, 1)], bf.x, bf.y);
  const uint8_t* zc = slice + mt::code_bytes(B);
  if constexpr (B == 2) {  // lane: group lane & 7, rows 4 (lane >> 3) + j
    const uint32_t z4 = reinterpret_cast<const uint32_t*>(zc)[lane];
    const float4 x4 = reinterpret_cast<const float4*>(xz)[lane >> 3];
    zacc[0] = fmaf(gemv::fbits(z4 & 0xffu), x4.x, zacc[0]);
    zacc[1] = fmaf(gemv::fbits(z4 & 0xff00u), x4.y, zacc[1]);
    zacc[2] = fmaf(gemv::fbits(z4 & 0xff0000u), x4.z, zacc[2]);
    zacc[3] = fmaf(gemv::fbits(z4 & 0xff000000u), x4.w, zacc[3]);
  } else {  // g = 64: lane: group lane >> 4, row lane & 15
    zacc[0] = fmaf(gemv::fbits((uint32_t)zc[lane]), xz[lane & 15], zacc[0]);
  }
}

// The slice's 128 outputs (without the per-CTA zoffset sum): code part
// rescaled per (tile, row class), plus the zero-point total of each output's
// group.  Lanes t == 0 write ys[o] for their rows o = 16 i + g + 8 c.
//   E: the B operand's power-of-two prescale (x carries 2^100 already)
template <int B>
MOE_DEV void finish(const float (&D)[8][4], const float (&zacc)[4], int E, int lane, float* ys) {
  const int g = lane >> 2, t = lane & 3;
  // zero-point totals: zacc[j] sums zc * 2^(8j-149) * (x * 2^100 * zscale)
  float z = 0.f;
#pragma unroll
  for (int j = 0; j < (B == 2 ? 4 : 1); ++j)
    z = fmaf(zacc[j], __uint_as_float(gemv::pow2_bits(49 - 8 * j)), z);
  if constexpr (B == 2) {  // group = lane & 7: sum over lane >> 3
    z += __shfl_xor_sync(0xffffffffu, z, 8);
    z += __shfl_xor_sync(0xffffffffu, z, 16);
  } else {  // group = lane >> 4: sum over lane & 15
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float zt = __shfl_sync(0xffffffffu, z, B == 2 ? i : 16 * (i >> 2));
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      // pieces: t = 0 holds columns 0, 1; t = 1 holds column 2 (and a copy in 3)
      float v = t == 0 ? D[i][2 * c] + D[i][2 * c + 1] : (t == 1 ? D[i][2 * c] : 0.f);
      v += __shfl_down_sync(0xffffffffu, v, 1);
      const int q = mt::pair_q(B, 2 * i + c);
      const float sc = __uint_as_float(gemv::pow2_bits(-76 - q - E));
      if (t == 0) ys[mt::out_of(i, c, g)] = fmaf(v, sc, zt);
    }
  }
}

// split of b = x * s * 2^E into three fp16 pieces, written to the B table
MOE_DEV void put_pieces(__half* tab, int k, float b) {
  const __half h0 = __float2half_rn(b);
  const float r1 = b - __half2float(h0);
  const __half h1 = __float2half_rn(r1);
  const float r2 = r1 - __half2float(h1);
  tab[mt::btab_half(k, 0)] = h0;
  tab[mt::btab_half(k, 1)] = h1;
  tab[mt::btab_half(k, 2)] = __float2half_rn(r2);
}

}  // namespace mg
