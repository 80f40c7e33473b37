// Fused dequantize + GEMV core (CUDA cores, fp32 accumulate) for the tiled
// device layout of common.cuh.  Replaces the reference's
// ``x @ quant.dequantize(block)`` (quant.py:267-304 + model.py:223-226,290-300).
//
// Dequant without unpack arithmetic: a b-bit code c masked in place at bit p of
// a 32-bit word is, read as an IEEE float, exactly c * 2^p * 2^-149 (subnormal,
// or the first normal binade while p + b <= 24).  So per weight the kernel
// issues one LOP3 (mask) and half an FFMA2:
//     acc_k += (x_i * 2^100 * s) * bits(w & (mask << p_k))
// and rescales acc_k by 2^(49 - p_k) once at the end (exact power of two).
// The zero-point term  sum_i x_i * zhat(i, group)  is accumulated once per
// (row, group) and added to every output of the group.  With zhat =
// zcode*zscale + zoffset exactly as quant.py:172-178 (exact in fp32), the only
// deviation from the reference is fp32 summation order.
#pragma once
#include "common.cuh"

namespace gemv {

constexpr float kXScale = 0x1p100f;      // x prescale (keeps products normal)
constexpr float kZUnscale = 0x1p-100f;

// bit position of output k inside its (possibly shifted) code word
__host__ __device__ constexpr int pos2(int k) { return k < 12 ? 2 * k : 2 * k - 16; }
__host__ __device__ constexpr int pos4(int k) { return k < 6 ? 4 * k : 4 * k - 16; }
__host__ __device__ constexpr int pos3(int j) {
  return j >= 30 ? 3 * (j - 30) : ((j % 10) < 8 ? 3 * (j % 10) : 3 * (j % 10) - 12);
}
template <int BITS> __host__ __device__ constexpr int posq(int k) {
  return BITS == 2 ? pos2(k) : BITS == 3 ? pos3(k) : pos4(k);
}

MOE_DEV float fbits(uint32_t v) { return __uint_as_float(v); }
// exact 2^e for a normal exponent
__host__ __device__ constexpr uint32_t pow2_bits(int e) { return (uint32_t)(e + 127) << 23; }

MOE_DEV void ffma_pair(float& a0, float& a1, float x, float m0, float m1) {
  float2 r = __ffma2_rn(make_float2(x, x), make_float2(m0, m1), make_float2(a0, a1));
  a0 = r.x;
  a1 = r.y;
}

// 16 two-bit codes of one row-chunk word
MOE_DEV void fma_codes2(float (&acc)[16], float xs, uint32_t w) {
  const uint32_t wh = w >> 16;
  float m[16];
#pragma unroll
  for (int k = 0; k < 12; ++k) m[k] = fbits(w & (3u << (2 * k)));
#pragma unroll
  for (int k = 12; k < 16; ++k) m[k] = fbits(wh & (3u << (2 * k - 16)));
#pragma unroll
  for (int k = 0; k < 16; k += 2) ffma_pair(acc[k], acc[k + 1], xs, m[k], m[k + 1]);
}

// 8 four-bit codes
MOE_DEV void fma_codes4(float (&acc)[8], float xs, uint32_t w) {
  const uint32_t wh = w >> 16;
  float m[8];
#pragma unroll
  for (int k = 0; k < 6; ++k) m[k] = fbits(w & (15u << (4 * k)));
#pragma unroll
  for (int k = 6; k < 8; ++k) m[k] = fbits(wh & (15u << (4 * k - 16)));
#pragma unroll
  for (int k = 0; k < 8; k += 2) ffma_pair(acc[k], acc[k + 1], xs, m[k], m[k + 1]);
}

// 32 three-bit codes = 96 bits = 3 words of the reference LE bitstream.
// Funnel shifts realign codes 10..19 and 20..29 to 3k positions.
MOE_DEV void fma_codes3(float (&acc)[32], float xs, uint32_t w0, uint32_t w1, uint32_t w2) {
  const uint32_t v[3] = {w0, __funnelshift_r(w0, w1, 30), __funnelshift_r(w1, w2, 28)};
  const uint32_t v3 = w2 >> 26;
  float m[32];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const uint32_t u = v[i] >> 12;
#pragma unroll
    for (int k = 0; k < 8; ++k) m[10 * i + k] = fbits(v[i] & (7u << (3 * k)));
    m[10 * i + 8] = fbits(u & (7u << 12));
    m[10 * i + 9] = fbits(u & (7u << 15));
  }
  m[30] = fbits(v3 & 7u);
  m[31] = fbits(v3 & (7u << 3));
#pragma unroll
  for (int k = 0; k < 32; k += 2) ffma_pair(acc[k], acc[k + 1], xs, m[k], m[k + 1]);
}

template <int BITS, int U>
struct Batch {
  uint4 r[U][Fmt<BITS>::NV];
  uint32_t z[U];
  uint2 s[U];
};

// Where this thread's data lives for the current job.
struct Lane {
  const uint4* rec;       // already offset to (cb, lane): index(quad, v) = rec[(quad*NV + v)*wcb]
  const uint32_t* zeros;  // offset to group column: zeros[quad*G]
  const uint2* scales;    // offset to scale column: scales[quad*S]
  const __half2* zmeta;
  int wcb, G, S, grp, sg_log2;
};

template <int BITS, int U>
MOE_DEV void load_batch(Batch<BITS, U>& b, const Lane& L, int q, int qend) {
  constexpr int NV = Fmt<BITS>::NV;
  constexpr bool QUANT = BITS <= 4;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int qq = q + u;
    if (qq < qend) {
#pragma unroll
      for (int v = 0; v < NV; ++v) b.r[u][v] = ld_nc_v4(L.rec + (int64_t)(qq * NV + v) * L.wcb);
      if (QUANT) {
        b.z[u] = ld_nc_u32(L.zeros + (int64_t)qq * L.G);
        b.s[u] = ld_nc_v2(L.scales + (int64_t)qq * L.S);
      }
    }
  }
}

// Accumulate one batch.  xs: smem x slice (prescaled for quant), row0 = its first row.
template <int BITS, int U>
MOE_DEV void compute_batch(float (&acc)[Fmt<BITS>::WC], float& zacc, const Batch<BITS, U>& b,
                           const Lane& L, const float* xs, int row0, int q, int qend) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int qq = q + u;
    if (qq >= qend) break;
    const uint32_t* w = reinterpret_cast<const uint32_t*>(&b.r[u][0]);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int row = qq * 4 + r;
      const float x = xs[row - row0];
      if constexpr (BITS <= 4) {
        const uint32_t sh = (r & 1) ? (((r >> 1) ? b.s[u].y : b.s[u].x) >> 16)
                                    : (((r >> 1) ? b.s[u].y : b.s[u].x) & 0xffffu);
        const float xsv = x * h2f_bits(sh);
        const uint32_t zc = (b.z[u] >> (8 * r)) & 0xffu;
        const int run = (row * L.G + L.grp) >> L.sg_log2;
        const __half2 zm = __ldg(L.zmeta + run);
        const float zh = fmaf((float)zc, __low2float(zm), __high2float(zm));
        zacc = fmaf(x, zh, zacc);
        if constexpr (BITS == 2) fma_codes2(acc, xsv, w[r]);
        if constexpr (BITS == 4) fma_codes4(acc, xsv, w[r]);
        if constexpr (BITS == 3) fma_codes3(acc, xsv, w[3 * r], w[3 * r + 1], w[3 * r + 2]);
      } else if constexpr (BITS == 16) {
        const uint32_t* h = w + 4 * r;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&h[k]));
          ffma_pair(acc[2 * k], acc[2 * k + 1], x, f.x, f.y);
        }
      } else {
        const float* f = reinterpret_cast<const float*>(w + 4 * r);
        ffma_pair(acc[0], acc[1], x, f[0], f[1]);
        ffma_pair(acc[2], acc[3], x, f[2], f[3]);
      }
    }
  }
}

// Runs this thread's quads [qbeg, qend) and returns per-output sums (unscaled).
template <int BITS, int U>
MOE_DEV void run_lane(float (&y)[Fmt<BITS>::WC], const Lane& L, const float* xs, int row0, int qbeg,
                      int qend) {
  constexpr int WC = Fmt<BITS>::WC;
  float acc[WC];
#pragma unroll
  for (int k = 0; k < WC; ++k) acc[k] = 0.f;
  float zacc = 0.f;
  if (qbeg < qend) {
    Batch<BITS, U> cur, nxt;
    load_batch<BITS, U>(cur, L, qbeg, qend);
    for (int q = qbeg; q < qend; q += U) {
      if (q + U < qend) load_batch<BITS, U>(nxt, L, q + U, qend);
      compute_batch<BITS, U>(acc, zacc, cur, L, xs, row0, q, qend);
      cur = nxt;
    }
  }
  if constexpr (BITS <= 4) {
    const float z = zacc * kZUnscale;
#pragma unroll
    for (int k = 0; k < WC; ++k) y[k] = fmaf(acc[k], __uint_as_float(pow2_bits(49 - posq<BITS>(k))), z);
  } else {
#pragma unroll
    for (int k = 0; k < WC; ++k) y[k] = acc[k];
  }
}

}  // namespace gemv
