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
// Right shifts as IMAD.HI: they issue on the FMA pipe, leaving the ALU pipe
// (rt 2 cycles / warp instruction, like the FMA pipe) to the code masks.
MOE_DEV uint32_t shr_fma(uint32_t v, int s) { return __umulhi(v, 1u << (32 - s)); }

MOE_DEV void fma_codes2(float (&acc)[16], float xs, uint32_t w) {
  const uint32_t wh = shr_fma(w, 16);
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
  const uint32_t wh = shr_fma(w, 16);
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
  // funnel shifts as (lo >> s) + hi * 2^(32-s), all on the FMA pipe
  const uint32_t v[3] = {w0, shr_fma(w0, 30) + w1 * 4u, shr_fma(w1, 28) + w2 * 16u};
  const uint32_t v3 = shr_fma(w2, 26);
  float m[32];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const uint32_t u = shr_fma(v[i], 12);
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

// ------------------------------------------------------------ async pipeline
MOE_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

MOE_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
MOE_DEV void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
MOE_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
MOE_DEV void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
MOE_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// one bulk global -> shared copy completing on `bar` (16-byte aligned, size % 16 == 0)
MOE_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// weight streams are read once per token: evict-first, so L2 keeps what a
// later kernel will read (prefetched weights, activations, split-K sums)
MOE_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
MOE_DEV void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                           uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// L2 prefetch of a byte range (16-byte aligned start and size)
MOE_DEV void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
MOE_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
MOE_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Accumulate the code part of one record (4 rows of one lane's chunk) from
// shared memory: acc_k += (x_r * s_r) * bits(code_{r,k} in place).
//   rec: the record in smem; wcb: chunks in this cb; x4: the quad's 4 x values
//   (prescaled by 2^100 for quant formats)
template <int BITS>
MOE_DEV void quad_codes(float (&acc)[Fmt<BITS>::WC], const uint8_t* rec, int wcb, int lane,
                        float4 x4, int g_log2, int sg_log2) {
  constexpr int NV = Fmt<BITS>::NV;
  constexpr int WC = Fmt<BITS>::WC;
  const uint4* cw = reinterpret_cast<const uint4*>(rec);
  uint4 r[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) r[v] = cw[v * wcb + lane];
  const uint32_t* w = reinterpret_cast<const uint32_t*>(&r[0]);
  const float xv[4] = {x4.x, x4.y, x4.z, x4.w};
  if constexpr (BITS <= 4) {
    const int outs = wcb * WC;
    const uint2 s4 = reinterpret_cast<const uint2*>(rec + 16 * NV * wcb + 4 * (outs >> g_log2))
        [(lane * WC) >> sg_log2];
    const float2 s01 = __half22float2(*reinterpret_cast<const __half2*>(&s4.x));
    const float2 s23 = __half22float2(*reinterpret_cast<const __half2*>(&s4.y));
    const float sv[4] = {s01.x, s01.y, s23.x, s23.y};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float xsv = xv[q] * sv[q];
      if constexpr (BITS == 2) fma_codes2(acc, xsv, w[q]);
      if constexpr (BITS == 4) fma_codes4(acc, xsv, w[q]);
      if constexpr (BITS == 3) fma_codes3(acc, xsv, w[3 * q], w[3 * q + 1], w[3 * q + 2]);
    }
  } else if constexpr (BITS == 16) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t* h = w + 4 * q;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&h[k]));
        ffma_pair(acc[2 * k], acc[2 * k + 1], xv[q], f.x, f.y);
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float* f = reinterpret_cast<const float*>(w + 4 * q);
      ffma_pair(acc[0], acc[1], xv[q], f[0], f[1]);
      ffma_pair(acc[2], acc[3], xv[q], f[2], f[3]);
    }
  }
}

// Zero-point terms of one quad: sum_r x_r * zhat(r, group) for the 4*ZPR
// (row, group) pairs of the record, spread over the warp's lanes.
//   mode 0 (32 % ZPR == 0): lane takes terms t = lane + 32 i, group t % ZPR,
//          so every lane keeps one group; mode 1: lane < ZPR takes its group
//   uniform runs: zhat*x = zc * xz[r] with xz = x * zscale(run of the row)
//   (the zoffset part is a per-CTA scalar added once); else the run is
//   looked up per term (quant.py:172-178: zhat = zc * zscale + zoffset).
struct ZeroCtx {
  const uint32_t* zeros;  // record's [ZPR] u32 (4 rows each)
  const float* xs;        // x slice (prescaled) at the quad's first row
  const float* xz;        // x * zscale at the quad's first row (uniform runs)
  const __half2* zmeta;
  int zpr, zpr_log2, mode, uniform, G, sg_log2, grow, gcb0;
};

MOE_DEV void quad_zero(float& zacc, const ZeroCtx& Z, int lane) {
  const int nterms = 4 * Z.zpr;
  if (Z.mode == 0) {
    for (int t = lane; t < nterms; t += 32) {
      const int j = t & (Z.zpr - 1), r = t >> Z.zpr_log2;
      const uint32_t zc = (Z.zeros[j] >> (8 * r)) & 0xffu;
      if (Z.uniform) {
        zacc = fmaf((float)zc, Z.xz[r], zacc);
      } else {
        const int run = ((Z.grow + r) * Z.G + Z.gcb0 + j) >> Z.sg_log2;
        const float2 zm = __half22float2(__ldg(Z.zmeta + run));
        zacc = fmaf(Z.xs[r], fmaf((float)zc, zm.x, zm.y), zacc);
      }
    }
  } else if (lane < Z.zpr) {
    const uint32_t z4 = Z.zeros[lane];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t zc = (z4 >> (8 * r)) & 0xffu;
      if (Z.uniform) {
        zacc = fmaf((float)zc, Z.xz[r], zacc);
      } else {
        const int run = ((Z.grow + r) * Z.G + Z.gcb0 + lane) >> Z.sg_log2;
        const float2 zm = __half22float2(__ldg(Z.zmeta + run));
        zacc = fmaf(Z.xs[r], fmaf((float)zc, zm.x, zm.y), zacc);
      }
    }
  }
}

// Fast zero-point path for the reference presets with full column blocks
// and uniform runs (2-bit g=16: ZPR=32; 3/4-bit g=64: ZPR=16 / 4): the
// lane -> (group, rows) split is a compile-time function of the lane.
//   zeros: the record's [ZPR] u32; xz: x * zscale for the quad's 4 rows
template <int BITS>
MOE_DEV void quad_zero_fast(float& zacc, const uint32_t* zeros, const float* xz, int lane) {
  if constexpr (BITS == 2) {  // lane = group, all 4 rows
    const uint32_t z4 = zeros[lane];
    const float4 x4 = *reinterpret_cast<const float4*>(xz);
    zacc = fmaf((float)(z4 & 0xffu), x4.x, zacc);
    zacc = fmaf((float)((z4 >> 8) & 0xffu), x4.y, zacc);
    zacc = fmaf((float)((z4 >> 16) & 0xffu), x4.z, zacc);
    zacc = fmaf((float)(z4 >> 24), x4.w, zacc);
  } else if constexpr (BITS == 3) {  // group lane & 15, rows (lane >> 4) and +2
    const uint32_t z4 = zeros[lane & 15];
    const int r = lane >> 4;
    zacc = fmaf((float)((z4 >> (8 * r)) & 0xffu), xz[r], zacc);
    zacc = fmaf((float)((z4 >> (8 * r + 16)) & 0xffu), xz[r + 2], zacc);
  } else {  // 4-bit: lanes < 16, group lane & 3, row lane >> 2
    if (lane < 16) {
      const uint32_t z4 = zeros[lane & 3];
      const int r = lane >> 2;
      zacc = fmaf((float)((z4 >> (8 * r)) & 0xffu), xz[r], zacc);
    }
  }
}

// lanes -> per-group totals for the fast path (then the lane's own group)
template <int BITS>
MOE_DEV float zero_total_fast(float zacc, int lane) {
  if constexpr (BITS == 2) return zacc;
  if constexpr (BITS == 3) {
    zacc += __shfl_xor_sync(0xffffffffu, zacc, 16);
    return __shfl_sync(0xffffffffu, zacc, lane >> 1);
  }
  zacc += __shfl_xor_sync(0xffffffffu, zacc, 4);
  zacc += __shfl_xor_sync(0xffffffffu, zacc, 8);
  zacc += __shfl_xor_sync(0xffffffffu, zacc, 16);
  return __shfl_sync(0xffffffffu, zacc, lane >> 3);
}

// final per-output value of one lane: exact power-of-two rescale of the
// masked-code accumulators plus the zero-point term
template <int BITS>
MOE_DEV void finish_lane(float (&y)[Fmt<BITS>::WC], const float (&acc)[Fmt<BITS>::WC], float ztot) {
  constexpr int WC = Fmt<BITS>::WC;
  if constexpr (BITS <= 4) {
    const float z = ztot * kZUnscale;
#pragma unroll
    for (int k = 0; k < WC; ++k)
      y[k] = fmaf(acc[k], __uint_as_float(pow2_bits(49 - posq<BITS>(k))), z);
  } else {
#pragma unroll
    for (int k = 0; k < WC; ++k) y[k] = acc[k];
  }
}

}  // namespace gemv
