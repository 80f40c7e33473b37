// Decode-path kernels of the B200 MoE offloading engine (sm_100a).
//
// Per token and layer (engine.cu enqueues them in this order):
//   layernorm(x -> xn, ln1) | gemv<attn bits>(Wq,Wk,Wv) | attention | gemv(Wo)
//   | tail (resid + LN2 + gate(l) + gate(l+lookahead) + top-k + device store)
//   | gemv<expert bits>(W1,W3 of the routed experts) | gemv(W2, SwiGLU prologue)
//   | combine (h + w0*y0 + w1*y1, reference order)
// then layernorm(ln_f) | gemv<f16>(lm_head) | logits (+ argmax on device).
// All reductions are in a fixed order, so results are run-to-run deterministic.
#include <atomic>
#include <cstdio>

#include "kernels.cuh"
#include "gemv.cuh"
#include "mma_gemv.cuh"

// profiling hooks in constant memory: every kernel tests them after
// griddepcontrol.wait, where a global-memory pointer load would cost an L2
// round trip on the critical path (a constant-cache hit costs a few cycles)
__constant__ TimelineSlot* g_timeline = nullptr;
__constant__ int g_timeline_n = 0;  // span slots; phase marks follow
__constant__ unsigned long long* g_cta_trace = nullptr;  // GEMV microbench: [cta][4]

namespace {

MOE_DEV unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// per-CTA timeline marks (thread 0 of the CTA)
MOE_DEV void tl_begin(int site) {
  TimelineSlot* t = g_timeline;
  if (t && site >= 0 && threadIdx.x == 0) atomicMin(&t[site].start, globaltimer());
}
// intra-kernel phase marks (block 0, thread 0): slot site*8 + phase of the
// mark table that follows the span table (profiling)
MOE_DEV void tl_mark(int site, int phase) {
  TimelineSlot* t = g_timeline;
  if (t && site >= 0 && threadIdx.x == 0 && blockIdx.x == 0)
    reinterpret_cast<unsigned long long*>(t + g_timeline_n)[site * 8 + phase] = globaltimer();
}
MOE_DEV void cta_mark(int slot) {
  unsigned long long* t = g_cta_trace;
  if (t && threadIdx.x == 0) {
    if (slot == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      t[blockIdx.x * 4 + 3] = smid;
    }
    t[blockIdx.x * 4 + slot] = globaltimer();
  }
}
MOE_DEV void tl_end(int site) {
  TimelineSlot* t = g_timeline;
  if (t && site >= 0 && threadIdx.x == 0) atomicMax(&t[site].end, globaltimer());
}

MOE_DEV float sigmoid_ref(float x) {  // model.py:229-235 branch-stable logistic
  if (x >= 0.f) return __fdiv_rn(1.f, __fadd_rn(1.f, expf(-x)));
  const float ex = expf(x);
  return __fdiv_rn(ex, __fadd_rn(1.f, ex));
}

// ------------------------------------------------------------------ GEMV
// One launch computes up to MOE_GEMV_MAXJOBS independent x@W products (e.g.
// W1 and W3 of both routed experts).  CTA = one (job, column block, split):
// a contiguous byte range of records, streamed through a ring of shared-memory
// stages by one producer thread with cp.async.bulk + mbarriers, consumed by 8
// warps (one quad per warp per stage).  Bytes in flight are bounded by the
// ring (80 KB per CTA, 2 CTAs per SM), not by registers.
// Expert matrices (rel_slot >= 0) live in pool buffers named by the route the
// tail kernel wrote; the producer waits for the buffer's copy generation
// (copy engine -> cuStreamWriteValue32) before streaming it.  Dense weights
// are prefetched before griddepcontrol.wait, overlapping the previous kernel
// (programmatic dependent launch).

MOE_DEV bool wait_flag(const uint32_t* f, uint32_t gen, int* err, unsigned long long wait_ns) {
  if ((int)(ld_acquire_u32(f) - gen) >= 0) return true;
  const unsigned long long t0 = globaltimer();
  while ((int)(ld_acquire_u32(f) - gen) < 0) {
    __nanosleep(256);
    if (globaltimer() - t0 > wait_ns) {
      if ((atomicOr(err, MOE_ERRF_TIMEOUT) & MOE_ERRF_TIMEOUT) == 0) {
        err[2] = (int)gen;  // diagnostics: generation waited for, flag value seen
        err[3] = (int)ld_acquire_u32(f);
        err[4] = (int)(reinterpret_cast<uintptr_t>(f) & 0x7fffffff);
      }
      return false;
    }
  }
  return true;
}

// sum over the GEMV's consumer warps (named barrier 1, fixed order); `red`
// needs 9 floats and is free again when this returns
MOE_DEV float cons_sum(float v, float* red, int nthr) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = nthr >> 5;
  v = warp_sum(v);
  if (lane == 0) red[w] = v;
  asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
  float t = 0.f;
  for (int i = 0; i < nw; ++i) t += red[i];
  asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
  return t;
}

// fixed-point image of one partial (0 and an error flag when out of range)
MOE_DEV unsigned long long fx_bits(float a, int* err) {
  const float q = a * MOE_FX_SCALE;
  if (!(fabsf(q) < 0x1p62f)) {
    if (err) atomicOr(err, MOE_ERRF_NONFINITE_GATE);
    return 0ull;
  }
  return (unsigned long long)__float2ll_rn(q);
}

// consumer side: fixed-point sum -> fp32 (one rounding); the consumer resets
// the sums (fx_clear) after all its loads are issued
MOE_DEV float fx_val(unsigned long long v) {
  // one rounding of the exact integer to fp32, then an exact power-of-two scale
  return __ll2float_rn((long long)v) * (float)MOE_FX_UNSCALE;
}

template <int BITS>
__global__ void __launch_bounds__(MOE_GEMV_THREADS, MOE_GEMV_MINB)
    k_gemv(const __grid_constant__ GLaunch P, int xs_cap, int zs_cap, int xin_cap, int nst,
           int stage_bytes) {
  constexpr int WC = Fmt<BITS>::WC;
  constexpr bool QUANT = BITS <= 4;
  constexpr int W = MOE_GEMV_WARPS, QPW = gemv_qpw(BITS), QS = gemv_qs(BITS);
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 16;
  float* misc = reinterpret_cast<float*>(smem + 256);  // [16]: zo partials, flags
  uint64_t* zbar = reinterpret_cast<uint64_t*>(smem + 384);  // zero-point slice landed
  float* xs = reinterpret_cast<float*>(smem + 512);
  float* xz = xs + xs_cap;  // x * zscale per row (uniform zero-point runs)
  uint64_t* xbar = reinterpret_cast<uint64_t*>(smem + 392);  // x rows landed
  __half2* zsm = reinterpret_cast<__half2*>(xz + xs_cap);  // the CTA's zmeta slice [zs_cap]
  const size_t xin_off = 512 + (((size_t)xs_cap * 8 + (size_t)zs_cap * 4 + 15) & ~(size_t)15);
  uint8_t* xin = smem + xin_off;  // the CTA's raw x rows (bulk copied) [xin_cap bytes]
  uint8_t* ring = smem + ((xin_off + (size_t)xin_cap + 127) & ~(size_t)127);

  int ji = 0, cnt_base = 0;
  for (int i = 1; i < P.nj; ++i)
    if ((int)blockIdx.x >= P.j[i].blk0) ji = i;
  for (int i = 0; i < ji; ++i) cnt_base += P.j[i].M.ncb;
  const GJob& J = P.j[ji];
  const int local = blockIdx.x - J.blk0;
  const int cb = local / J.S, s = local % J.S;
  MatDev M = J.M;
  // storage units: quads of 4 rows; a cb is 32 chunks (the tensor-core layout
  // of mma_layout.cuh runs in k_mgemv)
  const int qs = s * J.QPS, qe = min(M.nqp, qs + J.QPS);  // storage quads (pads are zero)
  const int wcb = min(32, M.nchunks - cb * 32);
  const int rb = rec_bytes(BITS, wcb, M.g_log2, M.sg_log2);
  const int QSr = QS;  // quads per pipeline stage
  const int nit = (max(qe - qs, 0) + QSr - 1) / QSr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qv = min(qe, M.nquads);  // real quads of this split
  const int row0 = qs * 4, nrows = max(qv - qs, 0) * 4;
  const int nout = wcb * WC;  // outputs of this cb
  const size_t obase = (size_t)cb * 32 * WC;
  const int gcb0 = QUANT ? (int)(obase >> M.g_log2) : 0;  // first zero group of the cb
  const bool uni = QUANT && M.runs_uniform;
  // uniform runs: the zero-point runs of the CTA's rows are one contiguous
  // zmeta slice [z0, z1], streamed to smem by the producer ahead of the
  // records (16-byte aligned bulk copy; `zlead` entries of alignment slack)
  const bool zstage = uni && nrows > 0 && zs_cap > 0;
  const int z0 = zstage ? (int)(((int64_t)row0 * M.G + gcb0) >> M.sg_log2) : 0;
  const int z1 = zstage ? (int)(((int64_t)(row0 + nrows - 1) * M.G + gcb0) >> M.sg_log2) : 0;
  // the CTA's x rows (outputs of the previous kernel, L2-resident) come through
  // the producer's bulk-copy queue ahead of the weight stream: consumer loads
  // issued next to a saturating weight stream wait behind it for microseconds
  const bool swiglu = J.xmode == X_SWIGLU;
  constexpr int xes = 4;  // bytes per x element
  const int xparts = J.xS > 1 ? J.xS : 1;  // producer partials per input array
  const bool xcomb = J.xmode == X_COMBINE;
  const bool xstage = !xcomb && xin_cap > 0 && nrows > 0 &&
                      (swiglu ? 2 : 1) * xparts * nrows * xes <= xin_cap;

  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) {
      gemv::mbar_init(full + i, 1);
      gemv::mbar_init(empty + i, W);
    }
    gemv::mbar_init(zbar, 1);
    gemv::mbar_init(xbar, 1);
    gemv::mbar_fence_init();
  }
  __syncthreads();
  gemv::pdl_trigger();

  if (warp == W) {  // ---------------------------------------------- producer
    if (J.rel_slot >= 0) {
      gemv::pdl_wait();  // the route is written by the previous kernel
      // expert parallel: another rank owns this expert -> the whole cluster
      // (same job) skips, before any cluster barrier
      if (P.route->buf[J.rel_slot] < 0) return;
    }
    // x rows: one bulk copy per input array (after the previous kernel completed)
    auto issue_x = [&]() {
      if (J.rel_slot < 0) gemv::pdl_wait();  // x: previous kernel's output
      if (!xstage) return;
      const uint32_t bytes = (uint32_t)(nrows * xes);
      gemv::mbar_arrive_tx(xbar, (swiglu ? 2u : 1u) * (uint32_t)xparts * bytes);
      const uint8_t* a = reinterpret_cast<const uint8_t*>(swiglu ? J.up1 : J.x);
      const size_t pstride = (size_t)J.xstride * xes;  // between producer partials
      for (int p = 0; p < xparts; ++p)
        gemv::bulk_g2s(xin + (size_t)p * bytes, a + p * pstride + (size_t)row0 * xes, bytes, xbar);
      if (swiglu)
        for (int p = 0; p < xparts; ++p)
          gemv::bulk_g2s(xin + (size_t)(xparts + p) * bytes,
                         reinterpret_cast<const uint8_t*>(J.up3) + p * pstride +
                             (size_t)row0 * xes,
                         bytes, xbar);
    };
    if (lane == 0) {
      if (J.rel_slot >= 0) {
        issue_x();
        const int buf = P.route->buf[J.rel_slot];
        // the tail saw the buffer's copy already published: no flag round trip
        if (!P.route->ready[J.rel_slot])
          wait_flag(P.flags + buf, P.route->gen[J.rel_slot], P.err, P.wait_ns);
        const uint8_t* b = P.pool + (long long)buf * P.slot_stride;
        M.base = b + reinterpret_cast<size_t>(M.base);
        M.zmeta = reinterpret_cast<const __half2*>(b + reinterpret_cast<size_t>(M.zmeta));
      }
      if (zstage) {
        const uintptr_t za = reinterpret_cast<uintptr_t>(M.zmeta + z0);
        const uint32_t lead = (uint32_t)(za & 15u);
        const uint32_t bytes = ((uint32_t)(z1 - z0 + 1) * 4u + lead + 15u) & ~15u;
        gemv::mbar_arrive_tx(zbar, bytes);
        gemv::bulk_g2s(zsm, reinterpret_cast<const void*>(za - lead), bytes, zbar);
      }
      const uint8_t* src = M.base + cb_offset(M, cb) + (int64_t)qs * rb;
      const uint64_t pol = gemv::policy_evict_first();
      int st = 0;
      uint32_t ph = 0;
      for (int it = 0; it < nit; ++it) {
        // dense weights: the ring is prefetched before the previous kernel ends
        if (it == nst && J.rel_slot < 0) issue_x();
        if (it >= nst) gemv::mbar_wait(empty + st, ph ^ 1);
        const int nq = min(QSr, qe - (qs + it * QSr));
        const uint32_t bytes = (uint32_t)(nq * rb);
        gemv::mbar_arrive_tx(full + st, bytes);
        gemv::bulk_g2s_hint(ring + (size_t)st * stage_bytes, src + (int64_t)it * QSr * rb, bytes,
                            full + st, pol);
        if (++st == nst) {
          st = 0;
          ph ^= 1;
        }
      }
      if (nit <= nst && J.rel_slot < 0) issue_x();
    }
    __syncwarp();
    return;
  }

  // ------------------------------------------------------------ consumers
  const int nthr = W * 32;
  gemv::pdl_wait();
  tl_begin(P.site);
  tl_mark(P.site, 5);  // block 0 released (profiling: its start vs the earliest CTA's)
  cta_mark(0);
  if (P.zero) {  // reset sums an earlier kernel consumed (e.g. the previous layer's up)
    const int per = (P.zero_n + gridDim.x - 1) / gridDim.x;
    const int z0 = blockIdx.x * per, z1 = min(P.zero_n, z0 + per);
    for (int i = z0 + threadIdx.x; i < z1; i += nthr) P.zero[i] = 0ull;
  }
  // expert jobs: the route load is issued with the x loads (independent)
  const int ebuf = J.rel_slot >= 0 ? P.route->buf[J.rel_slot] : 0;
  const float xscale = QUANT ? gemv::kXScale : 1.f;
  if (J.rel_slot >= 0) {
    if (ebuf < 0) {  // expert parallel: not ours; contribute zeros to the exchange
      float* zdst = J.reduce == 2 ? nullptr : J.reduce ? (s == 0 ? J.out : nullptr)
                                                      : J.part + (size_t)s * M.N;
      if (zdst)
        for (int t = threadIdx.x; t < nout; t += nthr) zdst[obase + t] = 0.f;
      cta_mark(2);
      tl_end(P.site);
      return;
    }
  }
  if (xcomb) {  // fused combine + LayerNorm of the previous layer's output
    float* xf = reinterpret_cast<float*>(xin);  // the full residual [K]
    const int K = M.K;
    const float w0 = P.route->w[0], w1 = J.ctop > 1 ? P.route->w[1] : 0.f;
    float s = 0.f;
    for (int i0 = threadIdx.x; i0 < K; i0 += 8 * nthr) {  // 24 loads in flight
      float hv[8];
      unsigned long long q0[8], q1[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * nthr;
        hv[u] = i < K ? __ldcg(J.x + i) : 0.f;
        q0[u] = i < K ? __ldcg(J.cacc + i) : 0ull;
        q1[u] = (i < K && J.ctop > 1) ? __ldcg(J.cacc + K + i) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * nthr;
        if (i < K) {
          float o = __fadd_rn(hv[u], __fmul_rn(w0, fx_val(q0[u])));  // model.py:251-254
          if (J.ctop > 1) o = __fadd_rn(o, __fmul_rn(w1, fx_val(q1[u])));
          xf[i] = o;
          s += o;
          if (blockIdx.x == 0) J.xout[i] = o;
        }
      }
    }
    tl_mark(P.site, 6);  // residual formed (profiling; the epilogue reuses the slot)
    // LayerNorm statistics over the consumer warps (named barrier), the
    // reference's rounding structure (model.py:186-189)
    const float mu = __fdiv_rn(cons_sum(s, misc, nthr), (float)K);
    float q = 0.f;
    for (int i = threadIdx.x; i < K; i += nthr) {
      const float t = __fsub_rn(xf[i], mu);
      q = fmaf(t, t, q);
    }
    const float var = __fdiv_rn(cons_sum(q, misc, nthr), (float)K);
    const float den = sqrtf(__fadd_rn(var, 1e-5f));
    tl_mark(P.site, 7);  // LN statistics
    for (int i = threadIdx.x; i < nrows; i += nthr) {
      const int r = row0 + i;
      const float v =
          __fadd_rn(__fmul_rn(__fdiv_rn(__fsub_rn(xf[r], mu), den), __ldg(J.lng + r)),
                    __ldg(J.lnb + r));
      xs[i] = v * xscale;
    }
  }
  if (xstage) {  // x rows from the producer's bulk copy
    gemv::mbar_wait(xbar, 0);
    const float* xf = reinterpret_cast<const float*>(xin);
    for (int i = threadIdx.x; i < nrows; i += nthr) {
      float a = 0.f, b = 0.f;  // fp32 producer partials, summed in split order
      for (int p = 0; p < xparts; ++p) a += xf[p * nrows + i];
      if (swiglu)
        for (int p = 0; p < xparts; ++p) b += xf[(xparts + p) * nrows + i];
      float xv = a;
      if (swiglu)  // SwiGLU of the up projections (model.py:223-226)
        xv = __fmul_rn(__fmul_rn(a, sigmoid_ref(a)), b);
      xs[i] = xv * xscale;
    }
  }
  // x (or the SwiGLU of the up projections) in batches of 4 rows per thread:
  // every load of a batch is issued before any use
  for (int i0 = 0; !xstage && !xcomb && i0 < nrows; i0 += 4 * nthr) {
    float va[4], vb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * nthr + threadIdx.x;
      const int r = row0 + i;
      const bool in = i < nrows;
      if (J.xS > 1) {  // unreduced producer partials: sum them in split order
        // (up to 8 splits per round, every load of the round in flight)
        float a = 0.f, b = 0.f;
        if (in) {
          const float* pa = J.xmode == X_PLAIN ? J.x : J.up1;
          const bool two = J.xmode != X_PLAIN;
          for (int s0 = 0; s0 < J.xS; s0 += 8) {
            float ta[8], tb[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const bool ok = s0 + k < J.xS;
              const size_t o = (size_t)(s0 + k) * J.xstride + r;
              ta[k] = ok ? __ldcg(pa + o) : 0.f;
              tb[k] = ok && two ? __ldcg(J.up3 + o) : 0.f;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (s0 + k < J.xS) {
                a += ta[k];
                b += tb[k];
              }
          }
        }
        va[u] = a;
        vb[u] = b;
      } else if (J.xmode == X_PLAIN) {
        va[u] = in ? __ldcg(J.x + r) : 0.f;
        vb[u] = 0.f;
      } else {
        va[u] = in ? __ldcg(J.up1 + r) : 0.f;
        vb[u] = in ? __ldcg(J.up3 + r) : 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * nthr + threadIdx.x;
      if (i >= nrows) continue;
      float xv = va[u];
      if (J.xmode != X_PLAIN)  // SwiGLU of the up projections (model.py:223-226)
        xv = __fmul_rn(__fmul_rn(va[u], sigmoid_ref(va[u])), vb[u]);
      xs[i] = xv * xscale;
    }
  }
  tl_mark(P.site, 0);  // x slice in smem
  if (J.rel_slot >= 0) {
    if (QUANT && (!uni || zs_cap == 0)) {  // zmeta is read from global
      M.zmeta = reinterpret_cast<const __half2*>(P.pool + (long long)ebuf * P.slot_stride +
                                                 reinterpret_cast<size_t>(M.zmeta));
      if (threadIdx.x == 0 && !P.route->ready[J.rel_slot])
        wait_flag(P.flags + ebuf, P.route->gen[J.rel_slot], P.err, P.wait_ns);
      asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
    }
  }
  float zo_part = 0.f;
  if (uni && nrows > 0) {  // x * zscale per row and the CTA's sum of x * zoffset
    int zlead = 0;
    if (zstage) {
      gemv::mbar_wait(zbar, 0);
      // expert slots are 256-byte aligned: the offset has the address's alignment
      const uintptr_t za = J.rel_slot >= 0
          ? (uintptr_t)(reinterpret_cast<size_t>(M.zmeta) + (size_t)z0 * 4)
          : reinterpret_cast<uintptr_t>(M.zmeta + z0);
      zlead = (int)(za & 15u) >> 2;
    }
    for (int i0 = 0; i0 < nrows; i0 += 4 * nthr)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * nthr + threadIdx.x;
        if (i >= nrows) continue;
        const int run = (int)(((int64_t)(row0 + i) * M.G + gcb0) >> M.sg_log2);
        const float2 zm =
            __half22float2(zstage ? zsm[zlead + run - z0] : __ldg(M.zmeta + run));
        const float xv = xs[i];
        xz[i] = xv * zm.x;
        zo_part = fmaf(xv, zm.y, zo_part);
      }
  }
  tl_mark(P.site, 1);  // zero-point slice landed, x * zscale done
  if (QUANT && M.runs_uniform) {
    zo_part = warp_sum(zo_part);
    if (lane == 0) misc[warp] = zo_part;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
  float zo_sum = 0.f;
  if (QUANT && M.runs_uniform)
#pragma unroll
    for (int w = 0; w < W; ++w) zo_sum += misc[w];

  tl_mark(P.site, 2);  // prologue done (x slice, zero-point rows)
  float acc[WC];
#pragma unroll
  for (int k = 0; k < WC; ++k) acc[k] = 0.f;
  float zacc = 0.f;
  gemv::ZeroCtx Z;
  if (QUANT) {
    Z.zpr = (wcb * WC) >> M.g_log2;
    Z.zpr_log2 = __ffs(Z.zpr) - 1;
    Z.mode = (Z.zpr & (Z.zpr - 1)) == 0 ? 0 : 1;
    Z.uniform = M.runs_uniform;
    Z.G = M.G;
    Z.sg_log2 = M.sg_log2;
    Z.gcb0 = gcb0;
    Z.zmeta = M.zmeta;
  }
  const bool active = lane < wcb;
  // fast path: reference preset grouping, full column block, uniform runs
  const bool fast = QUANT && wcb == 32 && M.runs_uniform &&
                    M.g_log2 == (BITS == 2 ? 4 : 6);
  float ztot = 0.f;
  if (fast || !QUANT) {
    int st = 0;
    uint32_t ph = 0;
    for (int it = 0; it < nit; ++it) {
      gemv::mbar_wait(full + st, ph);
#pragma unroll
      for (int u = 0; u < QPW; ++u) {
        const int q = qs + it * QS + u * W + warp;
        if (q < qv) {
          const uint8_t* rec = ring + (size_t)st * stage_bytes + (size_t)(u * W + warp) * rb;
          const int lr = (q - qs) * 4;
          const float4 x4 = *reinterpret_cast<const float4*>(xs + lr);
          if (QUANT) {
            gemv::quad_codes<BITS>(acc, rec, 32, lane, x4, M.g_log2, M.sg_log2);
            gemv::quad_zero_fast<BITS>(
                zacc, reinterpret_cast<const uint32_t*>(rec + 16 * Fmt<BITS>::NV * 32), xz + lr,
                lane);
          } else if (active) {
            gemv::quad_codes<BITS>(acc, rec, wcb, lane, x4, 0, 0);
          }
        }
      }
      __syncwarp();
      if (lane == 0) gemv::mbar_arrive(empty + st);
      if (++st == nst) {
        st = 0;
        ph ^= 1;
      }
    }
    if (QUANT) ztot = gemv::zero_total_fast<BITS>(zacc, lane);
  } else {
    int st = 0;
    uint32_t ph = 0;
    for (int it = 0; it < nit; ++it) {
      gemv::mbar_wait(full + st, ph);
      for (int u = 0; u < QPW; ++u) {
        const int q = qs + it * QS + u * W + warp;
        if (q < qv) {
          const uint8_t* rec = ring + (size_t)st * stage_bytes + (size_t)(u * W + warp) * rb;
          const int lr = (q - qs) * 4;
          const float4 x4 = *reinterpret_cast<const float4*>(xs + lr);
          if (active) gemv::quad_codes<BITS>(acc, rec, wcb, lane, x4, M.g_log2, M.sg_log2);
          Z.zeros = reinterpret_cast<const uint32_t*>(rec + 16 * Fmt<BITS>::NV * wcb);
          Z.xs = xs + lr;
          Z.xz = xz + lr;
          Z.grow = q * 4;
          gemv::quad_zero(zacc, Z, lane);
        }
      }
      __syncwarp();
      if (lane == 0) gemv::mbar_arrive(empty + st);
      if (++st == nst) {
        st = 0;
        ph ^= 1;
      }
    }
    if (Z.mode == 0)
      for (int o = Z.zpr; o < 32; o <<= 1) zacc += __shfl_xor_sync(0xffffffffu, zacc, o);
    ztot = __shfl_sync(0xffffffffu, zacc, (lane * WC) >> M.g_log2);
  }
  tl_mark(P.site, 3);  // streaming loop done
  cta_mark(1);
  float y[WC];
  gemv::finish_lane<BITS>(y, acc, ztot);
  // cross-warp reduction through the (now idle) ring, fixed order
  float* red = reinterpret_cast<float*>(ring);
  float* ysum = red + W * 32 * (WC + 1);  // the CTA's partial outputs
  asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
  if (!xcomb) tl_mark(P.site, 6);  // every consumer warp left the loop
#pragma unroll
  for (int k = 0; k < WC; ++k) red[(warp * 32 + lane) * (WC + 1) + k] = y[k];
  asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
  if (!xcomb) tl_mark(P.site, 7);  // per-warp results in smem
  const float zo_out = zo_sum * gemv::kZUnscale;
  const int SC = J.S;
  float* dst = (SC == 1 && J.reduce) ? J.out : J.part + (size_t)s * M.N;
  // the CTA's outputs leave with one bulk (TMA) copy: a plain store of the
  // split-K partials, or a bulk fixed-point add (cp.reduce.async.bulk .add.u64)
  const bool bulk_out = J.reduce != 1;
  unsigned long long* fxs = reinterpret_cast<unsigned long long*>(ysum);
  for (int t = threadIdx.x; t < 32 * WC; t += nthr) {
    const int l = t / WC, k = t % WC;
    if (l < wcb) {
      float a = 0.f;
#pragma unroll
      for (int w = 0; w < W; ++w) a += red[(w * 32 + l) * (WC + 1) + k];
      a += zo_out;
      if (bulk_out && J.reduce == 2)
        fxs[t] = fx_bits(a, P.err);
      else if (bulk_out)
        ysum[t] = a;
      else
        dst[obase + t] = a;
    }
  }
  if (bulk_out) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // smem writes -> TMA
    asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
    if (threadIdx.x == 0) {
      const size_t o = obase;
      if (J.reduce == 2)
        asm volatile(
            "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], %2;" ::"l"(
                J.acc + o),
            "r"(gemv::smem_u32(fxs)), "r"((uint32_t)(nout * 8))
            : "memory");
      else
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + o),
                     "r"(gemv::smem_u32(ysum)), "r"((uint32_t)(nout * 4))
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;" ::: "memory");
    }
  }
  tl_mark(P.site, 4);  // cross-warp (+ cluster) reduction, partial written
  if (SC == 1 || J.reduce != 1) {  // done, or the consumer sums the partials
    cta_mark(2);
    tl_end(P.site);
    return;
  }
  // split-K: the last CTA of this column block to finish sums the S partials
  // in order.
  // One thread publishes the CTA's partial (barrier, then a gpu-scope fence
  // and the arrival count) and, in the last CTA, acquires the others'.
  asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
  int* flag = reinterpret_cast<int*>(misc + 8);
  if (threadIdx.x == 0) {
    __threadfence();
    const int old = atomicAdd(P.cnt + cnt_base + cb, 1);
    __threadfence();
    *flag = old == J.S - 1;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
  if (!*flag) {
    cta_mark(2);
    tl_end(P.site);
    return;
  }
  // 4 outputs x 8 splits per thread in flight, then the in-order sums
  const int no = nout;
  const float* pbase = J.part + obase;
  for (int t0 = threadIdx.x; t0 < no; t0 += 4 * nthr) {
    float a[4] = {0.f, 0.f, 0.f, 0.f};
    for (int s0 = 0; s0 < SC; s0 += 8) {
      float v[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int t = t0 + u * nthr;
          v[u][k] = (t < no && s0 + k < SC) ? __ldcg(pbase + (size_t)(s0 + k) * M.N + t) : 0.f;
        }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (s0 + k < SC) a[u] += v[u][k];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (t0 + u * nthr < no) J.out[obase + t0 + u * nthr] = a[u];
  }
  if (threadIdx.x == 0) P.cnt[cnt_base + cb] = 0;
  cta_mark(2);
    tl_end(P.site);
}


// ------------------------------------------------------------------ wait
// Blocks the compute stream until every expert buffer of this position's route
// has landed (copy engine -> cuStreamWriteValue32 of the buffer generation).
// One thread per routed expert; hits pass straight through.
__global__ void k_wait_ready(const RouteRec* route, int n, const uint32_t* flags, int* err,
                             unsigned long long wait_ns) {
  const int j = threadIdx.x;
  if (j >= n) return;
  const int buf = route->buf[j];
  if (buf < 0) return;
  const uint32_t gen = route->gen[j];
  const uint32_t* f = flags + buf;
  if ((int)(ld_acquire_u32(f) - gen) >= 0) return;
  const unsigned long long t0 = globaltimer();
  while ((int)(ld_acquire_u32(f) - gen) < 0) {
    __nanosleep(200);
    if (globaltimer() - t0 > wait_ns) {
      atomicOr(err, MOE_ERRF_TIMEOUT);
      return;
    }
  }
}

// Event-timing pass only: one thread idles the compute stream for `ns` so the
// host has enqueued "start event, kernel, end event" before the stream reaches
// the start event.  Without it the GPU drains the stream between host launches
// and every event-timed span includes the host's launch gap.
__global__ void k_hold(unsigned long long ns) {
  const unsigned long long t0 = globaltimer();
  while (globaltimer() - t0 < ns) __nanosleep(1000);
}

// Block-wide fp32 sum in a fixed order (per-thread, warp tree, warp 0 over
// the warp sums): deterministic.  `red` needs 33 floats.
MOE_DEV float block_sum_f(float v, float* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    float t = lane < nw ? red[lane] : 0.f;
    t = warp_sum(t);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  const float r = red[32];
  __syncthreads();
  return r;
}

// LayerNorm with the reference's rounding structure (model.py:186-189):
// population mean / variance, then ((x - mu) / sqrt(var + eps)) * gamma + beta
// with separately rounded float32 ops.  x, g, b may live in shared memory.
// The statistics are reduced over exactly 256 lanes (thread t sums x[t +
// 256k] in k order, butterfly warp sums, then the 8 warp sums in order)
// whatever the block size, so every LN site -- the 512/1024-thread kernels and
// the QKV GEMV's fused combine + LN1 on its 8 consumer warps -- rounds alike.
MOE_DEV float ln_sum256(float v, float* red) {  // blockDim >= 256, all threads call
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0 && w < 8) red[w] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < 8; ++i) t += red[i];
  __syncthreads();
  return t;
}
// LN statistics (mu, sqrt(var + eps)) in that rounding structure
MOE_DEV float2 layernorm_stats(const float* x, int d, float* red) {
  const bool lane256 = threadIdx.x < 256;
  float s = 0.f;
  if (lane256)
    for (int i = threadIdx.x; i < d; i += 256) s += x[i];
  const float mu = __fdiv_rn(ln_sum256(s, red), (float)d);
  float q = 0.f;
  if (lane256)
    for (int i = threadIdx.x; i < d; i += 256) {
      const float t = __fsub_rn(x[i], mu);
      q = fmaf(t, t, q);
    }
  const float var = __fdiv_rn(ln_sum256(q, red), (float)d);
  return make_float2(mu, sqrtf(__fadd_rn(var, 1e-5f)));
}
MOE_DEV float layernorm_elem(float x, float2 st, float g, float b) {
  return __fadd_rn(__fmul_rn(__fdiv_rn(__fsub_rn(x, st.x), st.y), g), b);
}
MOE_DEV void layernorm_block(const float* x, const float* g, const float* b, float* y, float* ysh,
                             int d, float* red) {
  const float2 st = layernorm_stats(x, d, red);
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float v = layernorm_elem(x[i], st, g[i], b[i]);
    if (y) y[i] = v;
    if (ysh) ysh[i] = v;
  }
}

// ------------------------------------------------------------------ embed
__global__ void k_embed(EmbedParams P) {
  __shared__ float red[33];
  extern __shared__ float xsh[];  // x [d], then LN gamma / beta [d] each
  float* gs = xsh + P.d;
  float* bs = gs + P.d;
  gemv::pdl_trigger();
  if (P.xn)
    for (int i = threadIdx.x; i < P.d; i += blockDim.x) {
      gs[i] = __ldg(P.ln_g + i);
      bs[i] = __ldg(P.ln_b + i);
    }
  gemv::pdl_wait();
  tl_begin(P.site);
  const int tok = P.ds ? P.ds->tok : P.tok;
  const int pos = P.ds ? P.ds->pos : P.pos;
  const int step = P.xn ? blockDim.x : gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.d; i += step) {
    float a, b;
    if (P.half) {
      a = __half2float(reinterpret_cast<const __half*>(P.wte)[(size_t)tok * P.d + i]);
      b = __half2float(reinterpret_cast<const __half*>(P.wpe)[(size_t)pos * P.d + i]);
    } else {
      a = reinterpret_cast<const float*>(P.wte)[(size_t)tok * P.d + i];
      b = reinterpret_cast<const float*>(P.wpe)[(size_t)pos * P.d + i];
    }
    const float v = __fadd_rn(a, b);  // model.py:319
    P.x[i] = v;
    if (P.xn) xsh[i] = v;
  }
  if (P.xn) {  // fused LN1 of layer 0
    __syncthreads();
    layernorm_block(xsh, gs, bs, P.xn, nullptr, P.d, red);
  }
  tl_end(P.site);
}

__global__ void __launch_bounds__(1024) k_layernorm(const float* x, const float* g, const float* b,
                                                    float* y, int d) {
  __shared__ float red[33];
  gemv::pdl_trigger();
  gemv::pdl_wait();
  layernorm_block(x + (size_t)blockIdx.x * d, g, b, y + (size_t)blockIdx.x * d, nullptr, d, red);
}

// ------------------------------------------------------------------ attention
// One CTA per head (model.py:290-299): reduce q/k/v partials, append k/v to
// the fp32 KV cache, scores / sqrt(hd), softmax, ctx = alpha @ V.
__global__ void __launch_bounds__(256) k_attention(AttnParams P) {
  extern __shared__ float sh[];
  const int hd = P.hd, h = blockIdx.x, d = P.d;
  float* q = sh;
  float* sc = sh + hd;
  __shared__ float red[32];
  __shared__ float bval;
  gemv::pdl_trigger();
  gemv::pdl_wait();
  const int pos = P.ds ? P.ds->pos : P.pos;
  const size_t kvrow = (size_t)pos * P.H * hd + (size_t)h * hd;
  for (int i = threadIdx.x; i < hd; i += blockDim.x) {
    const int o = h * hd + i;
    float a = 0.f, bk = 0.f, bv = 0.f;
    if (P.acc) {
      a = fx_val(__ldcg(P.acc + o));
      bk = fx_val(__ldcg(P.acc + d + o));
      bv = fx_val(__ldcg(P.acc + 2 * d + o));
      P.acc[o] = P.acc[d + o] = P.acc[2 * d + o] = 0ull;
    } else {
      for (int s = 0; s < P.S; ++s) {
        a += __ldcg(P.qkv_part + ((size_t)0 * P.S + s) * d + o);
        bk += __ldcg(P.qkv_part + ((size_t)1 * P.S + s) * d + o);
        bv += __ldcg(P.qkv_part + ((size_t)2 * P.S + s) * d + o);
      }
    }
    q[i] = a;
    P.kc[kvrow + i] = bk;
    P.vc[kvrow + i] = bv;
  }
  __syncthreads();
  const int T = pos + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const float rs = sqrtf((float)hd);
  for (int t = warp; t < T; t += nw) {
    const float* kr = P.kc + (size_t)t * P.H * hd + (size_t)h * hd;
    float a = 0.f;
    for (int i = lane; i < hd; i += 32) a = fmaf(q[i], __ldcg(kr + i), a);
    a = warp_sum(a);
    if (lane == 0) sc[t] = __fdiv_rn(a, rs);
  }
  __syncthreads();
  float mx = -INFINITY;
  for (int t = threadIdx.x; t < T; t += blockDim.x) mx = fmaxf(mx, sc[t]);
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = red[0];
    for (int i = 1; i < nw; ++i) m = fmaxf(m, red[i]);
    bval = m;
  }
  __syncthreads();
  mx = bval;
  float su = 0.f;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const float e = expf(__fsub_rn(sc[t], mx));
    sc[t] = e;
    su += e;
  }
  su = warp_sum(su);
  __syncthreads();
  if (lane == 0) red[warp] = su;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = 0.f;
    for (int i = 0; i < nw; ++i) m += red[i];
    bval = m;
  }
  __syncthreads();
  su = bval;
  for (int t = threadIdx.x; t < T; t += blockDim.x) sc[t] = __fdiv_rn(sc[t], su);
  __syncthreads();
  for (int i = threadIdx.x; i < hd; i += blockDim.x) {
    float a = 0.f;
    for (int t = 0; t < T; ++t)
      a = fmaf(sc[t], __ldcg(P.vc + (size_t)t * P.H * hd + (size_t)h * hd + i), a);
    P.ctx[h * hd + i] = a;
  }
}

// Scores, softmax and alpha @ V of one head over positions 0..pos for a
// 256-thread CTA (model.py:294-299): q and the current position's k / v rows
// in shared memory, earlier rows from the KV cache (kc / vc point at this
// head's columns, row t at + t * rstride).  Scores use 4 threads per position
// (a quarter of the K row each, all loads in flight, quad shuffle reduce),
// then softmax, then alpha @ V with each head dimension split over two
// partial sums (even / odd positions).  Writes head dims [c0, c0 + nd) to
// out[0 .. nd).  Shared by k_attention128 and the Wo GEMV's fused attention
// prologue (X_ATTN), so every decode / prefill path rounds alike.
// sc: >= pos + 1 floats, hb: 2 * nd floats, red: 33 floats (shared).
__device__ __noinline__ void attend_head(const float* q, const float* kcur, const float* vcur, const float* kc,
                         const float* vc, size_t rstride, int pos, int HD, int c0, int nd,
                         float* sc, float* hb, float* red, float* out) {
  const int tid = threadIdx.x, T = pos + 1;
  const float rs = sqrtf((float)HD);
  {
    const int g = tid & 3, nf = HD / 16;  // float4s per quarter row
    const float4* q4 = reinterpret_cast<const float4*>(q) + g * nf;
    // warp-uniform trip count: every lane reaches the quad shuffles
    const int step = (int)blockDim.x >> 2, tw = (tid & ~31) >> 2;
    for (int t0 = tw; t0 < T; t0 += step) {
      const int t = t0 + ((tid & 31) >> 2);
      const bool live = t < T;
      const bool cur = t == pos;  // the current row lives in shared memory
      const float4* kr = reinterpret_cast<const float4*>(kc + (size_t)(live && !cur ? t : 0) *
                                                              rstride) + g * nf;
      const float4* ks = reinterpret_cast<const float4*>(kcur) + g * nf;
      float a0 = 0.f, a1 = 0.f;
      for (int c = 0; c < nf; c += 8) {
        float4 kv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) kv[u] = cur ? ks[c + u] : __ldcg(kr + c + u);
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
          const float4 x0 = q4[c + u], x1 = q4[c + u + 1];
          a0 = fmaf(x0.x, kv[u].x, fmaf(x0.y, kv[u].y, fmaf(x0.z, kv[u].z, fmaf(x0.w, kv[u].w, a0))));
          a1 = fmaf(x1.x, kv[u + 1].x,
                    fmaf(x1.y, kv[u + 1].y, fmaf(x1.z, kv[u + 1].z, fmaf(x1.w, kv[u + 1].w, a1))));
        }
      }
      float a = a0 + a1;
      a += __shfl_xor_sync(0xffffffffu, a, 1);
      a += __shfl_xor_sync(0xffffffffu, a, 2);
      if (g == 0 && live) sc[t] = __fdiv_rn(a, rs);
    }
  }
  __syncthreads();
  float mx = -INFINITY;
  for (int t = tid; t < T; t += blockDim.x) mx = fmaxf(mx, sc[t]);
  mx = warp_max(mx);
  if ((tid & 31) == 0) red[tid >> 5] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float su = 0.f;
  for (int t = tid; t < T; t += blockDim.x) {
    const float e = expf(__fsub_rn(sc[t], mx));
    sc[t] = e;
    su += e;
  }
  su = block_sum_f(su, red);
  for (int t = tid; t < T; t += blockDim.x) sc[t] = __fdiv_rn(sc[t], su);
  __syncthreads();
  // item (half, j): dim c0 + j summed over positions half, half + 2, ...
  for (int w = tid; w < 2 * nd; w += blockDim.x) {
    const int half = w / nd, j = w % nd, i = c0 + j;
    const float* vcol = vc + i;
    const float vp = vcur[i];
    auto ld = [&](int t) { return t == pos ? vp : __ldcg(vcol + (size_t)t * rstride); };
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    int t = half;
    // (unrolled so the loads of several groups are in flight; the FMA order,
    // hence the rounding, is the loop's)
#pragma unroll 4
    for (; t + 6 < T; t += 8) {
      const float v0 = ld(t), v1 = ld(t + 2), v2 = ld(t + 4), v3 = ld(t + 6);
      a0 = fmaf(sc[t], v0, a0);
      a1 = fmaf(sc[t + 2], v1, a1);
      a2 = fmaf(sc[t + 4], v2, a2);
      a3 = fmaf(sc[t + 6], v3, a3);
    }
#pragma unroll 4
    for (; t < T; t += 2) a0 = fmaf(sc[t], ld(t), a0);
    hb[half * nd + j] = (a0 + a1) + (a2 + a3);
  }
  __syncthreads();
  for (int j = tid; j < nd; j += blockDim.x) out[j] = hb[j] + hb[nd + j];
}

// pull a head's K/V cache rows of positions < pos into L2 (decode: they were
// evicted by the weight stream) -- issued before griddepcontrol.wait
MOE_DEV void prefetch_kv(const float* kc, const float* vc, size_t rstride, int pos, int HD) {
  const int lines = HD * 4 / 128;  // 128-byte lines per row
  for (int i = threadIdx.x; i < 2 * pos * lines; i += blockDim.x) {
    const int t = i / (2 * lines), r = i % (2 * lines);
    const float* base = (r < lines ? kc : vc) + (size_t)t * rstride;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(base + (r % lines) * 32));
  }
}

// Fast path for head_dim % 128 == 0: one CTA of 256 threads per head.  The
// current k/v row is appended to the cache, then attend_head.
__global__ void __launch_bounds__(256) k_attention128(AttnParams P) {
  // q [HD], k / v of this position [HD] each, scores [T_max], ctx halves [2][HD]
  extern __shared__ float asm_[];
  __shared__ float red[33];
  const int HD = P.hd, h = blockIdx.x, d = P.d;
  const int tid = threadIdx.x;
  float* q = asm_;
  float* kcur = q + HD;
  float* vcur = kcur + HD;
  float* sc = vcur + HD;
  float* half2buf = sc + P.T_max;
  gemv::pdl_trigger();
  const size_t rstride = (size_t)P.H * HD;
  if (P.ds)
    prefetch_kv(P.kc + (size_t)h * HD, P.vc + (size_t)h * HD, rstride, P.ds->pos, HD);
  gemv::pdl_wait();
  tl_begin(P.site);
  const int pos = P.ds ? P.ds->pos : P.pos + (int)blockIdx.y;
  const float* qg = P.qkv_part + (size_t)h * HD;
  float* krow = P.kc + (size_t)pos * rstride + (size_t)h * HD;
  float* vrow = P.vc + (size_t)pos * rstride + (size_t)h * HD;
  float* ctx = P.ctx + (size_t)blockIdx.y * d;
  // KV append (model.py:293, KVCache.append)
  const size_t sstride = (size_t)P.S * d;
  if (P.qbuf) {  // batched prefill: K/V rows appended by k_kv_append, q converted there
    const float* qs = P.qbuf + (size_t)blockIdx.y * d + (size_t)h * HD;
    for (int i = tid; i < HD; i += blockDim.x) {
      q[i] = qs[i];
      kcur[i] = krow[i];
      vcur[i] = vrow[i];
    }
  } else if (P.acc) {  // fixed-point sums of the QKV GEMV: read, then reset for the next layer
    unsigned long long* qa = P.acc + (size_t)h * HD;
    for (int i = tid; i < HD; i += blockDim.x) {
      const unsigned long long a = __ldcg(qa + i), bk = __ldcg(qa + d + i),
                               bv = __ldcg(qa + 2 * d + i);
      q[i] = fx_val(a);
      kcur[i] = krow[i] = fx_val(bk);
      vcur[i] = vrow[i] = fx_val(bv);
      qa[i] = qa[d + i] = qa[2 * d + i] = 0ull;
    }
  } else {  // split-K partials [3][S][d], summed in split order
    for (int i = tid; i < HD; i += blockDim.x) {
      float a = 0.f, bk = 0.f, bv = 0.f;
#pragma unroll 4
      for (int s = 0; s < P.S; ++s) {
        a += __ldcg(qg + (size_t)s * d + i);
        bk += __ldcg(qg + sstride + (size_t)s * d + i);
        bv += __ldcg(qg + 2 * sstride + (size_t)s * d + i);
      }
      q[i] = a;
      kcur[i] = krow[i] = bk;
      vcur[i] = vrow[i] = bv;
    }
  }
  __syncthreads();
  tl_mark(P.site, 0);
  attend_head(q, kcur, vcur, P.kc + (size_t)h * HD, P.vc + (size_t)h * HD, rstride, pos, HD, 0,
              HD, sc, half2buf, red, ctx + (size_t)h * HD);
  tl_end(P.site);
}

// the tensor-core dequant-GEMV (uses attend_head for the fused decode attention)
#include "mgemv_kernel.cuh"

// batched prefill: the Q/K/V fixed-point sums of `rows` positions -> q rows
// (qbuf) and the K/V cache rows of positions pos .. pos + rows - 1, sums reset
// (the same fx_val conversion k_attention128 applies in decode)
__global__ void __launch_bounds__(256) k_kv_append(AttnParams P) {
  const int r = blockIdx.y, d = P.d;
  unsigned long long* a = P.acc + (size_t)r * 3 * d;
  float* kr = P.kc + (size_t)(P.pos + r) * d;
  float* vr = P.vc + (size_t)(P.pos + r) * d;
  float* qr = const_cast<float*>(P.qbuf) + (size_t)r * d;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x) {
    qr[i] = fx_val(__ldcg(a + i));
    kr[i] = fx_val(__ldcg(a + d + i));
    vr[i] = fx_val(__ldcg(a + 2 * d + i));
    a[i] = a[d + i] = a[2 * d + i] = 0ull;
  }
}

// ------------------------------------------------------------------ tail
// resid = x + ctx@Wo; h = LN2(resid) (model.py:300-301); gate logits for this
// layer and the guessed layer on the same h (model.py:210, engine.py:60-68);
// stable top-k + softmax over the selected logits (model.py:211-215); trace
// record (engine.py:122-128); then the device store: acquire each selected
// expert in descending-weight order and speculative_load the guesses
// (engine.py:222-231).
// tail: hs = x + Wo output (fp32 partial or fixed-point sums, reset after
// the loads), V values per thread with every load in flight first
template <int V, bool FX, class Mid>
MOE_DEV void residual_in(const float* part, const float* xin, unsigned long long* acc, float* hs,
                         int tid, Mid&& mid, int d) {
  const int nt = (int)blockDim.x;
  float xa[V], pa[V];
  unsigned long long qa[FX ? V : 1];
#pragma unroll
  for (int u = 0; u < V; ++u) {
    const int i = tid + u * nt;
    xa[u] = i < d ? __ldcg(xin + i) : 0.f;
    if constexpr (FX)
      qa[u] = i < d ? __ldcg(acc + i) : 0ull;
    else
      pa[u] = i < d ? __ldcg(part + i) : 0.f;
  }
  mid();  // more independent loads (store state, flags) while these are in flight
#pragma unroll
  for (int u = 0; u < V; ++u) {
    const int i = tid + u * nt;
    if constexpr (FX) pa[u] = fx_val(qa[u]);
    if (i < d) hs[i] = __fadd_rn(xa[u], pa[u]);
  }
  if constexpr (FX)  // reset the fixed-point sums for the next Wo GEMV
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const int i = tid + u * nt;
      if (i < d) acc[i] = 0ull;
    }
}

// rows beyond 8 per thread (d > 8 * blockDim): further passes of 8
template <bool FX, class Mid>
MOE_DEV void residual_all(const TailParams& P, const float* xin, unsigned long long* acc,
                          float* hs, int tid, Mid&& mid) {
  const int d = P.d, span = 8 * (int)blockDim.x;
  auto none = []() {};
  for (int b = 0; b < d; b += span) {
    if (b == 0)
      residual_in<8, FX>(P.part, xin, acc, hs, tid, mid, min(span, d));
    else
      residual_in<8, FX>(P.part + b, xin + b, FX ? acc + b : acc, hs + b, tid, none,
                         min(span, d - b));
  }
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) k_tail(TailParams P) {
  extern __shared__ __align__(128) unsigned char tsm[];
  const int d = P.d, E = P.E;
  const bool guess = P.gate_g != nullptr;
  const bool hg = P.gh_l != nullptr && (!guess || P.gh_g != nullptr);
  // smem: hs[d] | g2[d] | b2[d] | gates (fp16, 1 or 2) | gpart[2*1024] dbl | store
  float* hs = reinterpret_cast<float*>(tsm);
  float* g2s = hs + d;
  float* b2s = g2s + d;
  __half* gls = reinterpret_cast<__half*>(b2s + d);
  __half* ggs = gls + (size_t)d * E;
  double* gpart = reinterpret_cast<double*>(
      tsm + ((3 * (size_t)d * 4 + (hg ? (guess ? 2 : 1) * (size_t)d * E * 2 : 0) + 15) & ~15));
  int* sst = reinterpret_cast<int*>(gpart + 2 * blockDim.x);
  uint32_t* fls = reinterpret_cast<uint32_t*>(sst + store::stage_ints(P.st) + 4);  // [nbuf]
  __shared__ float lg[64];
  __shared__ __align__(8) uint64_t wbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  gemv::pdl_trigger();
  // immutable weights (LN2 affine, gate matrices) stream into shared memory
  // with one bulk copy each while the Wo GEMV finishes
  if (tid == 0) {
    gemv::mbar_init(&wbar, 1);
    gemv::mbar_fence_init();
    const uint32_t vb = (uint32_t)d * 4, gb = (uint32_t)d * E * 2;
    gemv::mbar_arrive_tx(&wbar, 2 * vb + (hg ? (guess ? 2 : 1) * gb : 0));
    gemv::bulk_g2s(g2s, P.g2, vb, &wbar);
    gemv::bulk_g2s(b2s, P.b2, vb, &wbar);
    if (hg) {
      gemv::bulk_g2s(gls, P.gh_l, gb, &wbar);
      if (guess) gemv::bulk_g2s(ggs, P.gh_g, gb, &wbar);
    }
  } else if (!hg) {  // fp32 gates: pull them toward L2 instead
    for (int i = tid * 32; i < d * E; i += blockDim.x * 32) {
      asm volatile("prefetch.global.L2 [%0];" ::"l"(P.gate_l + i));
      if (guess) asm volatile("prefetch.global.L2 [%0];" ::"l"(P.gate_g + i));
    }
  }
  gemv::pdl_wait();
  tl_begin(P.site);
  if (P.zero)  // Q/K/V sums read by the Wo GEMV's fused attention: reset for the next layer
    for (int i = tid; i < P.zero_n; i += blockDim.x) P.zero[i] = 0ull;
  // batched prefill (mode 1): CTA r handles position P.pos + r
  const int row = P.mode == 1 ? (int)blockIdx.x : 0;
  const int pos = P.ds ? P.ds->pos : P.pos + row;
  const float* xin = P.x + (size_t)row * d;
  unsigned long long* accr = P.acc ? P.acc + (size_t)row * d : nullptr;
  float* hout = P.h + (size_t)row * d;
  RouteRec* route = P.route + row;
  const size_t slot = (size_t)pos * P.n_layers + P.layer;
  float* th = P.trace_hidden ? P.trace_hidden + slot * d : nullptr;
  StoreDev S = P.st;
  // the store state and the copy-flag snapshot (decode) load while the
  // residual's loads are in flight: one L2 round trip instead of three
  auto stage = [&]() {
    if (P.mode != 0) return;
    const int n4 = P.st.state_ints >> 2;
    if (n4 <= (int)blockDim.x && P.st.nbuf <= (int)blockDim.x) {
      // one element per thread: every load is issued before any shared store
      const int4* src = reinterpret_cast<const int4*>(P.st.state_base);
      int4 v = make_int4(0, 0, 0, 0);
      int vt = 0;
      uint32_t fv = 0;
      const int ti = 4 * n4 + tid;
      if (tid < n4) v = __ldcg(src + tid);
      if (ti < P.st.state_ints) vt = __ldcg(P.st.state_base + ti);
      // snapshot of the buffers' published copy generations: a routed buffer
      // whose copy had landed is marked ready, so the GEMVs skip the flag wait
      if (P.st.flags && tid < P.st.nbuf)
        fv = ld_acquire_u32(const_cast<const uint32_t*>(P.st.flags) + tid);
      if (tid < n4) reinterpret_cast<int4*>(sst)[tid] = v;
      if (ti < P.st.state_ints) sst[ti] = vt;
      if (P.st.flags && tid < P.st.nbuf) fls[tid] = fv;
      S = store::stage_view(P.st, sst);
    } else {
      S = store::stage_in(P.st, sst);
      if (P.st.flags)
        for (int i = tid; i < P.st.nbuf; i += blockDim.x)
          fls[i] = ld_acquire_u32(const_cast<const uint32_t*>(P.st.flags) + i);
    }
  };
  // residual: all loads first, then the stores (no load waits behind a store)
  if (accr) {
    if (d <= 4 * (int)blockDim.x)
      residual_in<4, true>(P.part, xin, accr, hs, tid, stage, d);
    else
      residual_all<true>(P, xin, accr, hs, tid, stage);
  } else {
    residual_all<false>(P, xin, accr, hs, tid, stage);
  }
  tl_mark(P.site, 0);
  gemv::mbar_wait(&wbar, 0);
  __syncthreads();
  tl_mark(P.site, 1);
  const float2 lst = layernorm_stats(hs, d, reinterpret_cast<float*>(gpart));
  tl_mark(P.site, 2);
  // gate logits of this layer and the guessed layer on the same h (model.py:210,
  // engine.py:60-68)
  const int nt = (blockDim.x / E) * E;
  const bool gate8 = hg && E == 8;  // fast path: one 16-byte fp16 gate row per load
  int bad = 0;
  if (gate8) {
    // LN2 (model.py:300-301) fused with the gate partials: thread t normalizes
    // rows t, t + nthreads, ... and accumulates them for all 8 experts (and the
    // guessed layer's 8) in that order -- fp32 partials, then double sums in a
    // fixed order
    float pa[8], pg[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) pa[e] = pg[e] = 0.f;
    for (int r = tid; r < d; r += blockDim.x) {
      const float hv = layernorm_elem(hs[r], lst, g2s[r], b2s[r]);
      hout[r] = hv;
      if (th) th[r] = hv;
      if (!isfinite(hv)) bad = 1;
      if (guess) hs[r] = hv;  // re-read by this thread for the guessed gate
      const uint4 gl4 = *reinterpret_cast<const uint4*>(gls + (size_t)r * 8);
      const __half2* gl2 = reinterpret_cast<const __half2*>(&gl4);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 g = __half22float2(gl2[e]);
        pa[2 * e] = fmaf(hv, g.x, pa[2 * e]);
        pa[2 * e + 1] = fmaf(hv, g.y, pa[2 * e + 1]);
      }
    }
    if (guess)  // same rows, same order (second pass keeps registers under 64)
      for (int r = tid; r < d; r += blockDim.x) {
        const float hv = hs[r];
        const uint4 gg4 = *reinterpret_cast<const uint4*>(ggs + (size_t)r * 8);
        const __half2* gg2 = reinterpret_cast<const __half2*>(&gg4);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 g = __half22float2(gg2[e]);
          pg[2 * e] = fmaf(hv, g.x, pg[2 * e]);
          pg[2 * e + 1] = fmaf(hv, g.y, pg[2 * e + 1]);
        }
      }
    // fp32 butterfly sums of the 8 (16) partials, interleaved so the
    // shuffles of different logits overlap; warp sums go to double below
#pragma unroll
    for (int o = 16; o; o >>= 1) {
#pragma unroll
      for (int e = 0; e < 8; ++e) pa[e] += __shfl_xor_sync(0xffffffffu, pa[e], o);
      if (guess)
#pragma unroll
        for (int e = 0; e < 8; ++e) pg[e] += __shfl_xor_sync(0xffffffffu, pg[e], o);
    }
    if (lane == 0) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        gpart[warp * 16 + e] = (double)pa[e];
        gpart[warp * 16 + 8 + e] = (double)pg[e];
      }
    }
    bad = __syncthreads_or(bad);
  } else {
    for (int i = tid; i < d; i += blockDim.x) {
      const float v = layernorm_elem(hs[i], lst, g2s[i], b2s[i]);
      hout[i] = v;
      if (th) th[i] = v;
      if (!isfinite(v)) bad = 1;
      hs[i] = v;
    }
    bad = __syncthreads_or(bad);
    if (tid < nt) {
      const int e = tid % E, rstep = nt / E;
      // per-thread fp32 partials over 2 interleaved accumulators, combined in
      // double across threads (fixed order below)
      float a0 = 0.f, a1 = 0.f, g0 = 0.f, g1 = 0.f;
      int r = tid / E;
      if (hg) {
        for (; r + rstep < d; r += 2 * rstep) {
          const float h0 = hs[r], h1 = hs[r + rstep];
          a0 = fmaf(h0, __half2float(gls[r * E + e]), a0);
          a1 = fmaf(h1, __half2float(gls[(r + rstep) * E + e]), a1);
          if (guess) {
            g0 = fmaf(h0, __half2float(ggs[r * E + e]), g0);
            g1 = fmaf(h1, __half2float(ggs[(r + rstep) * E + e]), g1);
          }
        }
        if (r < d) {
          a0 = fmaf(hs[r], __half2float(gls[r * E + e]), a0);
          if (guess) g0 = fmaf(hs[r], __half2float(ggs[r * E + e]), g0);
        }
      } else {
        for (; r < d; r += rstep) {
          a0 = fmaf(hs[r], __ldg(P.gate_l + r * E + e), a0);
          if (guess) g0 = fmaf(hs[r], __ldg(P.gate_g + r * E + e), g0);
        }
      }
      gpart[tid] = (double)a0 + (double)a1;
      gpart[blockDim.x + tid] = (double)g0 + (double)g1;
    }
    __syncthreads();
  }
  tl_mark(P.site, 3);
  const int nlog = guess ? 2 * E : E;
  if (gate8) {  // logit e: the warps' sums in warp order
    if (tid < nlog) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += gpart[w * 16 + tid];
      lg[tid] = (float)t;
    }
  } else if (warp < nlog) {  // warp w reduces logit w in a fixed order
    const int e = warp % E;
    const double* gp = gpart + (warp >= E ? blockDim.x : 0);
    double t = 0.0;
    for (int i = e + E * lane; i < nt; i += 32 * E) t += gp[i];
    t = warp_sum_d(t);
    if (lane == 0) lg[warp] = (float)t;
  }
  __syncthreads();
  tl_mark(P.site, 4);
  // top-k of this layer's logits and top-m of the guessed layer's, on warp 0:
  // lane e holds logit e; each round is a warp argmax with ties -> lower index
  // (np.argsort(-logits, kind="stable"), model.py:192-195, engine.py:60-68)
  __shared__ int sel_sh[MOE_MAX_TOPK], gsel_sh[16];
  if (warp < 2) {  // warp 0: this layer's top-k, warp 1: the guessed layer's top-m
    const int k = P.top_k, mg = (guess && P.m > 0) ? P.m : 0;
    {
      const int pass = warp;
      const float* lv = pass == 0 ? lg : lg + E;
      const int rounds = pass == 0 ? k : mg;
      bool taken = false;
      for (int j = 0; j < rounds; ++j) {
        float v = (lane < E && !taken) ? lv[lane] : -INFINITY;
        int idx = (lane < E && !taken) ? lane : 0x7fffffff;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, v, o);
          const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
          if (ov > v || (ov == v && oi < idx)) {
            v = ov;
            idx = oi;
          }
        }
        if (lane == idx) taken = true;
        if (lane == 0) (pass == 0 ? sel_sh : gsel_sh)[j] = idx;
      }
    }
  }
  __syncthreads();
  tl_mark(P.site, 5);
  // warp 1: routing weights (softmax over the top-k logits, sequential sum in
  // selection order), trace record and the route's expert/weight fields;
  // meanwhile thread 0 runs the store bookkeeping (buffers of the route)
  __shared__ int rbuf[MOE_MAX_TOPK];
  __shared__ uint32_t rgen[MOE_MAX_TOPK];
  if (warp == 1) {
    const int k = P.top_k;
    const float l0 = lg[sel_sh[0]];
    const float ez = lane < k ? expf(__fsub_rn(lg[sel_sh[lane]], l0)) : 0.f;
    float sum = 0.f;
    for (int t = 0; t < k; ++t) sum = __fadd_rn(sum, __shfl_sync(0xffffffffu, ez, t));
    const float wj = lane < k ? __fdiv_rn(ez, sum) : 0.f;
    const int ej = lane < k ? sel_sh[lane] : -1;
    if (lane < MOE_MAX_TOPK) {
      route->e[lane] = ej;
      route->w[lane] = wj;
    }
    TraceRecDev* tr = P.trace + slot;
    if (lane < 8) {
      tr->experts[lane] = ej;
      tr->weights[lane] = wj;
    }
    if (lane == 0) {
      tr->pos = pos;
      tr->layer = P.layer;
    }
  }
  if (tid == 0) {
    const int k = P.top_k;
    tl_mark(P.site + 4, 0);  // profiling: bookkeeping start (exchange slot unused on 1 GPU)
    for (int j = 0; j < MOE_MAX_TOPK; ++j) {
      rbuf[j] = -1;
      rgen[j] = 0u;
    }
    if (bad) {
      atomicOr(P.st.err, MOE_ERRF_NONFINITE_GATE);
      // first failing position (+1): the smallest over the CTAs of a batched prefill
      int cur = *(volatile int*)(P.st.err + 6);
      while (cur == 0 || cur > pos + 1) {
        const int prev = atomicCAS(P.st.err + 6, cur, pos + 1);
        if (prev == cur) break;
        cur = prev;
      }
    } else if (P.mode == 0) {
      const int m = (guess && P.m > 0) ? P.m : 0;
      const int msite = P.site + 4;  // profiling marks in the (unused) exchange slot
      store::resolve_token(S, P.layer, sel_sh, k, gsel_sh, m, m ? P.guess_layer : -1, pos, rbuf,
                           rgen, [msite](int i) { tl_mark(msite, i); });
    }
#pragma unroll
    for (int j = 0; j < MOE_MAX_TOPK; ++j) {
      const int b = rbuf[j];
      route->buf[j] = b;
      route->gen[j] = rgen[j];
      route->ready[j] = (P.mode == 0 && P.st.flags && b >= 0 && j < k)
                              ? (int)((int)(fls[b] - rgen[j]) >= 0) : 0;
    }
    tl_mark(P.site + 4, 7);  // route written
  }
  tl_mark(P.site, 6);
  if (P.mode == 0) {
    __syncthreads();
    store::stage_out(P.st, sst);
  }
  tl_mark(P.site, 7);
  tl_end(P.site);
}

// prefill: each distinct expert of the layer acquired once, first-use order
// over (position, descending weight), no speculation (engine.py:233-240).
__global__ void k_prefill_bk(PrefillBKParams P) {
  gemv::pdl_wait();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  StoreDev S = P.st;
  RouteRec* R = P.route;
  // a position's gate input was not finite: the reference raises in gate()
  // before any acquire of this layer (model.py:198-205, engine.py:233-240)
  if (ld_acquire_u32(reinterpret_cast<const uint32_t*>(S.err)) & MOE_ERRF_NONFINITE_GATE) {
    for (int p = 0; p < P.n; ++p)
      for (int j = 0; j < P.top_k; ++j) R[p].buf[j] = -1;
    return;
  }
  store::resolve_prefill(
      S, P.layer, P.n, P.top_k, [&](int p, int j) { return R[p].e[j]; },
      [&](int p, int j, int b, uint32_t g) {
        R[p].buf[j] = b;
        R[p].gen[j] = g;
        R[p].ready[j] = 0;
      });
}

__global__ void k_begin_call(StoreDev S) {
  if (threadIdx.x == 0 && blockIdx.x == 0) store::begin_call(S);
}

// combine decode fast path (top_k <= 2, one CTA): out = h + w0*y0 + w1*y1,
// V values per thread, every load in flight first
template <int V, bool FX>
MOE_DEV void combine_fast(const CombineParams& P, const float* part, const float* w, float* osh,
                          int i0, int step) {
  float hv[V], y0[V], y1[V];
  unsigned long long q0[FX ? V : 1], q1[FX ? V : 1];
#pragma unroll
  for (int u = 0; u < V; ++u) {
    const int i = i0 + u * step;
    hv[u] = i < P.d ? __ldcg(P.h + i) : 0.f;
    if constexpr (FX) {
      q0[u] = i < P.d ? __ldcg(P.acc + i) : 0ull;
      q1[u] = (i < P.d && P.top_k > 1) ? __ldcg(P.acc + (size_t)P.d + i) : 0ull;
    } else {
      y0[u] = i < P.d ? __ldcg(part + i) : 0.f;
      y1[u] = (i < P.d && P.top_k > 1) ? __ldcg(part + (size_t)P.d + i) : 0.f;
    }
  }
#pragma unroll
  for (int u = 0; u < V; ++u) {
    const int i = i0 + u * step;
    if constexpr (FX) {
      y0[u] = fx_val(q0[u]);
      y1[u] = fx_val(q1[u]);
    }
    if (i < P.d) {
      float out = __fadd_rn(hv[u], __fmul_rn(w[0], y0[u]));  // model.py:251-254
      if (P.top_k > 1) out = __fadd_rn(out, __fmul_rn(w[1], y1[u]));
      P.out[i] = out;
      osh[i] = out;
    }
  }
  if constexpr (FX)  // reset the sums for the next down GEMV
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const int i = i0 + u * step;
      if (i < P.d) {
        P.acc[i] = 0ull;
        if (P.top_k > 1) P.acc[(size_t)P.d + i] = 0ull;
      }
    }
}

// out = h + w0*y0 + w1*y1 in descending-weight order (model.py:251-254)
MOE_DEV unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
MOE_DEV void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(1024) k_combine(CombineParams P) {
  __shared__ float red[33];
  extern __shared__ float osh[];  // out [d], then LN gamma / beta [d] each
  float* gs = osh + P.d;
  float* bs = gs + P.d;
  gemv::pdl_trigger();
  if (P.xn)  // immutable LN affine: fetched before waiting for the down GEMV
    for (int i = threadIdx.x; i < P.d; i += blockDim.x) {
      gs[i] = __ldg(P.ln_g + i);
      bs[i] = __ldg(P.ln_b + i);
    }
  gemv::pdl_wait();
  tl_begin(P.site);
  const float* part = P.part;
  if (P.ep_flags) {  // fused exchange: wait for every rank's column blocks of this exchange
    __shared__ unsigned long long sq_sh;
    if (threadIdx.x == 0) {
      const unsigned long long sq = __ldcg(P.ep_seq) + 1ull;
      const unsigned long long want = sq * (unsigned long long)P.ep_ncbt;
      const unsigned long long t0 = globaltimer();
      for (int r = 0; r < P.S; ++r)
        while (ld_acquire_sys_u64(P.ep_flags + r) < want) {
          __nanosleep(64);
          if (globaltimer() - t0 > P.wait_ns) {
            atomicOr(P.err, MOE_ERRF_TIMEOUT);
            break;
          }
        }
      sq_sh = sq;
    }
    __syncthreads();
    part += (size_t)(sq_sh & 1ull) * P.ep_slab;
    if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) *P.ep_seq_w = sq_sh;
  } else if (P.ep_seq) {
    part += (size_t)(*P.ep_seq & 1ull) * P.ep_slab;
  }
  // batched prefill: grid.y = positions (h, acc, route, out advance per row)
  const int row = blockIdx.y;
  const float* hin = P.h + (size_t)row * P.d;
  unsigned long long* acc = P.acc ? P.acc + (size_t)row * P.top_k * P.d : nullptr;
  float* outp = P.out + (size_t)row * P.d;
  float w[MOE_MAX_TOPK];
  for (int j = 0; j < P.top_k; ++j) w[j] = P.route[row].w[j];
  const int step = P.xn ? blockDim.x : gridDim.x * blockDim.x;
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x;
  if (P.xn && (P.S == 1 || P.acc) && P.top_k <= 2) {  // decode fast path: all loads first
    if (P.acc && P.d <= 4 * step)
      combine_fast<4, true>(P, part, w, osh, i0, step);
    else if (P.acc)
      combine_fast<8, true>(P, part, w, osh, i0, step);
    else
      combine_fast<8, false>(P, part, w, osh, i0, step);  // d <= 8192 (one CTA)
  } else {
    for (int i = i0; i < P.d; i += step) {
      float out = __ldcg(hin + i);
      for (int j = 0; j < P.top_k; ++j) {
        float y = 0.f;
        if (acc) {
          y = fx_val(__ldcg(acc + (size_t)j * P.d + i));
          acc[(size_t)j * P.d + i] = 0ull;
        } else
          for (int s = 0; s < P.S; ++s)
            y += __ldcg(part + (P.rank_major ? (size_t)s * P.top_k + j : (size_t)j * P.S + s) *
                                   P.d + i);
        out = __fadd_rn(out, __fmul_rn(w[j], y));  // model.py:251-254, reference order
      }
      outp[i] = out;
      if (P.xn) osh[i] = out;
    }
  }
  if (P.zero)  // the up projections' fixed-point sums (read by the down GEMV): reset
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.zero_n; i += gridDim.x * blockDim.x)
      P.zero[i] = 0ull;
  tl_mark(P.site, 0);
  if (P.xn) {  // fused LayerNorm of the residual stream (next LN1 or LN_f)
    __syncthreads();
    tl_mark(P.site, 1);
    layernorm_block(osh, gs, bs, P.xn, nullptr, P.d, red);
  }
  tl_mark(P.site, 2);
  tl_end(P.site);
}

__global__ void __launch_bounds__(1024) k_exchange(ExchangeParams P) {
  __shared__ unsigned long long sq;
  gemv::pdl_trigger();
  gemv::pdl_wait();
  tl_begin(P.site);
  if (threadIdx.x == 0) {
    sq = *P.seq + 1;
    *P.seq = sq;
  }
  __syncthreads();
  const size_t slab = (size_t)P.top_k * P.N * P.d;
  const int n = P.top_k * P.d;
  for (int r = 0; r < P.N; ++r) {  // P2P stores into every rank's receive buffer
    float* dst = P.recv[r] + (size_t)(sq & 1ull) * slab;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int j = i / P.d, c = i - j * P.d;
      dst[((size_t)j * P.N + P.rank) * P.d + c] = __ldcg(P.src + i);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int r = 0; r < P.N; ++r) st_release_sys_u64(P.flag[r] + P.rank, sq);
    const unsigned long long t0 = globaltimer();
    for (int r = 0; r < P.N; ++r)
      while (ld_acquire_sys_u64(P.my_flag + r) < sq) {
        __nanosleep(128);
        if (globaltimer() - t0 > P.wait_ns) {
          atomicOr(P.err, MOE_ERRF_TIMEOUT);
          break;
        }
      }
  }
  __syncthreads();
  tl_end(P.site);
}

// logits = sum of lm_head partials; non-finite check (model.py:308-309);
// argmax with lowest index on ties (model.py:374-375) via a last-block reduce.
__global__ void __launch_bounds__(256) k_logits(LogitsParams P) {
  __shared__ float bv[256];
  __shared__ int bi[256];
  __shared__ bool last;
  gemv::pdl_trigger();
  gemv::pdl_wait();
  tl_begin(P.site);
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  float val = -INFINITY;
  int idx = 0x7fffffff;
  if (v < P.V) {
    float a = 0.f;
#pragma unroll 4
    for (int s = 0; s < P.S; ++s) a += __ldcg(P.part + (size_t)s * P.V + v);
    P.logits[v] = a;
    if (!isfinite(a)) {
      atomicOr(P.err, MOE_ERRF_NONFINITE_LOGITS);
      if (P.ds) atomicCAS(P.err + 7, 0, P.ds->pos + 1);  // first failing position (+1)
    }
    val = a;
    idx = v;
  }
  bv[threadIdx.x] = val;
  bi[threadIdx.x] = idx;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if (threadIdx.x < o) {
      const float a = bv[threadIdx.x + o];
      const int ai = bi[threadIdx.x + o];
      if (a > bv[threadIdx.x] || (a == bv[threadIdx.x] && ai < bi[threadIdx.x])) {
        bv[threadIdx.x] = a;
        bi[threadIdx.x] = ai;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    P.cand_val[blockIdx.x] = bv[0];
    P.cand_idx[blockIdx.x] = bi[0];
    __threadfence();
    const unsigned int t = atomicAdd(P.counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) {
    tl_end(P.site);
    return;
  }
  __threadfence();
  float best = -INFINITY;
  int besti = 0x7fffffff;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
    const float a = __ldcg(P.cand_val + b);
    const int ai = __ldcg(P.cand_idx + b);
    if (a > best || (a == best && ai < besti)) {
      best = a;
      besti = ai;
    }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = besti;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if (threadIdx.x < o) {
      const float a = bv[threadIdx.x + o];
      const int ai = bi[threadIdx.x + o];
      if (a > bv[threadIdx.x] || (a == bv[threadIdx.x] && ai < bi[threadIdx.x])) {
        bv[threadIdx.x] = a;
        bi[threadIdx.x] = ai;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int t = bi[0] == 0x7fffffff ? 0 : bi[0];
    *P.tok_out = t;
    if (P.ds) {  // decode: record the consumed token, feed the argmax, advance
      DecodeState* ds = P.ds;
      P.tok_hist[ds->step] = ds->tok;
      ds->tok = t;
      ds->step += 1;
      ds->pos += 1;
      ds->seq += 1;
    }
    *P.counter = 0u;
  }
  tl_end(P.site);
}

}  // namespace

// ------------------------------------------------------------------ launchers
static std::atomic<long long> g_launches{0};

cudaError_t set_cta_trace(unsigned long long* buf) {
  return cudaMemcpyToSymbol(g_cta_trace, &buf, sizeof(buf));
}

cudaError_t set_timeline(TimelineSlot* table, int nslots) {
  cudaError_t e = cudaMemcpyToSymbol(g_timeline_n, &nslots, sizeof(nslots));
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(g_timeline, &table, sizeof(table));
}
long long launch_count() { return g_launches.load(); }

// Loads every kernel and sets its shared-memory limit while the GPU is idle.
// With lazy module loading, the first launch of a kernel while another kernel
// spin-waits on the copy engine can block the runtime (and so the copy
// thread): everything is loaded up front instead.
cudaError_t preload_kernels() {
  cudaFuncAttributes a;
  const void* fns[] = {(const void*)k_gemv<2>,   (const void*)k_gemv<3>,  (const void*)k_gemv<4>,
                       (const void*)k_gemv<16>,  (const void*)k_gemv<32>, (const void*)k_embed,
                       (const void*)k_layernorm, (const void*)k_attention,
                       (const void*)k_tail<MOE_TAIL_THREADS>,
                       (const void*)k_prefill_bk, (const void*)k_begin_call,
                       (const void*)k_combine,   (const void*)k_logits, (const void*)k_wait_ready,
                       (const void*)k_exchange, (const void*)k_kv_append,
                       (const void*)k_mgemv<2, 1, 1>,
                       (const void*)k_mgemv<3, 1, 1>, (const void*)k_mgemv<4, 1, 1>,
                       (const void*)k_mgemv<2, MG_PREFILL_NM, MG_PREFILL_CPG>,
                       (const void*)k_mgemv<3, MG_PREFILL_NM, MG_PREFILL_CPG>,
                       (const void*)k_mgemv<4, MG_PREFILL_NM, MG_PREFILL_CPG>};
  for (const void* f : fns) {
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
  }
  for (int i = 0; i < 5; ++i) {
    cudaError_t e = cudaFuncSetAttribute(fns[i], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         200 * 1024);
    if (e != cudaSuccess) return e;
  }
  for (const void* f : {(const void*)k_embed, (const void*)k_combine,
                        (const void*)k_attention128, (const void*)k_mgemv<2, 1, 1>,
                        (const void*)k_mgemv<3, 1, 1>, (const void*)k_mgemv<4, 1, 1>,
                        (const void*)k_mgemv<2, MG_PREFILL_NM, MG_PREFILL_CPG>,
                        (const void*)k_mgemv<3, MG_PREFILL_NM, MG_PREFILL_CPG>,
                        (const void*)k_mgemv<4, MG_PREFILL_NM, MG_PREFILL_CPG>}) {
    cudaError_t e2 = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          224 * 1024);
    if (e2 != cudaSuccess) return e2;
  }
  cudaError_t e = cudaFuncSetAttribute((const void*)k_attention,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute((const void*)k_tail<MOE_TAIL_THREADS>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              226 * 1024);  // + static shared memory <= 227 KB
}

// shared memory of one GEMV CTA (CUDA-core layout): barriers, x slice, stage
// ring (which also holds the cross-warp reduction scratch at the end)
int gemv_smem_bytes(int bits, int xs_rows, int zs_cap, int xin_cap, int rb_full, int* nstages,
                    int* stage_bytes) {
  const int WC = fmt_wc(bits);
  const int head = 512 + (((xs_rows * 8 + zs_cap * 4 + 15) & ~15) + xin_cap + 15 & ~15);
  const int stage = gemv_qs(bits) * rb_full;
  int nst = MOE_GEMV_RING / stage;
  nst = nst < 2 ? 2 : (nst > 16 ? 16 : nst);
  int ring = nst * stage;
  const int red = MOE_GEMV_WARPS * 32 * (WC + 1) * 4 + 32 * WC * 4;
  if (ring < red) ring = red;
  if (nstages) *nstages = nst;
  if (stage_bytes) *stage_bytes = stage;
  return ((head + 127) & ~127) + ring;
}

// zmeta entries of the largest per-CTA slice of the launch's uniform-run
// jobs (0 when none, or when the slice would cost the kernel its 2 CTAs/SM:
// the kernel then reads zmeta from global memory)
static int gemv_zs_cap(const GLaunch& P, int bits, int xs_cap, int rbf, int mma) {
  int cap = 0;
  for (int i = 0; i < P.nj; ++i) {
    const MatDev& M = P.j[i].M;
    if (bits > 4 || !M.runs_uniform) continue;
    const long long rows = (long long)P.j[i].QPS * (M.mma ? mt::KS : 4);
    cap = max(cap, (int)(((rows * M.G) >> M.sg_log2) + 8));
  }
  if (cap && !mma && gemv_smem_bytes(bits, xs_cap, cap, 0, rbf, nullptr, nullptr) > 112 * 1024)
    cap = 0;
  return cap;
}

// bytes of the x staging region: the largest job's x rows (two arrays for the
// SwiGLU input), 0 when a job sums producer partials or the kernel would lose
// its 2 CTAs/SM (x then comes through ordinary loads)
static int gemv_xin_cap(const GLaunch& P, int bits, int xs_cap, int zs_cap, int rbf) {
  int cap = 0;
  for (int i = 0; i < P.nj; ++i) {
    const GJob& J = P.j[i];
    if (J.xmode == X_COMBINE) {  // the full residual
      cap = max(cap, J.M.K * 4);
      continue;
    }
    const int n = (J.xmode != X_PLAIN ? 2 : 1) * (J.xS > 1 ? J.xS : 1);
    cap = max(cap, n * 4 * J.QPS * 4);
  }
  if (cap && gemv_smem_bytes(bits, xs_cap, zs_cap, cap, rbf, nullptr, nullptr) > 112 * 1024)
    cap = 0;
  return cap;
}

template <int BITS>
static void launch_gemv_t(const GLaunch& P, int nblocks, cudaStream_t s, bool pdl) {
  int xs_cap = 0, rbf = 0;
  for (int i = 0; i < P.nj; ++i) {
    xs_cap = max(xs_cap, P.j[i].QPS * 4);
    rbf = max(rbf, P.j[i].M.rb_full);
  }
  int nst = 0, stage = 0;
  const int zs_cap = gemv_zs_cap(P, BITS, xs_cap, rbf, 0);
  const int xin_cap = gemv_xin_cap(P, BITS, xs_cap, zs_cap, rbf);
  const int smem = gemv_smem_bytes(BITS, xs_cap, zs_cap, xin_cap, rbf, &nst, &stage);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nblocks);
  cfg.blockDim = dim3(MOE_GEMV_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_gemv<BITS>, P, xs_cap, zs_cap, xin_cap, nst, stage);
  g_launches.fetch_add(1);
}

// tensor-core layout (k_mgemv): x staging for every job (the full residual for
// the fused combine), the zmeta slice, scales + B table, then the ring
template <int B, int NM, int CPG>
static void launch_mgemv_t(const GLaunch& P, int nblocks, cudaStream_t s, bool pdl) {
  constexpr int NC = mg_cols(NM, CPG);
  int xs_cap = 0, rbf = 0, xin_cap = 0;
  for (int i = 0; i < P.nj; ++i) {
    const GJob& J = P.j[i];
    const int rows = J.QPS * mt::KS;
    xs_cap = max(xs_cap, rows);
    rbf = max(rbf, J.M.rb_full);
    const int n = (J.xmode == X_SWIGLU ? 2 : 1) * (J.xS > 1 ? J.xS : 1);
    xin_cap = max(xin_cap, J.xmode == X_COMBINE ? J.M.K * 4
                           : J.xmode == X_ATTN ? (3 * P.att_hd + P.att_T + 2 * rows + 40) * 4
                                               : n * 4 * rows);
  }
  xin_cap = (xin_cap + 15) & ~15;
  const int zs_cap = gemv_zs_cap(P, B, xs_cap, rbf, 1);
  const MgSmem L(xs_cap, zs_cap, xin_cap, NM, CPG);
  const int stage = mma_units(B) * rbf;
  // 2 CTAs per SM for decode; the batched kernel runs 1 CTA per SM
  const long long cap = NM * CPG <= 2 ? MOE_GEMV_SMEM_CAP : 220 * 1024;
  int nst = (int)((cap - (long long)L.ring) / stage);
  nst = nst < 2 ? 2 : (nst > 8 ? 8 : nst);
  const int ring = max(nst * stage, NC * 12 * 1024);  // the epilogue reuses the ring
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nblocks);
  cfg.blockDim = dim3(MG_THREADS);
  cfg.dynamicSmemBytes = L.ring + ring;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_mgemv<B, NM, CPG>, P, xs_cap, zs_cap, xin_cap, nst, stage);
  g_launches.fetch_add(1);
}

void launch_gemv(int bits, const GLaunch& P, int nblocks, cudaStream_t s, bool pdl) {
  if (bits <= 4 && P.j[0].M.mma) {
    switch (bits) {
      case 2: launch_mgemv_t<2, 1, 1>(P, nblocks, s, pdl); return;
      case 3: launch_mgemv_t<3, 1, 1>(P, nblocks, s, pdl); return;
      default: launch_mgemv_t<4, 1, 1>(P, nblocks, s, pdl); return;
    }
  }
  switch (bits) {
    case 2: launch_gemv_t<2>(P, nblocks, s, pdl); break;
    case 3: launch_gemv_t<3>(P, nblocks, s, pdl); break;
    case 4: launch_gemv_t<4>(P, nblocks, s, pdl); break;
    case 16: launch_gemv_t<16>(P, nblocks, s, pdl); break;
    default: launch_gemv_t<32>(P, nblocks, s, pdl); break;
  }
}

// batched prefill: MG_PREFILL_NM column groups (2 columns each) per CTA
void launch_gemv_cols(int bits, const GLaunch& P, int nblocks, cudaStream_t s) {
  switch (bits) {
    case 2: launch_mgemv_t<2, MG_PREFILL_NM, MG_PREFILL_CPG>(P, nblocks, s, false); return;
    case 3: launch_mgemv_t<3, MG_PREFILL_NM, MG_PREFILL_CPG>(P, nblocks, s, false); return;
    default: launch_mgemv_t<4, MG_PREFILL_NM, MG_PREFILL_CPG>(P, nblocks, s, false); return;
  }
}

// small kernels: optionally launched with programmatic stream serialization so
// the next kernel (usually a GEMV streaming weights that do not depend on this
// kernel) is scheduled while this one runs
template <class... Params, class... Args>
static void launch_small(void (*kern)(Params...), dim3 grid, dim3 block, size_t smem,
                         cudaStream_t s, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
  g_launches.fetch_add(1);
}

void launch_embed(const EmbedParams& P, cudaStream_t s, bool pdl) {
  if (P.xn)
    launch_small(k_embed, dim3(1), dim3(1024), (size_t)P.d * 12, s, pdl, P);
  else
    launch_small(k_embed, dim3((P.d + 255) / 256), dim3(256), 0, s, pdl, P);
}

void launch_layernorm_rows(const float* x, const float* g, const float* b, float* y, int d,
                          int rows, cudaStream_t s) {
  launch_small(k_layernorm, dim3(rows), dim3(1024), 0, s, false, x, g, b, y, d);
}

void launch_layernorm(const float* x, const float* g, const float* b, float* y, int d,
                      cudaStream_t s, bool pdl) {
  launch_small(k_layernorm, dim3(1), dim3(1024), 0, s, pdl, x, g, b, y, d);
}

void launch_attention_rows(const AttnParams& P, int rows, cudaStream_t s) {
  launch_small(k_kv_append, dim3((P.d + 255) / 256, rows), dim3(256), 0, s, false, P);
  launch_small(k_attention128, dim3(P.H, rows), dim3(256),
               (size_t)(5 * P.hd + P.T_max) * sizeof(float), s, false, P);
}

void launch_attention(const AttnParams& P, cudaStream_t s, bool pdl) {
  if (P.hd % 128 == 0) {
    launch_small(k_attention128, dim3(P.H), dim3(256),
                 (size_t)(5 * P.hd + P.T_max) * sizeof(float), s, pdl, P);
    return;
  }
  const size_t smem = (size_t)(P.hd + P.T_max) * sizeof(float);
  launch_small(k_attention, dim3(P.H), dim3(256), smem, s, pdl, P);
}

int tail_smem_bytes(const TailParams& P) {
  const bool guess = P.gate_g != nullptr;
  const bool hg = P.gh_l != nullptr && (!guess || P.gh_g != nullptr);
  const size_t head = (3 * (size_t)P.d * 4 +
                       (hg ? (guess ? 2 : 1) * (size_t)P.d * P.E * 2 : 0) + 15) & ~(size_t)15;
  return (int)(head + 2 * 1024 * sizeof(double) + ((size_t)store::stage_ints(P.st) + 4) * 4 +
               (size_t)P.st.nbuf * 4);
}

void launch_tail(const TailParams& P, cudaStream_t s, bool pdl, int rows) {
  launch_small(k_tail<MOE_TAIL_THREADS>, dim3(rows), dim3(MOE_TAIL_THREADS),
               (size_t)tail_smem_bytes(P), s, pdl, P);
}

void launch_prefill_bk(const PrefillBKParams& P, cudaStream_t s) {
  k_prefill_bk<<<1, 32, 0, s>>>(P);
  g_launches.fetch_add(1);
}
void launch_begin_call(StoreDev st, cudaStream_t s) { k_begin_call<<<1, 32, 0, s>>>(st); }

void launch_wait_ready(const RouteRec* route, int n, const uint32_t* flags, int* err,
                       unsigned long long wait_ns, cudaStream_t s) {
  k_wait_ready<<<1, 32, 0, s>>>(route, n, flags, err, wait_ns);
  g_launches.fetch_add(1);
}

void launch_hold(unsigned long long ns, cudaStream_t s) {
  k_hold<<<1, 1, 0, s>>>(ns);
  g_launches.fetch_add(1);
}

void launch_combine(const CombineParams& P, cudaStream_t s, bool pdl, int rows) {
  if (rows > 1) {  // batched prefill: no fused LayerNorm
    launch_small(k_combine, dim3((P.d + 255) / 256, rows), dim3(256), 0, s, pdl, P);
    return;
  }
  if (P.xn)
    launch_small(k_combine, dim3(1), dim3(1024), (size_t)P.d * 12, s, pdl, P);
  else if (P.ep_flags)  // fused exchange: one CTA reads and then advances the counter
    launch_small(k_combine, dim3(1), dim3(1024), 0, s, pdl, P);
  else
    launch_small(k_combine, dim3((P.d + 255) / 256), dim3(256), 0, s, pdl, P);
}

void launch_exchange(const ExchangeParams& P, cudaStream_t s, bool pdl) {
  launch_small(k_exchange, dim3(1), dim3(1024), 0, s, pdl, P);
}

void launch_logits(const LogitsParams& P, cudaStream_t s, bool pdl) {
  launch_small(k_logits, dim3((P.V + 255) / 256), dim3(256), 0, s, pdl, P);
}
