/* Fast C restatement of the reference group quantizer and of x @ dequantize(W)
 * -- TEST INFRASTRUCTURE ONLY (oracle/, see oracle/__init__.py).
 *
 * Follows /root/reference/pkg/src/moe_offload/quant.py:
 *   quantize ............ quant.py:181-229 (group min/max, f32 group scale,
 *                         one f16 scale per scale_group_size weights, RNE codes)
 *   _affine_meta ........ quant.py:147-169 (u8 zero codes in runs of
 *                         scale_group_size groups; spread in float64, f16 step)
 *   pack_codes .......... quant.py:105-113 (LSB-first bitstream)
 *   dequantize .......... quant.py:267-304 (code*scale + zhat, zhat =
 *                         zcode*zscale + zoffset; separately rounded f32 ops)
 * and the matmul the reference applies to the dequantized matrix
 * (model.py:223-226, 290-300: x @ W), here fused with the dequantization and
 * accumulated in double (the checker is at least as exact as numpy's fp32 BLAS).
 *
 * Every float operation that the reference rounds separately is written so
 * that it is rounded separately here: build with -ffp-contract=off (no FMA
 * contraction).  f32 -> f16 and f64 -> f16 conversions go through _Float16
 * (round to nearest even, direct from the source type like numpy's
 * astype(np.float16)).  Byte-identity with quant.quantize and bit-identity with
 * quant.dequantize are pinned by tests/test_oracle_c.py against the numpy
 * oracle and the reference goldens.
 *
 * Restriction (as the device engine): no row padding (cols % group_size == 0).
 */
#include <math.h>
#include <stdlib.h>
#include <stdint.h>
#include <string.h>
#include <pthread.h>

typedef struct {
  const uint8_t* codes;   /* packed LSB-first bitstream */
  const uint8_t* zeros;   /* u8 zero code per group */
  const uint16_t* zs;     /* f16 bits, one per run of sg groups */
  const uint16_t* zo;     /* f16 bits, one per run of sg groups */
  const uint16_t* scales; /* f16 bits, one per sg weights */
  int64_t K, N;           /* original shape (rows, cols) */
  int bits, g, sg;
} oq_block;

static inline float h2f(uint16_t h) {
  _Float16 v;
  memcpy(&v, &h, 2);
  return (float)v;
}
static inline uint16_t f2h(float f) {
  _Float16 v = (_Float16)f;
  uint16_t h;
  memcpy(&h, &v, 2);
  return h;
}
static inline uint16_t d2h(double d) {
  _Float16 v = (_Float16)d;
  uint16_t h;
  memcpy(&h, &v, 2);
  return h;
}

/* f32 -> f16 -> bits and f64 -> f16 -> bits, exposed for the conversion tests */
uint16_t oq_f2h(float f) { return f2h(f); }
uint16_t oq_d2h(double d) { return d2h(d); }

int oq_version(void) { return 1; }

/* ------------------------------------------------------------ threads
 * (the image's gcc has no OpenMP spec): static split of [0, n) over nthreads */
typedef void (*oq_body)(int64_t lo, int64_t hi, void* ctx);
typedef struct { oq_body fn; void* ctx; int64_t lo, hi; } oq_task;
static void* oq_run(void* a) {
  oq_task* t = (oq_task*)a;
  t->fn(t->lo, t->hi, t->ctx);
  return NULL;
}
static void par_for(int64_t n, int nthreads, oq_body fn, void* ctx) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (n < nthreads) nthreads = n > 0 ? (int)n : 1;
  pthread_t th[256];
  oq_task tk[256];
  for (int t = 0; t < nthreads; ++t) {
    tk[t].fn = fn;
    tk[t].ctx = ctx;
    tk[t].lo = n * t / nthreads;
    tk[t].hi = n * (t + 1) / nthreads;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, oq_run, &tk[t]);
  oq_run(&tk[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* ------------------------------------------------------------ quantize */
typedef struct {
  const float* w;
  int64_t n, ngroups, per_sg, nsg;
  int bits, g, sg, top;
  float *gmin, *gsc;
  uint8_t *codes, *zeros;
  uint16_t *zs, *zo, *scales;
} qctx;

static void q_groups(int64_t lo, int64_t hi, void* c) {
  qctx* q = (qctx*)c;
  for (int64_t gi = lo; gi < hi; ++gi) {
    const float* p = q->w + gi * q->g;
    float mn = p[0], mx = p[0];
    for (int k = 1; k < q->g; ++k) {
      mn = p[k] < mn ? p[k] : mn;
      mx = p[k] > mx ? p[k] : mx;
    }
    q->gmin[gi] = mn;
    q->gsc[gi] = (mx - mn) / (float)q->top; /* float32 per-group scale */
  }
}
/* one f16 scale per scale group: max of the groups' scales (padding groups
 * count as 0), 1.0 when the max is not positive */
static void q_scales(int64_t lo, int64_t hi, void* c) {
  qctx* q = (qctx*)c;
  for (int64_t si = lo; si < hi; ++si) {
    float m = 0.f;
    for (int64_t k = 0; k < q->per_sg; ++k) {
      const int64_t gi = si * q->per_sg + k;
      const float v = gi < q->ngroups ? q->gsc[gi] : 0.f;
      if (k == 0 || v > m) m = v;
    }
    q->scales[si] = f2h(m > 0.f ? m : 1.f);
  }
}
/* codes: rint((w - gmin) / s) clipped, packed LSB-first.  g * bits is a
 * multiple of 8 for every accepted scheme (checked in oq_quantize), so each
 * group owns whole bytes and groups pack independently. */
static void q_codes(int64_t lo, int64_t hi, void* c) {
  qctx* q = (qctx*)c;
  const int gb = q->g * q->bits / 8;
  for (int64_t gi = lo; gi < hi; ++gi) {
    const float s = h2f(q->scales[gi / q->per_sg]), mn = q->gmin[gi];
    const float* p = q->w + gi * q->g;
    uint8_t* out = q->codes + gi * gb;
    uint64_t acc = 0;
    int nb = 0, o = 0;
    for (int k = 0; k < q->g; ++k) {
      float cv = rintf((p[k] - mn) / s);
      cv = cv < 0.f ? 0.f : (cv > (float)q->top ? (float)q->top : cv);
      acc |= (uint64_t)(uint32_t)cv << nb;
      nb += q->bits;
      while (nb >= 8) {
        out[o++] = (uint8_t)acc;
        acc >>= 8;
        nb -= 8;
      }
    }
  }
}
/* zero points: u8 codes of the group minima in runs of sg groups */
static void q_runs(int64_t lo, int64_t hi, void* c) {
  qctx* q = (qctx*)c;
  const int64_t run = q->sg;
  for (int64_t r = lo; r < hi; ++r) {
    float mn = 0.f, mx = 0.f;
    for (int64_t k = 0; k < run; ++k) {
      int64_t gi = r * run + k;
      if (gi >= q->ngroups) gi = q->ngroups - 1; /* padded with the last value */
      const float v = q->gmin[gi];
      if (k == 0 || v < mn) mn = v;
      if (k == 0 || v > mx) mx = v;
    }
    const double spread = (double)mx - (double)mn;
    const double step = spread > 0.0 ? spread / 255.0 : 1.0;
    const uint16_t step16 = d2h(step);
    const float stepf = h2f(step16);
    q->zs[r] = step16;
    q->zo[r] = f2h(mn);
    for (int64_t k = 0; k < run; ++k) {
      const int64_t gi = r * run + k;
      if (gi >= q->ngroups) break;
      float cv = rintf((q->gmin[gi] - mn) / stepf);
      cv = cv < 0.f ? 0.f : (cv > 255.f ? 255.f : cv);
      q->zeros[gi] = (uint8_t)cv;
    }
  }
}

int oq_quantize(const float* w, int64_t K, int64_t N, int bits, int g, int sg, uint8_t* codes,
                uint8_t* zeros, uint16_t* zs, uint16_t* zo, uint16_t* scales, int nthreads) {
  if (bits < 2 || bits > 4 || g < 1 || sg % g || N % g || (g * bits) % 8) return -1;
  qctx q;
  q.w = w;
  q.n = K * N;
  q.ngroups = q.n / g;
  q.per_sg = sg / g;
  q.nsg = (q.ngroups + q.per_sg - 1) / q.per_sg;
  q.bits = bits;
  q.g = g;
  q.sg = sg;
  q.top = (1 << bits) - 1;
  q.gmin = (float*)malloc(sizeof(float) * q.ngroups);
  q.gsc = (float*)malloc(sizeof(float) * q.ngroups);
  if (!q.gmin || !q.gsc) return -2;
  q.codes = codes;
  q.zeros = zeros;
  q.zs = zs;
  q.zo = zo;
  q.scales = scales;
  par_for(q.ngroups, nthreads, q_groups, &q);
  par_for(q.nsg, nthreads, q_scales, &q);
  par_for(q.ngroups, nthreads, q_codes, &q);
  par_for((q.ngroups + sg - 1) / sg, nthreads, q_runs, &q);
  free(q.gmin);
  free(q.gsc);
  return 0;
}

/* ------------------------------------------------------------ dequantize */
static inline uint32_t code_at(const uint8_t* codes, int64_t nbytes, int64_t i, int bits) {
  const int64_t bit = i * bits, byte = bit >> 3;
  uint32_t v = 0;
  for (int k = 0; k < 2 && byte + k < nbytes; ++k) v |= (uint32_t)codes[byte + k] << (8 * k);
  return (v >> (bit & 7)) & ((1u << bits) - 1u);
}

/* w_i = code*scale + zhat (f32 ops, quant.py:298-304), zhat = zc*zscale + zoffset
 * (quant.py:172-178) */
static inline float deq_at(const oq_block* B, int64_t nbytes, int64_t i) {
  const int64_t gi = i / B->g, per_sg = B->sg / B->g;
  const float zhat = (float)B->zeros[gi] * h2f(B->zs[gi / B->sg]) + h2f(B->zo[gi / B->sg]);
  const float s = h2f(B->scales[gi / per_sg]);
  return (float)code_at(B->codes, nbytes, i, B->bits) * s + zhat;
}

typedef struct {
  const oq_block* B;
  float* out;
  int64_t nbytes;
} dctx;
static void d_body(int64_t lo, int64_t hi, void* c) {
  dctx* d = (dctx*)c;
  for (int64_t i = lo; i < hi; ++i) d->out[i] = deq_at(d->B, d->nbytes, i);
}
int oq_dequantize(const oq_block* B, float* out, int nthreads) {
  dctx d = {B, out, (B->K * B->N * B->bits + 7) / 8};
  par_for(B->K * B->N, nthreads, d_body, &d);
  return 0;
}

/* Y[v][j] = sum_i X[v][i] * dequantize(W)[i][j], double accumulation, for nx
 * input vectors (X row-major [nx][K], Y [nx][N]).  Columns are split into
 * blocks over the threads; each row's dequantized segment is formed once and
 * applied to every vector.  bits 16 / 32: plain f16 / f32 matrices. */
#define OQ_JB 256
#define OQ_MAXX 64
typedef struct {
  const oq_block* B;
  const float* X;
  double* Y;
  int nx;
  int64_t nbytes;
} gctx;
static void g_body(int64_t lo, int64_t hi, void* c) {
  gctx* G = (gctx*)c;
  const oq_block* B = G->B;
  const int64_t K = B->K, N = B->N;
  double* acc = (double*)malloc(sizeof(double) * OQ_MAXX * OQ_JB);
  float wseg[OQ_JB];
  for (int64_t b = lo; b < hi; ++b) {
    /* segments start on a group boundary: OQ_JB % g == 0 and N % g == 0 */
    const int64_t j0 = b * OQ_JB, j1 = j0 + OQ_JB < N ? j0 + OQ_JB : N, nj = j1 - j0;
    memset(acc, 0, sizeof(double) * G->nx * OQ_JB);
    for (int64_t i = 0; i < K; ++i) {
      if (B->bits == 32) {
        const float* row = (const float*)B->codes + i * N + j0;
        for (int64_t j = 0; j < nj; ++j) wseg[j] = row[j];
      } else if (B->bits == 16) {
        const uint16_t* row = (const uint16_t*)B->codes + i * N + j0;
        for (int64_t j = 0; j < nj; ++j) wseg[j] = h2f(row[j]);
      } else {  /* per group: zhat and scale once, then the group's codes */
        const int64_t per_sg = B->sg / B->g, f0 = i * N + j0;
        for (int64_t j = 0; j < nj; j += B->g) {
          const int64_t gi = (f0 + j) / B->g;
          const float zhat = (float)B->zeros[gi] * h2f(B->zs[gi / B->sg]) + h2f(B->zo[gi / B->sg]);
          const float s = h2f(B->scales[gi / per_sg]);
          for (int k = 0; k < B->g && j + k < nj; ++k)
            wseg[j + k] = (float)code_at(B->codes, G->nbytes, f0 + j + k, B->bits) * s + zhat;
        }
      }
      for (int v = 0; v < G->nx; ++v) {
        const double xv = (double)G->X[(int64_t)v * K + i];
        double* a = acc + (int64_t)v * OQ_JB;
        for (int64_t j = 0; j < nj; ++j) a[j] += xv * (double)wseg[j];
      }
    }
    for (int v = 0; v < G->nx; ++v)
      memcpy(G->Y + (int64_t)v * N + j0, acc + (int64_t)v * OQ_JB, sizeof(double) * nj);
  }
  free(acc);
}
int oq_gemv(const oq_block* B, const float* X, int nx, double* Y, int nthreads) {
  if (nx < 1 || nx > OQ_MAXX) return -1;
  gctx G = {B, X, Y, nx, (B->K * B->N * B->bits + 7) / 8};
  par_for((B->N + OQ_JB - 1) / OQ_JB, nthreads, g_body, &G);
  return 0;
}
