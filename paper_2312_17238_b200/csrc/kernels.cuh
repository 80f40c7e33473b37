// Kernel parameter blocks shared by kernels.cu (device) and engine.cu (host).
#pragma once
#include "common.cuh"
#include "store_dev.cuh"

#define MOE_GEMV_WARPS 8     // consumer warps per CTA (+1 producer warp)
#define MOE_GEMV_THREADS (MOE_GEMV_WARPS * 32 + 32)
#define MOE_GEMV_QS 8        // quads per pipeline stage for dense formats (one per warp)
// quant formats: each consumer warp takes 2 quads per stage (more independent
// work between barrier waits)
__host__ __device__ constexpr int gemv_qpw(int bits) { return bits <= 4 ? 2 : 1; }
__host__ __device__ constexpr int gemv_qs(int bits) { return MOE_GEMV_WARPS * gemv_qpw(bits); }
#define MOE_GEMV_MAXJOBS 8
#define MOE_EP_MAX 8
#define MOE_GEMV_MINB 2            // CTAs per SM the kernel is register-limited for
#define MOE_GEMV_RING (80 * 1024)  // bytes of stage ring per CTA (2 CTAs / SM)
#define MOE_XS_MAX 4096            // rows of x kept in smem per CTA
#define MOE_GEMV_SMEM_CAP (112 * 1024)  // dynamic smem per CTA at 2 CTAs / SM
#ifndef MOE_UPS24
#define MOE_UPS24 2
#endif
#ifndef MOE_UPS3
#define MOE_UPS3 2
#endif
// threads of the tail kernel (one CTA per position)
#ifndef MOE_TAIL_THREADS
#define MOE_TAIL_THREADS 512
#endif
#define MOE_MMA_UNITS_MAX 64       // k-steps per CTA in the tensor-core layout (B table)
// k-steps per pipeline stage of the tensor-core layout (a compile-time count so
// the consumer loop is unrolled and its shared-memory loads run ahead)
__host__ __device__ constexpr int mma_units(int bits) { return bits == 3 ? MOE_UPS3 : MOE_UPS24; }

// X_COMBINE: the input row slice is LayerNorm(h + w0*y0 + w1*y1) (the MoE
// combine of the previous layer, model.py:251-254, fused with the next LN):
// every CTA forms the full residual (fixed-point expert sums, reference
// order) and its LN statistics; block 0 also stores the residual
// X_ATTN (decode Wo): the input rows are the CTA's head dims of the attention
// context, computed in the prologue (attend_head, model.py:294-299) from the
// QKV fixed-point sums and the KV cache; one CTA per head appends the k / v rows
enum XMode { X_PLAIN = 0, X_SWIGLU = 1, X_COMBINE = 2, X_ATTN = 3 };

struct GJob {
  MatDev M;            // absolute pointers, or byte offsets when rel_slot >= 0
  int rel_slot;        // >= 0: expert matrix, base = pool + route.buf[rel_slot]*stride
  int xmode;
  const float* x;      // X_PLAIN input (length K)
  const float* up1;    // X_SWIGLU: x@W1 [K]
  const float* up3;    //           x@W3 [K]
  int xS;              // the inputs are xS split-K partials [xS][xstride], summed in
  int xstride;         //   order on load (a producer GEMV left them unreduced); 0/1: plain
  // X_COMBINE inputs: x = h, expert sums `cacc` [ctop][K] (fixed point), LN
  // affine, and the residual output (block 0)
  const unsigned long long* cacc;
  const float* lng;
  const float* lnb;
  float* xout;
  int ctop;
  float* part;         // split-K partial outputs [S][N]
  float* out;          // final outputs [N] when reduce == 1 (the last CTA of a cb sums
  int reduce;          //   the partials in order); 0: the consumer sums part[0..S);
                       //   2: every CTA adds its partial into `acc` in fixed point
  unsigned long long* acc;  // reduce == 2: [N] int64 sums, 2^-32 units (consumer zeroes)
  int S, QPS, blk0;    // splits of the quad range, quads per split (multiple of QS)
  // batched prefill (tensor-core layout): `ncol` input columns, (input index,
  // output index) pairs in device memory; column c reads x (up1/up3) at
  // + in * xcs floats and writes part/acc at + out * ocs.  cols == null: the
  // single decode column (indices 0).  ncg = column groups of the launch's
  // columns per CTA (the grid covers ncb * S * ncg CTAs of this job).
  const int2* cols;
  int ncol, ncg;
  long long xcs, ocs;
  int rel_pos;         // expert jobs: the route is P.route[rel_pos] (decode: 0)
};

struct DecodeState;

struct GLaunch {
  GJob j[MOE_GEMV_MAXJOBS];
  int nj;
  const RouteRec* route;
  const uint8_t* pool;
  long long slot_stride;
  const uint32_t* flags;        // buffer ready generations (copy engine)
  int* cnt;                     // split-K arrival counters [sum of ncb] (zero between launches)
  unsigned long long* zero;     // optional: fixed-point sums consumed by an earlier kernel,
  int zero_n;                   //   reset by this launch's CTAs (a slice each)
  int* err;
  unsigned long long wait_ns;
  int site;  // timeline slot of this launch (profiling), -1 none
  // X_ATTN jobs: q/k/v sums [3][d] (reset later by the tail), this layer's KV
  // cache [T][H][hd], the position (decode cursor, else att_pos)
  const unsigned long long* att_acc;
  float* att_kc;
  float* att_vc;
  const DecodeState* att_ds;
  int att_pos, att_hd, att_T;
  // expert parallel, exchange fused into the down GEMV (reduce == 1 jobs,
  // ep_n > 1): the CTA that completes a column block of slot j stores those
  // outputs straight into every rank's receive buffer [2][top_k][N][d] at
  // (j, ep_rank) over peer memory, then bumps that rank's arrival counter
  // ep_flag[r][ep_rank] (system scope).  ep_seq: exchanges completed so far
  // (advanced by the combine that consumes this one).
  float* ep_recv[MOE_EP_MAX];
  unsigned long long* ep_flag[MOE_EP_MAX];
  const unsigned long long* ep_seq;
  int ep_rank, ep_n, ep_topk;
};

// Split-K by fixed-point atomics (GJob.reduce == 2): each CTA adds its fp32
// partial p as round(p * 2^32) into an int64 sum; integer addition makes the
// result independent of CTA order (deterministic), and the one rounding back
// to fp32 happens in the consumer.  |p| >= 2^30 or non-finite raises an error.
#define MOE_FX_SCALE 0x1p32f
#define MOE_FX_UNSCALE 0x1p-32

// Device-resident decode cursor: the kernels of one decode token read the
// position and input token from here, and k_logits advances it, so one
// captured CUDA graph serves every token (no per-token parameters).
struct DecodeState {
  int pos;   // position of the token being decoded
  int step;  // index of this token within the current decode call
  int tok;   // token to embed
  unsigned int seq;  // decode tokens since the engine was created (never reused)
};

struct AttnParams {
  const float* qkv_part;  // [3][S][d]
  int S;
  unsigned long long* acc;  // or: q/k/v as fixed-point sums [3][d] (read, then zeroed)
  float* kc;              // this layer's K cache [max_seq][H][hd]
  float* vc;
  float* ctx;             // [d] (batched prefill: [rows][d])
  const float* qbuf;      // batched prefill: q rows [rows][d] (K/V rows already appended)
  const DecodeState* ds;  // decode: position from here (else `pos`)
  int pos, H, hd, d, T_max;
  int site;  // timeline slot of this launch (profiling), -1 none
};

struct TailParams {
  const float* x;         // residual input [d]
  const float* part;      // Wo partials [S][d]
  int S;
  unsigned long long* acc;  // or: Wo output as fixed-point sums [d] (read, then zeroed)
  const float* g2;        // ln2 gamma / beta
  const float* b2;
  const float* gate_l;    // [d][E] gate of this layer
  const float* gate_g;    // [d][E] gate of the guessed layer (or null)
  const __half* gh_l;     // the same gates as exact fp16 copies (fp16-passthrough
  const __half* gh_g;     //   roles, quant.py:428), or null: staged in smem by TMA
  float* h;               // pre-MoE hidden out [d]
  RouteRec* route;        // route of this position
  TraceRecDev* trace;     // trace records [T][L]; slot pos*L + layer
  float* trace_hidden;    // [T][L][d] or null
  const DecodeState* ds;  // decode: position from here (else `pos`)
  int n_layers;
  StoreDev st;
  int d, E, top_k, m, layer, guess_layer, pos, mode;  // mode 0 decode, 1 prefill (no store)
  int ep_rank, ep_size;   // expert parallel (ep_size 1 = off)
  int site;  // timeline slot of this launch (profiling), -1 none
  unsigned long long* zero;  // optional: sums consumed by the fused attention (Q/K/V), reset
  int zero_n;
};

struct PrefillBKParams {
  RouteRec* route;  // [n]
  StoreDev st;
  int layer, n, top_k;
};

struct CombineParams {
  const float* h;     // [d]
  const float* part;  // [top_k][S][d]
  int S;
  unsigned long long* acc;  // or: expert outputs as fixed-point sums [top_k][d] (zeroed)
  const RouteRec* route;
  float* out;         // [d]
  int d, top_k;
  // expert parallel: `part` is the local receive buffer [2][top_k][S=N][d];
  // the half in use is picked by the exchange counter's parity
  const unsigned long long* ep_seq;
  long long ep_slab;
  // fused exchange (GLaunch.ep_*): wait until every rank's arrival counter
  // ep_flags[r] reaches (exchange number) x ep_ncbt, then advance *ep_seq_w
  const unsigned long long* ep_flags;
  unsigned long long* ep_seq_w;
  long long ep_ncbt;
  int* err;
  unsigned long long wait_ns;
  // expert parallel over NCCL: `part` is the all-gather output [S=N][top_k][d]
  // (rank-major); summed in rank order like the peer-memory layout
  int rank_major;
  // optional fused LayerNorm of `out` (next layer's LN1, or LN_f after the
  // last layer): one CTA, xn = LN(out)
  const float* ln_g;
  const float* ln_b;
  float* xn;
  unsigned long long* zero;  // optional: fixed-point sums consumed by this layer's down
  int zero_n;                //   GEMV (the up projections), reset here for the next layer
  int site;  // timeline slot of this launch (profiling), -1 none
};

// Expert-parallel slot exchange (one per layer and position): every rank
// stores its (top_k x d) slot buffer -- the outputs of the routed experts it
// owns, zeros elsewhere -- into the receive buffer of every rank over peer
// memory (NVLink P2P / CUDA IPC), then raises its flag on every rank and
// waits for all flags.  Receive buffers are double-buffered by the exchange
// sequence number (a rank can be at most one exchange ahead of any other).
struct ExchangeParams {
  const float* src;                      // [top_k][d]
  float* recv[MOE_EP_MAX];               // per rank: its receive buffer [2][top_k][N][d]
  unsigned long long* flag[MOE_EP_MAX];  // per rank: its flag array [N]
  unsigned long long* seq;               // local exchange counter
  const unsigned long long* my_flag;     // local flags [N]
  int rank, N, top_k, d;
  int* err;
  unsigned long long wait_ns;
  int site;
};

struct LogitsParams {
  const float* part;  // [S][V]
  int S, V;
  float* logits;      // [V]
  float* cand_val;    // [nblk]
  int* cand_idx;
  unsigned int* counter;
  int* tok_out;       // argmax
  int* tok_hist;      // decode: argmax history, slot ds->step
  DecodeState* ds;    // decode: advanced (tok, step, pos) by the last block
  int* err;
  int site;  // timeline slot of this launch (profiling), -1 none
};

struct EmbedParams {
  const void* wte;
  const void* wpe;
  int half;               // 1: fp16 tables
  const DecodeState* ds;  // decode: token and position from here
  int tok, pos, d;        // prefill
  float* x;
  const float* ln_g;      // optional fused LN1 of layer 0 (one CTA): xn = LN(x)
  const float* ln_b;
  float* xn;
  int site;  // timeline slot of this launch (profiling), -1 none
};

// Kernel timeline (profiling): when enabled, every kernel records the
// earliest CTA start and the latest CTA end (%globaltimer, ns) into slot
// `site` of a device table; with PDL the spans overlap like the real run.
struct TimelineSlot {
  unsigned long long start, end;
};
cudaError_t set_timeline(TimelineSlot* table, int nslots);  // null disables
cudaError_t set_cta_trace(unsigned long long* buf);          // GEMV microbench only

// launchers (kernels.cu)
void launch_gemv(int bits, const GLaunch& P, int nblocks, cudaStream_t s, bool pdl);
// batched prefill (tensor-core layout only): jobs with `cols`, MG_PREFILL_COLS
// input columns per CTA
#ifndef MG_PREFILL_NM
#define MG_PREFILL_NM 1
#endif
#ifndef MG_PREFILL_CPG
#define MG_PREFILL_CPG 2
#endif
#define MG_PREFILL_COLS (MG_PREFILL_CPG * MG_PREFILL_NM)
void launch_gemv_cols(int bits, const GLaunch& P, int nblocks, cudaStream_t s);
int gemv_smem_bytes(int bits, int xs_rows, int zs_cap, int xin_cap, int rb_full, int* nstages,
                    int* stage_bytes);
void launch_embed(const EmbedParams& P, cudaStream_t s, bool pdl = false);
void launch_layernorm(const float* x, const float* g, const float* b, float* y, int d,
                      cudaStream_t s, bool pdl = false);
// one CTA per row: y[r] = LN(x[r]) for r < rows (batched prefill)
void launch_layernorm_rows(const float* x, const float* g, const float* b, float* y, int d,
                           int rows, cudaStream_t s);
// batched prefill (head_dim % 128 == 0): k_kv_append then attention with
// grid (H, rows), positions pos .. pos + rows - 1
void launch_attention_rows(const AttnParams& P, int rows, cudaStream_t s);
void launch_attention(const AttnParams& P, cudaStream_t s, bool pdl = false);
// rows > 1 (batched prefill, mode 1 only): CTA r handles position pos + r
// (x, acc, h, route advance by r rows)
void launch_tail(const TailParams& P, cudaStream_t s, bool pdl = false, int rows = 1);
int tail_smem_bytes(const TailParams& P);
void launch_prefill_bk(const PrefillBKParams& P, cudaStream_t s);
// rows > 1 (batched prefill, no fused LN): grid.y = positions (h, acc, route,
// out advance per row)
void launch_combine(const CombineParams& P, cudaStream_t s, bool pdl = false, int rows = 1);
void launch_exchange(const ExchangeParams& P, cudaStream_t s, bool pdl = false);
void launch_wait_ready(const RouteRec* route, int n, const uint32_t* flags, int* err,
                       unsigned long long wait_ns, cudaStream_t s);
void launch_logits(const LogitsParams& P, cudaStream_t s, bool pdl = false);
void launch_hold(unsigned long long ns, cudaStream_t s);  // event-timing pass only
void launch_begin_call(StoreDev st, cudaStream_t s);
cudaError_t preload_kernels();
long long launch_count();  // kernels launched (or captured) by this process
cudaError_t preload_tile_kernels();

// tiling + quantization + synthesis (tile.cu)
struct RefMat {  // reference-layout matrix resident on device
  int bits, g, sg, K, N;
  const uint8_t* codes;
  const uint8_t* zeros;
  const uint16_t* zs;
  const uint16_t* zo;
  const uint16_t* scales;
  int64_t nruns;
};
void launch_tile(const RefMat& R, const MatDev& M, uint8_t* rec, __half2* zmeta,
                 cudaStream_t s);
void launch_quantize(const float* w, int K, int N, int bits, int g, int sg, uint8_t* codes,
                     uint8_t* zeros, uint16_t* zs, uint16_t* zo, uint16_t* scales, float* gmin_ws,
                     float* gscale_ws, cudaStream_t s);
void launch_synth(uint64_t seed, uint64_t tid, int64_t count, float scale, int to_half_round,
                  float* out, cudaStream_t s);
