/*
 * moeb200.h — C ABI of the B200-native decode-time MoE offloading engine.
 *
 * The reference (``moe_offload``, /root/reference/pkg/src/moe_offload) is a
 * pure-Python package with no FFI; its drop-in seams for this hot path are the
 * ``_Session`` / ``OffloadEngine`` methods listed beside each entry point.
 * The Python mirror ``paper_2312_17238_b200.engine.OffloadEngine`` binds these
 * symbols with ctypes and maps the status codes onto the
 * reference exception classes.
 *
 * Conventions: plain pointers and sizes, no torch types; every call returns a
 * MOE_* status and ``moe_last_error()`` returns the thread-local message of the
 * last failure.  One host thread drives one engine; the engine owns its CUDA
 * streams, device memory, pinned host arena and copy-engine thread.
 */
#ifndef MOEB200_H
#define MOEB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -> reference exceptions (engine.py maps them) */
#define MOE_OK 0
#define MOE_ERR_VALUE 1           /* ValueError                                  */
#define MOE_ERR_RUNTIME 2         /* RuntimeError (e.g. decode before prefill)   */
#define MOE_ERR_NONFINITE 3       /* model.NonFiniteError (model.py:36)          */
#define MOE_ERR_UNKNOWN_EXPERT 4  /* store.UnknownExpertError (store.py:42)      */
#define MOE_ERR_FORMAT 5          /* quant.QuantFormatError (quant.py:30)        */
#define MOE_ERR_CUDA 6            /* CUDA / driver failure                       */
#define MOE_ERR_TIMEOUT 7         /* a slot-ready flag never arrived             */

/* event kinds, numbered like store.EVENT_KINDS (store.py:29-30) */
#define MOE_EV_HIT 0
#define MOE_EV_STAGING_HIT 1
#define MOE_EV_MISS_LOAD 2
#define MOE_EV_EVICT_TO_HOST 3
#define MOE_EV_SPECULATIVE_LOAD 4
#define MOE_EV_PROMOTE_FROM_STAGING 5

typedef struct moe_engine moe_engine;

/* model.ModelConfig (model.py:40-77) */
typedef struct {
  int32_t vocab_size, d_model, n_layers, n_heads, d_ffn, n_experts, top_k, max_seq_len;
} moe_model_desc;

/* store.CacheConfig (store.py:46-56); expert_bytes already resolved the way
 * OffloadEngine.__init__ does (engine.py:211-214) */
typedef struct {
  int32_t k, b;
  int64_t expert_bytes;
} moe_cache_cfg;

/* engine.SpeculationConfig (engine.py:43-57) */
typedef struct {
  int32_t enabled, m, lookahead;
} moe_spec_cfg;

/* One 2-D matrix.  bits 2/3/4: a quant.QuantizedBlock in the reference layout
 * (quant.py:76-102; ``zeros`` unpacked, one u8 code per group; f16 arrays as
 * raw uint16).  bits 16 / 32: raw row-major float16 / float32 values in
 * ``codes``. */
typedef struct {
  int32_t bits, group_size, scale_group_size, meta_bits;
  int32_t rows, cols, pad_count;
  const void* codes;
  int64_t codes_len;
  const uint8_t* zeros;
  int64_t n_groups;
  const uint16_t* zero_scales;
  const uint16_t* zero_offsets;
  int64_t n_zruns;
  const uint16_t* scales;
  int64_t n_scales;
} moe_matrix;

/* store.StoreEvent (store.py:59-73) */
typedef struct {
  int64_t seq;
  int32_t kind, layer, expert, token_pos;
  int64_t bytes_moved;
} moe_event;

/* trace.TraceRecord without the hidden vector (trace.py:38-51) */
typedef struct {
  int32_t token_pos, layer;
  int32_t experts[8];
  float weights[8];
} moe_trace_rec;

typedef struct {
  int64_t h2d_copies, h2d_bytes;
  double h2d_busy_ms;       /* copy-stream busy time, CUDA events            */
  double h2d_peak_gbs;      /* best single-copy GB/s seen                      */
  int64_t n_buffers;        /* physical expert buffers in HBM                  */
  int64_t slot_bytes;       /* bytes per expert buffer                         */
  int64_t device_bytes;     /* total device allocation                         */
  int64_t arena_bytes;      /* pinned host arena                               */
  int64_t kernel_launches;  /* kernels launched by the last API call           */
  double last_call_ms;      /* device time of the last prefill/decode/step     */
} moe_stats;

/* OffloadEngine.__init__ (engine.py:204-220): validates the geometry (k <= E,
 * m <= b) and allocates device state; weights are loaded afterwards. */
int moe_create(const moe_model_desc* model, const moe_cache_cfg* cache,
               const moe_spec_cfg* spec, int32_t device, int32_t record_hidden,
               moe_engine** out);

/* Model.params[name] (model.py:145-175 naming): "wte", "wpe", "lm_head",
 * "ln_f.gamma", "ln_f.beta", "layers.{l}.ln1.gamma", ..., "layers.{l}.attn.wq",
 * "layers.{l}.gate".  Attention projections may be quantized blocks. */
int moe_load_tensor(moe_engine* eng, const char* name, const moe_matrix* m);

/* One host-arena payload (the store's canonical copy, store.py:85-92):
 * w_gate_proj, w_up_proj, w_down_proj of expert (layer, expert). */
int moe_load_expert(moe_engine* eng, int32_t layer, int32_t expert, const moe_matrix* w_gate,
                    const moe_matrix* w_up, const moe_matrix* w_down);

/* quant.deserialize_block (quant.py:364-421): parse one serialized block
 * (quant.serialize_block bytes, e.g. read from disk) into a moe_matrix view of
 * `buf`; the meta_bits-packed zero codes are unpacked into `zeros_out`
 * (zeros_cap bytes).  zeros_out == NULL: validate and report the group count
 * only.  Malformed input -> MOE_ERR_FORMAT with the reference's message.
 * Host only (no GPU needed). */
int moe_parse_block(const uint8_t* buf, int64_t len, moe_matrix* out, uint8_t* zeros_out,
                    int64_t zeros_cap, int64_t* n_groups_out);

/* moe_load_tensor / moe_load_expert from serialized blocks (the store's
 * host-arena payloads loaded from their on-disk form, store.py:85-92). */
int moe_load_tensor_serialized(moe_engine* eng, const char* name, const uint8_t* buf,
                               int64_t len);
int moe_load_expert_serialized(moe_engine* eng, int32_t layer, int32_t expert,
                               const uint8_t* w_gate, int64_t n_gate, const uint8_t* w_up,
                               int64_t n_up, const uint8_t* w_down, int64_t n_down);

/* Device-side synthetic weights (counter hash, see oracle/model.py
 * synth_params), quantized on device with the reference quantizer
 * (quant.py:181-229); attn_bits/expert_bits in {2,3,4,32}. */
int moe_synth_model(moe_engine* eng, uint64_t seed, int32_t attn_bits, int32_t expert_bits);

/* Checks that every tensor/expert is present, builds the expert buffer pool
 * and starts the copy engine.  Must precede prefill/step/decode. */
int moe_finalize(moe_engine* eng);

/* _Session.prefill (engine.py:148-156) incl. _resolve_prefill_layer
 * (engine.py:233-240).  logits_out: n*vocab floats or NULL. */
int moe_prefill(moe_engine* eng, const int32_t* tokens, int32_t n, float* logits_out);

/* _Session.run_token (engine.py:158-166) with _resolve_token
 * (engine.py:222-231); logits_out: vocab floats or NULL. */
int moe_step(moe_engine* eng, int32_t token, float* logits_out);

/* _Session.decode with the greedy sampler (engine.py:168-182,
 * model.py:374-375), sampling on device: tokens_out n ids, final_logits_out
 * vocab floats (or NULL). */
int moe_decode_greedy(moe_engine* eng, int32_t n, int32_t* tokens_out, float* final_logits_out);

/* OffloadEngine.events / store.events (engine.py:242-244) */
int64_t moe_num_events(moe_engine* eng);
int moe_read_events(moe_engine* eng, int64_t start, int64_t count, moe_event* out);

/* _Session._records / trace() (engine.py:122-144), current session only,
 * (token_pos, layer) order; hidden_out: count*d_model floats or NULL. */
int64_t moe_num_trace(moe_engine* eng);
int moe_read_trace(moe_engine* eng, int64_t start, int64_t count, moe_trace_rec* out,
                   float* hidden_out);

/* _Session.reset_session (engine.py:100-110): KV and position, not the store */
int moe_reset_session(moe_engine* eng);

/* device LRU state (store.device_state, store.py:108-109): out[l*k + i] =
 * expert id (MRU first), -1 padded; staged: b entries of layer*E+expert or -1 */
int moe_device_state(moe_engine* eng, int32_t* lru_out, int32_t* staged_out);

int moe_get_stats(moe_engine* eng, moe_stats* out);

/* Host-link peak for the roofline (SURVEY §8(d) "H2D_peak must be measured on
 * the box"): `reps` copies of one whole expert (expert_bytes) from the pinned
 * arena into an HBM pool buffer on the copy engine's demand stream, timed
 * with CUDA events; best and median GB/s.  Engine must be idle (between
 * calls).  No reference counterpart. */
int moe_measure_h2d(moe_engine* eng, int32_t reps, double* best_gbs, double* median_gbs);

/* Expert parallel over N GPUs; no reference counterpart (the
 * reference is single-process).  configure: before any expert is loaded; this
 * rank then owns experts e with e*world/E == rank in every layer (its arena,
 * cache and store, store.py restricted to the owned keys).  After finalize,
 * exchange every rank's 64-byte handle (moe_ep_handle) and moe_ep_connect
 * with all of them, in rank order: the per-layer slot exchange then runs
 * over peer memory (NVLink P2P / CUDA IPC) inside the decode graph, fused
 * into the down-projection GEMV (each completed column block is stored into
 * every rank's receive buffer and counted there). */
int moe_ep_configure(moe_engine* eng, int32_t rank, int32_t world);
int moe_ep_handle(moe_engine* eng, void* out64);
int moe_ep_connect(moe_engine* eng, const void* handles);

/* Expert parallel over NCCL instead of peer memory (north_star: "hidden states
 * exchanged by NCCL all-to-all over NVLink").  Rank 0 calls
 * moe_nccl_unique_id, the 128-byte id reaches every rank out of band
 * (torch.distributed broadcast), and every rank calls moe_ep_connect_nccl
 * after finalize and before its first decode.  The per-layer slot exchange is
 * then one ncclAllGather of the (top_k x d) slot buffers on the compute stream
 * (captured in the decode graph), summed in rank order by the combine: the
 * same exact sum as the peer-memory exchange.  NCCL is resolved at run time
 * (libnccl.so.2).  world = 1 is allowed (a one-rank all-gather), which is how
 * the transport is tested on one GPU. */
int moe_nccl_unique_id(void* out128);
int moe_ep_connect_nccl(moe_engine* eng, const void* id128);

/* Profiling: when on, every GEMV launch is bracketed by CUDA events on the
 * compute stream; moe_kernel_times returns summed milliseconds and launch
 * counts per class [qkv, wo, expert_up, expert_down, lm_head] (5 entries). */
int moe_set_profiling(moe_engine* eng, int32_t on);
int moe_kernel_times(moe_engine* eng, double* ms_out, int64_t* count_out);
/* Kernel timeline (profiling aid): on = reset the table and make every kernel
 * record its earliest CTA start (after its programmatic-launch wait) and
 * latest CTA end (%globaltimer ns) into slot: 0 embed, 1+8l+{0 qkv, 1 attn,
 * 2 wo, 3 tail, 4 up, 5 down, 6 combine}, 1+8L lm_head, 2+8L logits.
 * moe_read_timeline: out[2*i] = start, out[2*i+1] = end (cap slots). */
int moe_timeline(moe_engine* eng, int32_t on);
int moe_read_timeline(moe_engine* eng, uint64_t* out, int32_t cap, int32_t* n_out);

/* cudaProfilerStart/Stop, so `ncu --profile-from-start off` captures only the
 * bench's timed decode region. */
int moe_profiler_range(int32_t on);

/* cudaSetDevice for the library's own runtime (host helpers such as
 * moe_quantize_device run on the calling thread's current device). */
int moe_set_device(int32_t device);
const char* moe_last_error(void);
int moe_destroy(moe_engine* eng);

/* Standalone kernels exposed for parity tests (no engine needed):
 * quantize a row-major fp32 matrix on device into the reference layout
 * (quant.py:181-229); outputs sized as quant.py's arrays. */
int moe_quantize_device(const float* w, int32_t rows, int32_t cols, int32_t bits,
                        int32_t group_size, int32_t scale_group_size, uint8_t* codes_out,
                        uint8_t* zeros_out, uint16_t* zscales_out, uint16_t* zoffsets_out,
                        uint16_t* scales_out);

/* y = x @ dequantize(m) through the engine's GEMV kernel (fp32 accumulate). */
int moe_gemv_device(const moe_matrix* m, const float* x, float* y);

/* GEMV microbenchmark (profiling aid): njobs K x N synthetic matrices of
 * `bits` per launch, weight sets rotated beyond L2; average us per launch and
 * algorithmic GB/s (reference payload bytes / time); detail_out (4 doubles, or
 * NULL): one timeline-traced launch's span and block 0's prologue / loop /
 * reduction end times, us from the first CTA start. */
int moe_bench_gemv(int32_t bits, int32_t K, int32_t N, int32_t njobs, int32_t iters, int32_t pdl,
                   double* us_out, double* gbs_out, double* detail_out);

/* synthetic tensor (oracle/model.py synth_tensor) generated on device */
int moe_synth_tensor_device(uint64_t seed, uint64_t tensor_id, int64_t count, float scale,
                            float* out);

/* ------------------------------------------------------------------------
 * Host execution of the device store (store_dev.cuh), for CPU tests and the
 * expert-parallel ownership logic.  Runs the very functions the bookkeeping
 * kernels run (store::resolve_token / resolve_prefill), so it replaces the
 * reference TieredExpertStore (store.py:76-220) driven the way
 * OffloadEngine._resolve_token / _resolve_prefill_layer drive it
 * (engine.py:222-240).  `owned` (L*E bytes or NULL) restricts the store to
 * one expert-parallel rank's keys. */
typedef struct moe_store_sim moe_store_sim;
int moe_store_sim_create(int32_t n_layers, int32_t n_experts, int32_t k, int32_t b,
                         int64_t expert_bytes, int32_t top_k, int32_t m, const uint8_t* owned,
                         moe_store_sim** out);
/* one decode layer: acquire experts[0..k) then speculative_load guesses[0..m)
 * of guess_layer (-1: none); bufs_out[k] physical buffers (-1: not owned) */
int moe_store_sim_token(moe_store_sim* s, int32_t layer, int32_t pos, const int32_t* experts,
                        int32_t k, const int32_t* guesses, int32_t m, int32_t guess_layer,
                        int32_t* bufs_out);
/* one prefill layer: experts[n][k]; bufs_out[n][k] */
int moe_store_sim_prefill(moe_store_sim* s, int32_t layer, const int32_t* experts, int32_t n,
                          int32_t k, int32_t* bufs_out);
int64_t moe_store_sim_num_events(moe_store_sim* s);
int moe_store_sim_events(moe_store_sim* s, moe_event* out, int64_t cap);
int moe_store_sim_state(moe_store_sim* s, int32_t* lru_out, int32_t* staged_out,
                        int32_t* content_out, int32_t* res_buf_out, int32_t* stg_buf_out,
                        int32_t* nbuf_out);
int64_t moe_store_sim_copies(moe_store_sim* s);
/* simulate the engine's copy-engine policy (copy_sched.h): expert jobs of
 * job_bytes in chunks of chunk_bytes (0 = whole), `progress` chunks executed
 * after each bookkeeping call before the GEMVs pull their buffers; a routed
 * buffer that can never be published returns MOE_ERR_TIMEOUT (deadlock) */
int moe_store_sim_copy_policy(moe_store_sim* s, int64_t job_bytes, int64_t chunk_bytes,
                              int32_t progress);
int64_t moe_store_sim_chunks(moe_store_sim* s);
/* speculative jobs parked so far (their target layer had passed), and the
 * parking switch of the simulated copy engine (engine: MOE_COPY_PARK) */
int64_t moe_store_sim_parked(moe_store_sim* s);
int moe_store_sim_set_park(moe_store_sim* s, int32_t on);
const char* moe_store_sim_last_error(void);
int moe_store_sim_destroy(moe_store_sim* s);

#ifdef __cplusplus
}
#endif
#endif /* MOEB200_H */
