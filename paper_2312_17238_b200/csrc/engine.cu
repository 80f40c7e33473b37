// Host side of the B200 MoE offloading engine: the C ABI of include/moeb200.h.
//
// Owns: device weights in the tiled layout, the pinned host arena (canonical
// expert copies, store.py:85-92), the HBM expert-buffer pool, the device
// store state (store_dev.cuh), and a copy-engine thread that drains the
// device's copy-request mailbox with cudaMemcpyAsync on a side stream and
// marks each buffer ready with cuStreamWriteValue32 (kernels wait on it).
#include <cuda.h>
#include <cuda_profiler_api.h>
#include <nvtx3/nvToolsExt.h>
#include <dlfcn.h>
#include <nccl.h>
#include <atomic>
#include <chrono>
#include <algorithm>
#include <cmath>
#include <deque>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "copy_sched.h"
#include "kernels.cuh"

namespace {
// NCCL, resolved at run time (the process's libnccl.so.2: torch's bundled one
// when torch is loaded) so the library has no link-time NCCL dependency; only
// the expert-parallel NCCL transport (moe_ep_connect_nccl) uses it.
struct NcclApi {
  decltype(&ncclGetUniqueId) unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  std::string why;
};
const NcclApi& nccl_api() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.why = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
      return a;
    }
    a.unique_id = reinterpret_cast<decltype(a.unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.init_rank = reinterpret_cast<decltype(a.init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
    a.destroy = reinterpret_cast<decltype(a.destroy)>(dlsym(h, "ncclCommDestroy"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!a.unique_id || !a.init_rank || !a.all_gather || !a.destroy || !a.error_string)
      a.why = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

// NVTX range over one C-ABI call (header-only nvtx3: a no-op unless a tool
// such as nsys / ncu --nvtx injects itself)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CU(call)                                                                             \
  do {                                                                                       \
    cudaError_t _e = (call);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      return fail(MOE_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e));         \
  } while (0)

int ilog2(int v) {
  int r = 0;
  while ((1 << r) < v) ++r;
  return ((1 << r) == v) ? r : -1;
}

struct DevMat {  // one tiled matrix in device memory
  MatDev M{};
  void* mem = nullptr;
  size_t bytes = 0;
  int bits = 0;
};

// split the quad range of every job so one launch is ~2 CTAs per SM
// (MOE_GEMV_THREADS threads, ~100 KB smem each); QPS is a multiple of the
// pipeline stage so every bulk copy stays 16-byte aligned
int plan_qps(int total_cb, int nquads, int qs, bool mma = false, int nwaves = 1) {
  const int waves = MOE_GEMV_MINB * nwaves;  // CTAs per SM x resident waves
  // splits need not be whole pipeline stages (the last stage of a split is
  // partial), so S is the largest split count that fits the resident wave:
  // every SM gets the same number of CTAs whenever total_cb * S == target
  const int target = waves * 148;
  const int S = std::max(1, target / total_cb);  // at most one wave
  int qps = (nquads + S - 1) / S;
  (void)qs;
  if (mma) return std::max(1, std::min(qps, MOE_MMA_UNITS_MAX));  // k-steps (B table)
  while (qps * 4 > MOE_XS_MAX) qps -= 1;
  return std::max(qps, 1);
}

struct Layout {  // byte sections of one tiled matrix
  int bits = 0, K = 0, N = 0, g = 0, sg = 0;
  int runs_uniform = 0;  // see MatDev::runs_uniform
  int mma = 0;           // tensor-core tile layout (mma_layout.cuh)
  size_t rec = 0, scales = 0, zeros = 0, zmeta = 0;
  int64_t nruns = 0;
  size_t total() const { return rec + scales + zeros + zmeta; }
};

// record bytes of a laid-out matrix, including zero pad quads (K % 32 != 0)
size_t layout_rec_bytes(const Layout& L) {
  const int wc = fmt_wc(L.bits), nchunks = L.N / wc, ncb = (nchunks + 31) / 32;
  const int nqp = ((L.K / 4) + 7) / 8 * 8;
  const int gl = L.bits <= 4 ? ilog2(L.g) : 0, sl = L.bits <= 4 ? ilog2(L.sg) : 0;
  const int last = nchunks - (ncb - 1) * 32;
  return (size_t)nqp * ((size_t)(ncb - 1) * rec_bytes(L.bits, 32, gl, sl) +
                        rec_bytes(L.bits, last, gl, sl));
}

int make_layout(const moe_matrix* m, Layout* L, const char* what) {
  const int bits = m->bits;
  if (bits != 2 && bits != 3 && bits != 4 && bits != 16 && bits != 32)
    return fail(MOE_ERR_VALUE, std::string(what) + ": unsupported bits " + std::to_string(bits));
  const int K = m->rows, N = m->cols;
  if (K < 1 || N < 1) return fail(MOE_ERR_VALUE, std::string(what) + ": empty matrix");
  const int wc = fmt_wc(bits);
  if (K % 4) return fail(MOE_ERR_VALUE, std::string(what) + ": rows must be a multiple of 4");
  if (N % wc)
    return fail(MOE_ERR_VALUE,
                std::string(what) + ": cols must be a multiple of " + std::to_string(wc));
  L->bits = bits;
  L->K = K;
  L->N = N;
  if (bits >= 16) {
    const int64_t need = (int64_t)K * N * (bits / 8);
    if (m->codes_len != need) return fail(MOE_ERR_FORMAT, std::string(what) + ": payload size mismatch");
    L->rec = layout_rec_bytes(*L);
    return MOE_OK;
  }
  const int g = m->group_size, sg = m->scale_group_size;
  if (m->meta_bits != 8) return fail(MOE_ERR_VALUE, std::string(what) + ": meta_bits must be 8");
  if (m->pad_count != 0 || N % g)
    return fail(MOE_ERR_VALUE, std::string(what) + ": cols must be a multiple of group_size");
  if (ilog2(g) < 0 || ilog2(sg) < 0 || g % wc || sg % g || N % sg || (32 * wc) % sg)
    return fail(MOE_ERR_VALUE, std::string(what) + ": unsupported grouping for the device layout");
  if (((int64_t)g * bits) % 32) return fail(MOE_ERR_VALUE, std::string(what) + ": group not word aligned");
  const int64_t ng = (int64_t)K * N / g;
  const int64_t nsg = (ng + sg / g - 1) / (sg / g);
  const int64_t nruns = (ng + sg - 1) / sg;
  if (m->codes_len != (int64_t)K * N * bits / 8 || m->n_groups != ng || m->n_scales != nsg ||
      m->n_zruns != nruns)
    return fail(MOE_ERR_FORMAT, std::string(what) + ": block arrays inconsistent with shape");
  L->g = g;
  L->sg = sg;
  L->zmeta = (size_t)nruns * 4;
  L->nruns = nruns;
  // tensor-core layout for the reference presets (mma_layout.cuh): records of
  // codes + zero codes per (1024-output cb, 16-row k-step), then the scales
  // section; the zero-point runs of a row's cb must be one run (uniform)
  static const bool no_mma = getenv("MOE_NO_MMA") && atoi(getenv("MOE_NO_MMA")) != 0;
  if (!no_mma && N % mt::SO == 0 && K % mt::KS == 0 && (g == 16 || g == 64) && mt::SO % g == 0 &&
      (sg == 128 || sg == 256) && N % sg == 0) {
    const int64_t G = N / g, cbg = mt::CBO / g;
    const int ncb = (N + mt::CBO - 1) / mt::CBO, lg = ilog2(sg);
    bool uni = true;
    for (int64_t r = 0; r < K && uni; ++r)
      for (int c = 0; c < ncb && uni; ++c) {
        const int64_t f0 = r * G + c * cbg, n = std::min<int64_t>(cbg, G - c * cbg);
        uni = (f0 >> lg) == ((f0 + n - 1) >> lg);
      }
    if (uni) {
      L->mma = 1;
      L->runs_uniform = 1;
      L->rec = (size_t)K * N * bits / 8 + (size_t)K * N / g;
      L->scales = (size_t)K * N / sg * 2;
      return MOE_OK;
    }
  }
  // records = codes + zeros (1 B per group) + scales (f16 per scale group);
  // equal to the reference byte count whenever K % 32 == 0 (no pad quads)
  L->rec = layout_rec_bytes(*L);
  // does any row's slice of a column block straddle a zero-point run?
  {
    const int64_t G = N / g, cbg = 32 * wc / g;
    const int ncb = (N / wc + 31) / 32, lg = ilog2(sg);
    bool uni = true;
    for (int64_t r = 0; r < K && uni; ++r)
      for (int c = 0; c < ncb && uni; ++c) {
        const int64_t f0 = r * G + c * cbg, n = std::min<int64_t>(cbg, G - c * cbg);
        uni = (f0 >> lg) == ((f0 + n - 1) >> lg);
      }
    L->runs_uniform = uni ? 1 : 0;
  }
  return MOE_OK;
}

MatDev matdev_from(const Layout& L, const uint8_t* base) {
  MatDev M{};
  M.base = base;
  M.zmeta = reinterpret_cast<const __half2*>(base + L.rec + L.scales + L.zeros);
  M.K = L.K;
  M.N = L.N;
  M.bits = L.bits;
  if (L.mma) {  // units are 16-row k-steps, cbs 1024 outputs of 128-output slices
    M.mma = 1;
    M.scl = reinterpret_cast<const __half*>(base + L.rec);
    M.nquads = L.K / mt::KS;
    M.nqp = M.nquads;
    M.nchunks = L.N / mt::SO;
    M.ncb = (L.N + mt::CBO - 1) / mt::CBO;
    M.G = L.N / L.g;
    M.g_log2 = ilog2(L.g);
    M.sg_log2 = ilog2(L.sg);
    M.rb_full = mt::CBS * mt::slice_bytes(L.bits, L.g);
    M.runs_uniform = 1;
    return M;
  }
  M.nquads = L.K / 4;
  M.nqp = (M.nquads + 7) / 8 * 8;
  M.nchunks = L.N / fmt_wc(L.bits);
  M.ncb = (M.nchunks + 31) / 32;
  if (L.bits <= 4) {
    M.G = L.N / L.g;
    M.g_log2 = ilog2(L.g);
    M.sg_log2 = ilog2(L.sg);
  }
  M.rb_full = rec_bytes(L.bits, 32, M.g_log2, M.sg_log2);
  M.runs_uniform = L.runs_uniform;
  return M;
}

// tile a reference-layout matrix already resident on device into `dst`
int tile_device(const RefMat& R, const Layout& L, uint8_t* dst, cudaStream_t s) {
  CU(cudaMemsetAsync(dst, 0, L.rec, s));  // pad quads / pad bytes are zero
  const MatDev M = matdev_from(L, dst);
  launch_tile(R, M, dst, const_cast<__half2*>(M.zmeta), s);
  CU(cudaGetLastError());
  return MOE_OK;
}

RefMat refmat_of(const Layout& L) {
  RefMat R{};
  R.bits = L.bits;
  R.K = L.K;
  R.N = L.N;
  R.g = L.g;
  R.sg = L.sg;
  R.nruns = L.nruns;
  return R;
}

// upload a reference-layout matrix and tile it into `dst` (device, L.total() bytes)
int upload_and_tile(const moe_matrix* m, const Layout& L, uint8_t* dst, cudaStream_t s) {
  uint8_t* scratch = nullptr;
  const size_t cbytes = m->codes_len;
  size_t tot = cbytes + 16;
  if (L.bits <= 4) tot += m->n_groups + 16 + 2 * (2 * m->n_zruns + m->n_scales) + 64;
  CU(cudaMalloc(&scratch, tot));
  uint8_t* p = scratch;
  RefMat R = refmat_of(L);
  CU(cudaMemcpyAsync(p, m->codes, cbytes, cudaMemcpyHostToDevice, s));
  R.codes = p;
  p += (cbytes + 15) & ~size_t(15);
  if (L.bits <= 4) {
    CU(cudaMemcpyAsync(p, m->zeros, m->n_groups, cudaMemcpyHostToDevice, s));
    R.zeros = p;
    p += (m->n_groups + 15) & ~int64_t(15);
    CU(cudaMemcpyAsync(p, m->zero_scales, 2 * m->n_zruns, cudaMemcpyHostToDevice, s));
    R.zs = reinterpret_cast<const uint16_t*>(p);
    p += (2 * m->n_zruns + 15) & ~int64_t(15);
    CU(cudaMemcpyAsync(p, m->zero_offsets, 2 * m->n_zruns, cudaMemcpyHostToDevice, s));
    R.zo = reinterpret_cast<const uint16_t*>(p);
    p += (2 * m->n_zruns + 15) & ~int64_t(15);
    CU(cudaMemcpyAsync(p, m->scales, 2 * m->n_scales, cudaMemcpyHostToDevice, s));
    R.scales = reinterpret_cast<const uint16_t*>(p);
  }
  int rc = tile_device(R, L, dst, s);
  CU(cudaStreamSynchronize(s));
  CU(cudaFree(scratch));
  return rc;
}

struct CopyRec {
  cudaEvent_t a, b;
  int64_t bytes;
};

// cuStreamWriteValue32 resolved through the runtime (no link-time libcuda
// dependency, so the library loads on hosts without a driver).
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_writeValue32 write_value32() {
  static PFN_writeValue32 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_writeValue32>(p);
  }
  return fn;
}

}  // namespace

// pinned readback block of finish_call: the device error words, the event
// count of the call and the head of its event log (one token's worth)
#define MOE_HSTAT_EV 1024
struct HostStatus {
  int err[8];
  int nev;
  int pad[3];
  moe_event ev[MOE_HSTAT_EV];
};

struct moe_engine {
  moe_model_desc md{};
  moe_cache_cfg cc{};
  moe_spec_cfg sc{};
  int dev = 0;
  bool rec_hidden = true;
  cudaStream_t s_comp = nullptr, s_copy = nullptr, s_copy2 = nullptr;  // copy: demand, spec
  int attn_bits = 0, expert_bits = 0, lm_bits = 0;
  int d = 0, f = 0, V = 0, L = 0, E = 0, H = 0, hd = 0, T = 0, topk = 0;

  // dense weights
  void* wte = nullptr;
  void* wpe = nullptr;
  int emb_half = -1;
  DevMat lm_head;
  std::vector<DevMat> wq, wk, wv, wo;
  std::vector<float*> ln1g, ln1b, ln2g, ln2b, gate;
  std::vector<__half*> gate_h;  // exact fp16 copies of the gates (null if not exact)
  float *lnfg = nullptr, *lnfb = nullptr;
  std::vector<bool> have;  // named tensor presence

  // experts
  Layout xl[3];
  bool xl_set = false;
  size_t xoff[3][4] = {};  // per matrix: rec, scales, zeros, zmeta offsets in a buffer
  size_t xbytes = 0, slot_stride = 0;
  uint8_t* arena = nullptr;
  // expert parallel (moe_ep_configure): this rank owns experts e with
  // e * world / E == rank in every layer; the arena holds only those
  int ep_rank = 0, ep_world = 1;
  std::vector<int> arena_idx;          // layer*E + expert -> arena slot, -1 not owned
  int n_owned = 0;
  uint8_t* owned_dev = nullptr;        // [L][E] mask for the device store
  uint8_t* xch = nullptr;              // exchange block: recv [2][topk][N][d] f32, flags [N], seq
  float* xrecv = nullptr;
  unsigned long long *xflag = nullptr, *xseq = nullptr;
  float* peer_recv[MOE_EP_MAX] = {};
  unsigned long long* peer_flag[MOE_EP_MAX] = {};
  std::vector<void*> ipc_opened;
  bool ep_connected = false;
  // NCCL transport (moe_ep_connect_nccl): one ncclAllGather of the slot
  // buffers per layer and position on the compute stream (graph-captured)
  bool ep_nccl = false;
  ncclComm_t nccl_comm = nullptr;
  float* nrecv = nullptr;  // [N][topk][d] all-gather output (rank-major)
  size_t arena_off(int l, int x) const { return (size_t)arena_idx[(size_t)l * E + x] * xbytes; }
  bool owns(int l, int x) const { return arena_idx[(size_t)l * E + x] >= 0; }
  std::vector<bool> loaded;
  uint8_t* pool = nullptr;
  uint32_t* flags = nullptr;
  int nbuf = 0;

  // activations
  float *x = nullptr, *h = nullptr, *xn = nullptr, *ctx = nullptr, *logits = nullptr;
  unsigned int tok_seq = 0;  // decode tokens issued (DecodeState.seq)
  bool pend_comb = false;  // decode: layer l's combine + LN1(l+1) is fused into QKV(l+1)
  bool pend_qkv_reset = false;  // Q/K/V sums read by the fused attention, reset by W2
  // fixed-point split-K sums (reduce == 2)
  unsigned long long *wo_acc = nullptr, *dn_acc = nullptr, *qkv_acc = nullptr;
  float *qkv_part = nullptr, *wo_part = nullptr, *up_part = nullptr, *dn_part = nullptr,
        *lm_part = nullptr;  // split-K partials
  float *qkv_out = nullptr, *wo_out = nullptr, *up_out = nullptr, *dn_out = nullptr;  // finals
  int* cnt = nullptr;  // split-K arrival counters
  int S_qkv = 1, S_wo = 1, S_up = 1, S_dn = 1, S_lm = 1;   // splits of the quad range
  int Q_qkv = 8, Q_wo = 8, Q_up = 8, Q_dn = 8, Q_lm = 8;   // quads per split
  float *kc = nullptr, *vc = nullptr;
  RouteRec* route = nullptr;
  TraceRecDev* trace = nullptr;
  float* trace_hidden = nullptr;
  int* tok_dev = nullptr;
  int* tok_hist = nullptr;
  int* tok_in = nullptr;
  float* cand_val = nullptr;
  int* cand_idx = nullptr;
  unsigned int* counter = nullptr;
  int* err = nullptr;

  // store
  StoreDev st{};
  void* st_mem = nullptr;
  Mailbox* mb_host = nullptr;
  Mailbox* mb_dev = nullptr;
  int ev_cap = 0;

  // copy engine
  std::thread copier;
  std::atomic<bool> stop{false};
  std::mutex cmu;
  std::vector<CopyRec> copies;
  int64_t n_copies = 0, copy_bytes = 0;
  double busy_ms = 0, peak_gbs = 0;
  std::vector<cudaEvent_t> free_events;

  // session
  int pos = 0;
  bool has_logits = false;
  bool finalized = false;
  std::vector<moe_event> events;
  int64_t launches = 0;
  double last_ms = 0;
  unsigned long long wait_ns = 60000000000ull;
  bool debug = false;
  bool serial_copies = false;  // MOE_SERIAL_COPIES=1
  bool trace_copies = false;   // MOE_COPY_TRACE=1: copier log on stderr
  bool pdl = true;             // programmatic dependent launch (MOE_PDL=0 disables)
  bool use_graph = true;       // one CUDA graph per decode token (MOE_GRAPH=0 disables)
  bool attn_fused = true;      // decode attention in the Wo GEMV prologue (MOE_ATTN_FUSED=0)
  bool copy_park = true;       // park speculative copies of passed layers (MOE_COPY_PARK=0)
  bool capturing = false;
  cudaGraphExec_t gexec = nullptr;
  int64_t graph_launches = 0;
  cudaEvent_t tok_ev[4] = {};
  DecodeState* ds_dev = nullptr;        // device decode cursor
  DecodeState* ds_host = nullptr;       // pinned staging for the cursor
  HostStatus* hstat = nullptr;          // pinned: status words + event-log head
  float* logits_h = nullptr;            // pinned logits of the last position
  const DecodeState* cur_ds = nullptr;  // non-null while enqueuing a decode token
  std::atomic<uint64_t> copier_tail{0};   // mailbox entries fully copied (serial mode)
  size_t copy_chunk = 2u << 20;           // speculative H2D chunk (demand copies go whole)
  // run-ahead bound: the host may enqueue at most `ahead` units (one layer of
  // one position) beyond the oldest unfinished one, so the launch queue never
  // fills while a kernel waits for the copy engine.
  std::vector<cudaEvent_t> ring;
  int64_t units_issued = 0, units_done = 0;
  int ahead = 3;
  int throttle();
  int unit_done();
  // per-class GEMV timing with CUDA events on the compute stream (profiling)
  enum { K_QKV = 0, K_WO, K_UP, K_DOWN, K_LM, K_N };
  bool prof = false;
  unsigned long long prof_hold_ns = 40000;
  std::vector<cudaEvent_t> pev;  // pairs
  std::vector<int> pcls;
  size_t pused = 0;
  double prof_ms[K_N] = {};
  int64_t prof_cnt[K_N] = {};
  void prof_begin(int c) {
    if (!prof) return;
    if (pused + 2 > pev.size()) {
      const size_t old = pev.size();
      pev.resize(old + 256);
      pcls.resize(pev.size() / 2);
      for (size_t i = old; i < pev.size(); ++i) cudaEventCreate(&pev[i]);
    }
    pcls[pused / 2] = c;
    launch_hold(prof_hold_ns, s_comp);  // stream busy while the host enqueues the span
    cudaEventRecord(pev[pused], s_comp);
  }
  void prof_end(int) {
    if (!prof) return;
    cudaEventRecord(pev[pused + 1], s_comp);
    pused += 2;
  }
  void prof_collect() {
    for (size_t i = 0; i < pused; i += 2) {
      float ms = 0;
      cudaEventElapsedTime(&ms, pev[i], pev[i + 1]);
      prof_ms[pcls[i / 2]] += ms;
      prof_cnt[pcls[i / 2]] += 1;
    }
    pused = 0;
  }
  int dbg(const char* what, int l, int p);
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  size_t dev_bytes = 0;

  ~moe_engine();
  template <class T>
  int dalloc(T** p, size_t n) {
    CU(cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T)));
    CU(cudaMemset(*p, 0, n * sizeof(T)));
    dev_bytes += n * sizeof(T);
    return MOE_OK;
  }
  int run_copier();
  // batched prefill (tensor-core layout, one GPU): buffers for PB positions
  int PB = 0;
  float *pf_xn = nullptr, *pf_ctx = nullptr, *pf_up = nullptr, *pf_q = nullptr;
  unsigned long long *pf_qkv_acc = nullptr, *pf_wo_acc = nullptr, *pf_dn_acc = nullptr;
  int2* pf_cols = nullptr;       // device: [PB] identity, then up / down column tables
  int2* pf_cols_h = nullptr;     // pinned staging of the expert column tables
  RouteRec* pf_route_h = nullptr;  // pinned: the layer's routes (read after bookkeeping)
  bool batched_prefill_ok(int n) const;
  int prefill_alloc();
  int prefill_batched(int n);
  int enq_attention(int l, int p, int mode);
  int enq_experts(int l, int p);
  int enq_logits(int p, float* out);
  int enq_token();
  int run_tokens(int n);
  int finish_call(bool want_logits = false);
  int bad_pos = -1;  // set by finish_call: first position that raised a non-finite error
  GJob dense_job(const DevMat& D, const float* x, float* part, float* out, int qps) const;
  int site_of(int l, int kind) const { return 1 + 8 * l + kind; }  // timeline slots
  TimelineSlot* timeline = nullptr;
};

moe_engine::~moe_engine() {
  stop.store(true);
  if (copier.joinable()) copier.join();
  if (s_copy) cudaStreamSynchronize(s_copy);
  if (s_copy2) cudaStreamSynchronize(s_copy2);
  if (s_comp) cudaStreamSynchronize(s_comp);
  for (auto& c : copies) {
    cudaEventDestroy(c.a);
    cudaEventDestroy(c.b);
  }
  for (auto e : free_events) cudaEventDestroy(e);
  for (auto e : ring) cudaEventDestroy(e);
  for (auto e : pev) cudaEventDestroy(e);
  for (auto e : tok_ev)
    if (e) cudaEventDestroy(e);
  if (gexec) cudaGraphExecDestroy(gexec);
  if (timeline) {
    set_timeline(nullptr, 0);
    cudaFree(timeline);
  }
  if (ds_host) cudaFreeHost(ds_host);
  if (hstat) cudaFreeHost(hstat);
  if (logits_h) cudaFreeHost(logits_h);
  void* ptrs[] = {wte, wpe, lm_head.mem, lnfg, lnfb, pool, flags, x, h, xn, ctx, logits,
                  qkv_part, wo_part, up_part, dn_part, lm_part, wo_acc, dn_acc, qkv_acc, qkv_out, wo_out, up_out, dn_out,
                  cnt, kc, vc, route, trace,
                  trace_hidden, tok_dev, tok_hist, tok_in, cand_val, cand_idx, counter, err,
                  st_mem, ds_dev};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto* v : {&wq, &wk, &wv, &wo})
    for (auto& m : *v)
      if (m.mem) cudaFree(m.mem);
  for (auto* v : {&ln1g, &ln1b, &ln2g, &ln2b, &gate})
    for (auto p : *v)
      if (p) cudaFree(p);
  for (auto p : gate_h)
    if (p) cudaFree(p);
  if (arena) cudaFreeHost(arena);
  for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
  if (owned_dev) cudaFree(owned_dev);
  if (xch) cudaFree(xch);
  if (nccl_comm) nccl_api().destroy(nccl_comm);
  if (nrecv) cudaFree(nrecv);
  if (mb_host) cudaFreeHost(mb_host);
  if (t0) cudaEventDestroy(t0);
  if (t1) cudaEventDestroy(t1);
  for (void* p : {(void*)pf_xn, (void*)pf_ctx, (void*)pf_up, (void*)pf_q, (void*)pf_qkv_acc,
                  (void*)pf_wo_acc, (void*)pf_dn_acc, (void*)pf_cols})
    if (p) cudaFree(p);
  if (pf_cols_h) cudaFreeHost(pf_cols_h);
  if (pf_route_h) cudaFreeHost(pf_route_h);
  if (s_comp) cudaStreamDestroy(s_comp);
  if (s_copy) cudaStreamDestroy(s_copy);
  if (s_copy2) cudaStreamDestroy(s_copy2);
}

// The copy engine: drains the device mailbox in FIFO order.  Each request is
// one contiguous H2D copy of a whole expert (paper §3.3 contiguous buffers)
// from the pinned arena into an HBM buffer, then a stream write of the
// buffer's generation into its ready flag.
int moe_engine::run_copier() {
  cudaSetDevice(dev);
  struct Inflight {
    cudaEvent_t a, b;
    int64_t bytes;
    int buf;
  };
  CopySched sched;
  sched.init(nbuf, xbytes, copy_chunk, sc.lookahead);
  sched.park = copy_park;
  std::deque<Inflight> dq, sq;                    // demand / speculative stream chunks
  std::vector<cudaEvent_t> last_ev(nbuf, nullptr);  // last chunk issued to each buffer
  std::vector<cudaStream_t> last_stream(nbuf, nullptr);
  uint64_t tail = 0;
  int idle = 0;
  auto get_events = [&](cudaEvent_t& a, cudaEvent_t& b) {
    std::lock_guard<std::mutex> g(cmu);
    if (free_events.size() < 2) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
    } else {
      a = free_events.back();
      free_events.pop_back();
      b = free_events.back();
      free_events.pop_back();
    }
  };
  while (!stop.load(std::memory_order_acquire)) {
    bool work = false;
    // 1. drain the device mailbox into the scheduler (copy_sched.h): an entry
    //    is valid once its stamp equals its index + 1 (single 16-byte write)
    for (;;) {
      const CopyReq* slot = &mb_host->ring[tail % MOE_MAILBOX_CAP];
      if (__atomic_load_n(&slot->stamp, __ATOMIC_ACQUIRE) != (uint32_t)(tail + 1)) break;
      const CopyReq r = *const_cast<const CopyReq*>(slot);
      const int kind = (r.layer >> 24) & 0xff, layer = r.layer & 0xffffff;
      if (debug || trace_copies) {
        fprintf(stderr, "[moe-copy %.3f] req %llu kind %d buf %d key (%d,%d) gen %u\n",
                std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
                    .count(),
                (unsigned long long)tail, kind, req_buf(r), layer, req_expert(r), r.gen);
        fflush(stderr);
      }
      sched.on_request(kind, req_buf(r), layer, req_expert(r), r.gen);
      ++tail;
      work = true;
    }
    // 2. retire finished chunks (per stream, in order)
    for (auto* q : {&dq, &sq})
      while (!q->empty() && cudaEventQuery(q->front().b) == cudaSuccess) {
        std::lock_guard<std::mutex> g(cmu);
        const Inflight& c = q->front();
        copies.push_back({c.a, c.b, c.bytes});
        if (last_ev[c.buf] == c.b) last_ev[c.buf] = nullptr;
        q->pop_front();
        work = true;
      }
    // 3. demand copies on their own stream (<= 2 queued); speculative chunks
    //    on a second stream, one at a time and only while no demand copy is
    //    pending or running, so a demand copy never queues behind speculation
    auto issue = [&](const CopySched::Chunk& c, cudaStream_t st, std::deque<Inflight>& q) {
      const uint8_t* src = arena + arena_off(c.layer, c.expert) + c.off;
      uint8_t* dst = pool + (size_t)c.buf * slot_stride + c.off;
      // a chunk to this buffer still in flight on the other stream lands first
      if (last_ev[c.buf] && last_stream[c.buf] != st &&
          cudaEventQuery(last_ev[c.buf]) != cudaSuccess)
        cudaStreamWaitEvent(st, last_ev[c.buf], 0);
      Inflight f;
      get_events(f.a, f.b);
      f.bytes = (int64_t)c.bytes;
      f.buf = c.buf;
      cudaEventRecord(f.a, st);
      nvtxMarkA(c.last ? "copy chunk (last)" : "copy chunk");
      cudaMemcpyAsync(dst, src, c.bytes, cudaMemcpyHostToDevice, st);
      cudaEventRecord(f.b, st);
      last_ev[c.buf] = f.b;
      last_stream[c.buf] = st;
      if (c.last)  // whole expert landed: publish its generation
        write_value32()(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(flags + c.buf),
                        c.gen, CU_STREAM_WRITE_VALUE_DEFAULT);
      if (debug || trace_copies) {
        fprintf(stderr, "[moe-copy %.3f] %s chunk buf %d gen %u off %zu bytes %zu last %d\n",
                std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
                    .count(),
                st == s_copy ? "demand" : "spec", c.buf, c.gen, c.off, c.bytes, (int)c.last);
        fflush(stderr);
      }
      q.push_back(f);
      work = true;
    };
    CopySched::Chunk c;
    while (dq.size() < 2 && sched.next_demand(&c)) issue(c, s_copy, dq);
    if (dq.empty() && sq.empty() && !sched.has_demand() && sched.next_spec(&c))
      issue(c, s_copy2, sq);
    const bool idle_now = dq.empty() && sq.empty() && sched.empty();
    if (idle_now) copier_tail.store(tail, std::memory_order_release);
    if (!work) {
      if (++idle > 20000) std::this_thread::yield();
#if defined(__x86_64__)
      __builtin_ia32_pause();
#endif
    } else {
      idle = 0;
    }
  }
  return MOE_OK;
}

GJob moe_engine::dense_job(const DevMat& D, const float* xin, float* part, float* out,
                          int qps) const {
  GJob j{};
  j.M = D.M;
  j.rel_slot = -1;
  j.xmode = X_PLAIN;
  j.x = xin;
  j.part = part;
  j.out = out;
  j.reduce = 1;
  j.QPS = qps;
  j.S = (D.M.nqp + qps - 1) / qps;
  return j;
}

// block offsets of the jobs; returns the grid size
static int finalize_launch(GLaunch& P) {
  int blk = 0;
  for (int i = 0; i < P.nj; ++i) {
    P.j[i].blk0 = blk;
    blk += P.j[i].M.ncb * P.j[i].S * (P.j[i].ncg > 1 ? P.j[i].ncg : 1);
  }
  return blk;
}

int moe_engine::enq_attention(int l, int p, int mode) {
  throttle();
  float* xp = x + (size_t)p * d;
  float* hp = h + (size_t)p * d;
  const bool pl = pdl && !prof;
  if (!cur_ds)  // decode: LN1 is fused into the embed / previous combine kernel
    launch_layernorm(xp, ln1g[l], ln1b[l], xn, d, s_comp, pl);
  dbg("ln1", l, p);
  GLaunch q{};
  q.nj = 3;
  q.cnt = cnt;
  q.site = site_of(l, 0);
  q.j[0] = dense_job(wq[l], xn, qkv_part, qkv_out, Q_qkv);
  q.j[1] = dense_job(wk[l], xn, qkv_part + (size_t)S_qkv * d, qkv_out + d, Q_qkv);
  q.j[2] = dense_job(wv[l], xn, qkv_part + (size_t)2 * S_qkv * d, qkv_out + 2 * d, Q_qkv);
  q.err = err;
  for (int i = 0; i < 3; ++i) {  // fixed-point sums, read (and reset) by the attention
    q.j[i].reduce = 2;
    q.j[i].acc = qkv_acc + (size_t)i * d;
  }
  if (pend_comb) {  // previous layer's combine + this layer's LN1 in the QKV prologue
    q.route = route + p;
    for (int i = 0; i < 3; ++i) {
      GJob& J = q.j[i];
      J.xmode = X_COMBINE;
      J.x = h + (size_t)p * d;
      J.cacc = dn_acc;
      J.ctop = topk;
      J.lng = ln1g[l];
      J.lnb = ln1b[l];
      J.xout = xp;
    }
  }
  const int nq = finalize_launch(q);
  prof_begin(K_QKV);
  launch_gemv(attn_bits, q, nq, s_comp, pdl && !prof);
  prof_end(K_QKV);
  dbg("qkv", l, p);
  // decode attention fused into the Wo GEMV's prologue (each Wo CTA computes its
  // head dims of the context) when a CTA's input rows lie inside one head
  const int wo_rows = Q_wo * mt::KS;
  const bool fuse_attn = attn_fused && wo[l].M.mma && hd % 128 == 0 && wo_rows <= hd &&
                         hd % wo_rows == 0 && q.j[0].reduce == 2;
  // the fused attention reads the Q/K/V sums; decode: this layer's W2 GEMV resets
  // them, a slice per CTA; per-position prefill: the tail (the next position's
  // QKV GEMV adds into them before any W2 runs)
  pend_qkv_reset = fuse_attn && cur_ds;
  if (!fuse_attn) {
  AttnParams a{};
  a.qkv_part = qkv_part;
  a.S = S_qkv;
  a.acc = q.j[0].reduce == 2 ? qkv_acc : nullptr;
  a.kc = kc + (size_t)l * T * d;
  a.vc = vc + (size_t)l * T * d;
  a.ctx = ctx;
  a.ds = cur_ds;
  a.site = site_of(l, 1);
  a.pos = p;
  a.H = H;
  a.hd = hd;
  a.d = d;
  a.T_max = T;
  launch_attention(a, s_comp, pl);
  dbg("attn", l, p);
  }
  GLaunch o{};
  o.nj = 1;
  o.cnt = cnt;
  o.site = site_of(l, 2);
  o.err = err;
  o.j[0] = dense_job(wo[l], ctx, wo_part, wo_out, Q_wo);
  o.j[0].reduce = 2;  // fixed-point split-K sums, read (and reset) by the tail
  o.j[0].acc = wo_acc;
  if (fuse_attn) {
    o.j[0].xmode = X_ATTN;
    o.att_acc = qkv_acc;
    o.att_kc = kc + (size_t)l * T * d;
    o.att_vc = vc + (size_t)l * T * d;
    o.att_ds = cur_ds;
    o.att_pos = p;
    o.att_hd = hd;
    o.att_T = T;
  }
  const int no = finalize_launch(o);
  prof_begin(K_WO);
  launch_gemv(attn_bits, o, no, s_comp, pdl && !prof);
  prof_end(K_WO);
  dbg("wo", l, p);
  TailParams t{};
  t.x = xp;
  t.part = wo_out;
  t.S = 1;
  t.acc = o.j[0].reduce == 2 ? wo_acc : nullptr;
  t.g2 = ln2g[l];
  t.b2 = ln2b[l];
  t.gate_l = gate[l];
  const int gl = l + sc.lookahead;
  const bool guess = mode == 0 && sc.enabled && sc.m > 0 && gl < L;
  t.gate_g = guess ? gate[gl] : nullptr;
  t.gh_l = gate_h[l];
  t.gh_g = guess ? gate_h[gl] : nullptr;
  t.guess_layer = guess ? gl : -1;
  t.m = guess ? sc.m : 0;
  t.h = hp;
  t.route = route + p;
  t.trace = trace;
  t.trace_hidden = rec_hidden ? trace_hidden : nullptr;
  t.ds = cur_ds;
  t.n_layers = L;
  t.site = site_of(l, 3);
  t.st = st;
  t.d = d;
  t.E = E;
  t.top_k = topk;
  t.layer = l;
  t.pos = p;
  t.mode = mode;
  t.ep_size = 1;
  if (fuse_attn && !cur_ds) {
    t.zero = qkv_acc;
    t.zero_n = 3 * d;
  }
  if (tail_smem_bytes(t) > 226 * 1024) t.gh_l = t.gh_g = nullptr;  // gates too big to stage
  launch_tail(t, s_comp, pl);
  dbg("tail", l, p);
  unit_done();
  return MOE_OK;
}

int moe_engine::enq_experts(int l, int p) {
  throttle();
  GLaunch u{};
  u.route = route + p;
  u.pool = pool;
  u.slot_stride = slot_stride;
  u.flags = flags;
  u.err = err;
  u.wait_ns = wait_ns;
  u.cnt = cnt;
  u.site = site_of(l, 4);
  GLaunch dn = u;
  dn.site = site_of(l, 5);
  for (int j = 0; j < topk; ++j) {
    for (int m = 0; m < 2; ++m) {
      GJob& J = u.j[2 * j + m];
      J = GJob{};
      J.M = matdev_from(xl[m], reinterpret_cast<const uint8_t*>(xoff[m][0]));
      J.M.zmeta = reinterpret_cast<const __half2*>(xoff[m][3]);
      J.M.scl = reinterpret_cast<const __half*>(xoff[m][1]);
      J.rel_slot = j;
      J.xmode = X_PLAIN;
      J.x = h + (size_t)p * d;
      J.part = up_part + ((size_t)(2 * j + m) * S_up) * f;
      J.out = up_out + (size_t)(2 * j + m) * f;
      // split-K partials, bulk-copied and summed in order by the down GEMV's
      // SwiGLU prologue (fewer atomics than fixed-point sums for 5 splits)
      J.reduce = 0;
      J.QPS = Q_up;
      J.S = S_up;
    }
    GJob& J = dn.j[j];
    J = GJob{};
    J.M = matdev_from(xl[2], reinterpret_cast<const uint8_t*>(xoff[2][0]));
    J.M.zmeta = reinterpret_cast<const __half2*>(xoff[2][3]);
    J.M.scl = reinterpret_cast<const __half*>(xoff[2][1]);
    J.rel_slot = j;
    J.xmode = X_SWIGLU;
    J.up1 = up_part + (size_t)(2 * j) * S_up * f;
    J.up3 = up_part + (size_t)(2 * j + 1) * S_up * f;
    J.xstride = f;
    J.part = dn_part + ((size_t)j * S_dn) * d;
    J.out = dn_out + (size_t)j * d;
    // single GPU: fixed-point split-K sums read (and reset) by the combine;
    // expert parallel: reduced in-kernel, the exchange ships dn_out
    J.reduce = (ep_world > 1 || ep_nccl) ? 1 : 2;
    J.acc = dn_acc + (size_t)j * d;
    J.QPS = Q_dn;
    J.S = S_dn;
  }
  u.nj = 2 * topk;
  dn.nj = topk;
  if (pend_qkv_reset) {  // the fused attention (Wo prologue) read them: reset, a slice per CTA
    dn.zero = qkv_acc;
    dn.zero_n = 3 * d;
    pend_qkv_reset = false;
  }
  if (pend_comb) {  // the fused combine read dn_acc: reset it before W2 adds
    u.zero = dn_acc;
    u.zero_n = topk * d;
  }
  pend_comb = false;
  const int nu = finalize_launch(u);
  const int ndn = finalize_launch(dn);
  for (int j = 0; j < topk; ++j) dn.j[j].xS = S_up;
  if (serial_copies) {  // ncu / debugging: the host drains the mailbox before the GEMV
    CU(cudaStreamSynchronize(s_comp));
    {  // entries posted so far = device-side head (seq[1])
      long long posted = 0;
      CU(cudaMemcpy(&posted, st.seq + 1, sizeof(posted), cudaMemcpyDeviceToHost));
      while ((long long)copier_tail.load(std::memory_order_acquire) < posted)
        std::this_thread::yield();
    }
    CU(cudaStreamSynchronize(s_copy));
  }
  if (prof)  // keep copy waits out of the GEMV's event-timed span
    launch_wait_ready(route + p, topk, flags, err, wait_ns, s_comp);
  prof_begin(K_UP);
  launch_gemv(expert_bits, u, nu, s_comp, pdl && !prof);
  prof_end(K_UP);
  dbg("up", -1, p);
  // expert parallel over peer memory: the exchange is fused into the down
  // GEMV (tensor-core layout; the CUDA-core layout keeps k_exchange)
  const bool epx = ep_world > 1 && !ep_nccl && dn.j[0].M.mma != 0;
  if (epx) {
    dn.ep_n = ep_world;
    dn.ep_rank = ep_rank;
    dn.ep_topk = topk;
    dn.ep_seq = xseq;
    for (int r = 0; r < ep_world; ++r) {
      dn.ep_recv[r] = peer_recv[r];
      dn.ep_flag[r] = peer_flag[r];
    }
  }
  prof_begin(K_DOWN);
  launch_gemv(expert_bits, dn, ndn, s_comp, pdl && !prof);
  prof_end(K_DOWN);
  dbg("down", -1, p);
  CombineParams c{};
  c.h = h + (size_t)p * d;
  c.part = dn_out;
  c.S = 1;
  c.acc = dn.j[0].reduce == 2 ? dn_acc : nullptr;
  if (ep_nccl) {  // NCCL transport: all-gather of the slot buffers (rank-major)
    const ncclResult_t r = nccl_api().all_gather(dn_out, nrecv, (size_t)topk * d, ncclFloat32,
                                                 nccl_comm, s_comp);
    if (r != ncclSuccess) return fail(MOE_ERR_CUDA, std::string("ncclAllGather: ") +
                                                        nccl_api().error_string(r));
    c.part = nrecv;
    c.S = ep_world;
    c.rank_major = 1;
  } else if (epx) {  // the down GEMV stored the slots into every rank's receive buffer
    c.part = xrecv;
    c.S = ep_world;
    c.ep_seq = xseq;
    c.ep_seq_w = xseq;
    c.ep_flags = xflag;
    c.ep_ncbt = (long long)topk * dn.j[0].M.ncb;
    c.ep_slab = (long long)topk * ep_world * d;
    c.err = err;
    c.wait_ns = wait_ns;
  } else if (ep_world > 1) {  // sum-exchange of the slot buffers over peer memory
    ExchangeParams xp{};
    xp.src = dn_out;
    for (int r = 0; r < ep_world; ++r) {
      xp.recv[r] = peer_recv[r];
      xp.flag[r] = peer_flag[r];
    }
    xp.seq = xseq;
    xp.my_flag = xflag;
    xp.rank = ep_rank;
    xp.N = ep_world;
    xp.top_k = topk;
    xp.d = d;
    xp.err = err;
    xp.wait_ns = wait_ns;
    xp.site = site_of(l, 7);
    launch_exchange(xp, s_comp, pdl && !prof);
    c.part = xrecv;
    c.S = ep_world;
    c.ep_seq = xseq;
    c.ep_slab = (long long)topk * ep_world * d;
  }
  c.route = route + p;
  c.out = x + (size_t)p * d;
  c.d = d;
  c.top_k = topk;
  c.site = site_of(l, 6);
  if (cur_ds) {  // decode: fuse the next LayerNorm (LN1 of l+1, or LN_f)
    c.ln_g = l + 1 < L ? ln1g[l + 1] : lnfg;
    c.ln_b = l + 1 < L ? ln1b[l + 1] : lnfb;
    c.xn = xn;
  }
  if (cur_ds && ep_world == 1 && !ep_nccl && c.acc && l + 1 < L) {
    pend_comb = true;  // QKV(l+1) forms the residual and LN1 itself
  } else {
    launch_combine(c, s_comp, pdl && !prof);
    dbg("combine", -1, p);
  }
  unit_done();
  return MOE_OK;
}

// ---------------------------------------------------------------- batched prefill
// The reference encodes a prompt layer by layer (model.py:343-367): attention
// of every position, the gates, one store resolution of the layer
// (engine.py:233-240: each distinct expert acquired once), then every
// position's MoE.  On B200 every weight byte of a layer is streamed once per
// group of MG_PREFILL_COLS positions: the Q/K/V and Wo GEMVs take the
// positions as input columns, and the expert GEMVs take, per distinct routed
// expert, the (position, slot) pairs that chose it.  Each column is computed
// exactly like the decode kernel computes it (same split geometry and
// fixed-point sums), so prefill equals teacher-forced decode bit for bit.
bool moe_engine::batched_prefill_ok(int n) const {
  if (ep_world > 1 || ep_nccl || !xl_set) return false;
  int min_n = 4;  // shorter prompts: the per-position path is faster (profiles/r2_prefill.md)
  if (const char* v = getenv("MOE_PREFILL_BATCH")) {
    if (atoi(v) == 0) return false;
    min_n = 1;  // forced on (tests)
  }
  if (n < min_n) return false;
  if (attn_bits > 4 || expert_bits > 4) return false;
  for (int l = 0; l < L; ++l)
    if (!wq[l].M.mma || !wk[l].M.mma || !wv[l].M.mma || !wo[l].M.mma) return false;
  for (int m = 0; m < 3; ++m)
    if (!matdev_from(xl[m], nullptr).mma) return false;
  return true;
}

int moe_engine::prefill_alloc() {
  if (PB) return MOE_OK;
  const int pb = std::min(T, 64);
  int rc;
  if ((rc = dalloc(&pf_xn, (size_t)pb * d))) return rc;
  if ((rc = dalloc(&pf_ctx, (size_t)pb * d))) return rc;
  if ((rc = dalloc(&pf_q, (size_t)pb * d))) return rc;
  if ((rc = dalloc(&pf_up, (size_t)pb * topk * 2 * S_up * f))) return rc;
  if ((rc = dalloc(&pf_qkv_acc, (size_t)pb * 3 * d))) return rc;
  if ((rc = dalloc(&pf_wo_acc, (size_t)pb * d))) return rc;
  if ((rc = dalloc(&pf_dn_acc, (size_t)pb * topk * d))) return rc;
  if ((rc = dalloc(&pf_cols, (size_t)pb * (1 + 2 * topk)))) return rc;
  // one staging region per chunk: a chunk's tables are still being copied
  // (async, stream order) while the host fills the next chunk's
  const int nchunk = (T + pb - 1) / pb;
  CU(cudaHostAlloc(&pf_cols_h, (size_t)nchunk * pb * 2 * topk * sizeof(int2),
                   cudaHostAllocDefault));
  CU(cudaHostAlloc(&pf_route_h, (size_t)T * sizeof(RouteRec), cudaHostAllocDefault));
  std::vector<int2> id(pb);
  for (int i = 0; i < pb; ++i) id[i] = make_int2(i, i);
  CU(cudaMemcpy(pf_cols, id.data(), pb * sizeof(int2), cudaMemcpyHostToDevice));
  PB = pb;
  return MOE_OK;
}

int moe_engine::prefill_batched(int n) {
  int rc = prefill_alloc();
  if (rc) return rc;
  const int NCc = MG_PREFILL_COLS;
  auto dense_cols = [&](GJob& J, int nc, long long xcs, long long ocs) {
    J.cols = pf_cols;
    J.ncol = nc;
    J.ncg = (nc + NCc - 1) / NCc;
    J.xcs = xcs;
    J.ocs = ocs;
  };
  int2* up_cols = pf_cols + PB;
  int2* dn_cols = up_cols + (size_t)PB * topk;
  for (int l = 0; l < L; ++l) {
    // ---- attention of every position, chunk by chunk
    for (int c0 = 0; c0 < n; c0 += PB) {
      const int nc = std::min(PB, n - c0);
      launch_layernorm_rows(x + (size_t)c0 * d, ln1g[l], ln1b[l], pf_xn, d, nc, s_comp);
      GLaunch q{};
      q.nj = 3;
      q.cnt = cnt;
      q.site = -1;
      q.err = err;
      const DevMat* W[3] = {&wq[l], &wk[l], &wv[l]};
      for (int i = 0; i < 3; ++i) {
        q.j[i] = dense_job(*W[i], pf_xn, qkv_part, qkv_out, Q_qkv);
        q.j[i].reduce = 2;
        q.j[i].acc = pf_qkv_acc + (size_t)i * d;
        dense_cols(q.j[i], nc, d, 3LL * d);
      }
      launch_gemv_cols(attn_bits, q, finalize_launch(q), s_comp);
      if (hd % 128 == 0) {  // all positions of the chunk in two launches
        AttnParams a{};
        a.acc = pf_qkv_acc;
        a.qbuf = pf_q;
        a.kc = kc + (size_t)l * T * d;
        a.vc = vc + (size_t)l * T * d;
        a.ctx = pf_ctx;
        a.site = -1;
        a.pos = c0;
        a.H = H;
        a.hd = hd;
        a.d = d;
        a.T_max = T;
        launch_attention_rows(a, nc, s_comp);
      } else {
        for (int i = 0; i < nc; ++i) {
          AttnParams a{};
          a.qkv_part = qkv_part;
          a.S = S_qkv;
          a.acc = pf_qkv_acc + (size_t)i * 3 * d;
          a.kc = kc + (size_t)l * T * d;
          a.vc = vc + (size_t)l * T * d;
          a.ctx = pf_ctx + (size_t)i * d;
          a.site = -1;
          a.pos = c0 + i;
          a.H = H;
          a.hd = hd;
          a.d = d;
          a.T_max = T;
          launch_attention(a, s_comp, false);
        }
      }
      GLaunch o{};
      o.nj = 1;
      o.cnt = cnt;
      o.site = -1;
      o.err = err;
      o.j[0] = dense_job(wo[l], pf_ctx, wo_part, wo_out, Q_wo);
      o.j[0].reduce = 2;
      o.j[0].acc = pf_wo_acc;
      dense_cols(o.j[0], nc, d, d);
      launch_gemv_cols(attn_bits, o, finalize_launch(o), s_comp);
      {
        TailParams t{};
        t.x = x + (size_t)c0 * d;
        t.part = wo_out;
        t.S = 1;
        t.acc = pf_wo_acc;
        t.g2 = ln2g[l];
        t.b2 = ln2b[l];
        t.gate_l = gate[l];
        t.gh_l = gate_h[l];
        t.guess_layer = -1;
        t.h = h + (size_t)c0 * d;
        t.route = route + c0;
        t.trace = trace;
        t.trace_hidden = rec_hidden ? trace_hidden : nullptr;
        t.n_layers = L;
        t.site = -1;
        t.st = st;
        t.d = d;
        t.E = E;
        t.top_k = topk;
        t.layer = l;
        t.pos = c0;
        t.mode = 1;
        t.ep_size = 1;
        if (tail_smem_bytes(t) > 226 * 1024) t.gh_l = t.gh_g = nullptr;
        launch_tail(t, s_comp, false, nc);  // one CTA per position
      }
      dbg("prefill attention", l, c0);
    }
    // ---- one store resolution of the layer (store.py acquire per distinct expert)
    PrefillBKParams pb{};
    pb.route = route;
    pb.st = st;
    pb.layer = l;
    pb.n = n;
    pb.top_k = topk;
    launch_prefill_bk(pb, s_comp);
    CU(cudaMemcpyAsync(pf_route_h, route, (size_t)n * sizeof(RouteRec), cudaMemcpyDeviceToHost,
                       s_comp));
    CU(cudaStreamSynchronize(s_comp));
    // ---- the experts, grouped by buffer (= distinct expert), chunk by chunk
    for (int c0 = 0; c0 < n; c0 += PB) {
      const int nc = std::min(PB, n - c0);
      int2* cols_h = pf_cols_h + (size_t)(c0 / PB) * PB * 2 * topk;
      std::vector<int> bufs;                 // distinct buffers in first-use order
      std::vector<std::vector<int2>> refs;   // per buffer: (position, slot)
      for (int i = 0; i < nc; ++i)
        for (int j = 0; j < topk; ++j) {
          const int b = pf_route_h[c0 + i].buf[j];
          if (b < 0) continue;  // error raised by the bookkeeping / not owned
          size_t k = 0;
          while (k < bufs.size() && bufs[k] != b) ++k;
          if (k == bufs.size()) {
            bufs.push_back(b);
            refs.emplace_back();
          }
          refs[k].push_back(make_int2(c0 + i, j));
        }
      // column tables: up (h row, slot column), down (slot column twice)
      std::vector<int> first(bufs.size());
      size_t ncols = 0;
      for (size_t k = 0; k < bufs.size(); ++k) {
        first[k] = (int)ncols;
        for (const int2& r : refs[k]) {
          const int q = (r.x - c0) * topk + r.y;
          cols_h[ncols] = make_int2(r.x, q);
          cols_h[(size_t)PB * topk + ncols] = make_int2(q, q);
          ++ncols;
        }
      }
      if (ncols) {
        CU(cudaMemcpyAsync(up_cols, cols_h, ncols * sizeof(int2), cudaMemcpyHostToDevice,
                           s_comp));
        CU(cudaMemcpyAsync(dn_cols, cols_h + (size_t)PB * topk, ncols * sizeof(int2),
                           cudaMemcpyHostToDevice, s_comp));
      }
      const long long upcs = 2LL * S_up * f;  // floats per (position, slot) of pf_up
      auto expert_job = [&](GJob& J, int m, size_t k) {
        J = GJob{};
        J.M = matdev_from(xl[m], reinterpret_cast<const uint8_t*>(xoff[m][0]));
        J.M.zmeta = reinterpret_cast<const __half2*>(xoff[m][3]);
        J.M.scl = reinterpret_cast<const __half*>(xoff[m][1]);
        J.rel_pos = refs[k][0].x;
        J.rel_slot = refs[k][0].y;
        J.ncol = (int)refs[k].size();
        J.ncg = (J.ncol + NCc - 1) / NCc;
      };
      // W1 || W3 (split-K partials), four experts per launch
      for (size_t k0 = 0; k0 < bufs.size(); k0 += MOE_GEMV_MAXJOBS / 2) {
        GLaunch u{};
        u.route = route;
        u.pool = pool;
        u.slot_stride = slot_stride;
        u.flags = flags;
        u.err = err;
        u.wait_ns = wait_ns;
        u.cnt = cnt;
        u.site = -1;
        for (size_t k = k0; k < std::min(bufs.size(), k0 + MOE_GEMV_MAXJOBS / 2); ++k)
          for (int m = 0; m < 2; ++m) {
            GJob& J = u.j[u.nj++];
            expert_job(J, m, k);
            J.xmode = X_PLAIN;
            J.x = h;
            J.xcs = d;
            J.cols = up_cols + first[k];
            J.part = pf_up + (size_t)m * S_up * f;
            J.ocs = upcs;
            J.reduce = 0;
            J.QPS = Q_up;
            J.S = S_up;
          }
        launch_gemv_cols(expert_bits, u, finalize_launch(u), s_comp);
      }
      // W2 with the SwiGLU prologue (fixed-point sums per (position, slot))
      for (size_t k0 = 0; k0 < bufs.size(); k0 += MOE_GEMV_MAXJOBS) {
        GLaunch dn{};
        dn.route = route;
        dn.pool = pool;
        dn.slot_stride = slot_stride;
        dn.flags = flags;
        dn.err = err;
        dn.wait_ns = wait_ns;
        dn.cnt = cnt;
        dn.site = -1;
        for (size_t k = k0; k < std::min(bufs.size(), k0 + MOE_GEMV_MAXJOBS); ++k) {
          GJob& J = dn.j[dn.nj++];
          expert_job(J, 2, k);
          J.xmode = X_SWIGLU;
          J.up1 = pf_up;
          J.up3 = pf_up + (size_t)S_up * f;
          J.xcs = upcs;
          J.xstride = f;
          J.xS = S_up;
          J.cols = dn_cols + first[k];
          J.acc = pf_dn_acc;
          J.ocs = d;
          J.reduce = 2;
          J.QPS = Q_dn;
          J.S = S_dn;
        }
        launch_gemv_cols(expert_bits, dn, finalize_launch(dn), s_comp);
      }
      {
        CombineParams c{};
        c.h = h + (size_t)c0 * d;
        c.part = dn_out;
        c.S = 1;
        c.acc = pf_dn_acc;
        c.route = route + c0;
        c.out = x + (size_t)c0 * d;
        c.d = d;
        c.top_k = topk;
        c.site = -1;
        launch_combine(c, s_comp, false, nc);  // grid.y = positions
      }
      dbg("prefill experts", l, c0);
    }
  }
  return MOE_OK;
}

int moe_engine::enq_logits(int p, float* out) {
  const bool pl = pdl && !prof;
  if (!cur_ds)  // decode: LN_f is fused into the last combine kernel
    launch_layernorm(x + (size_t)p * d, lnfg, lnfb, xn, d, s_comp, pl);
  GLaunch g{};
  g.nj = 1;
  g.cnt = cnt;
  g.site = 1 + 8 * L;
  g.j[0] = dense_job(lm_head, xn, lm_part, out, Q_lm);
  g.j[0].reduce = 0;  // the logits kernel sums the splits
  const int ng = finalize_launch(g);
  prof_begin(K_LM);
  launch_gemv(lm_bits, g, ng, s_comp, pl);
  prof_end(K_LM);
  LogitsParams lp{};
  lp.part = lm_part;
  lp.S = S_lm;
  lp.V = V;
  lp.logits = out;
  lp.cand_val = cand_val;
  lp.cand_idx = cand_idx;
  lp.counter = counter;
  lp.tok_out = tok_dev;
  lp.tok_hist = tok_hist;
  lp.ds = const_cast<DecodeState*>(cur_ds);
  lp.site = 2 + 8 * L;
  lp.err = err;
  launch_logits(lp, s_comp, pl);
  dbg("logits", -1, p);
  return MOE_OK;
}

// One decode token (embed -> L x (attention, experts) -> logits + argmax) with
// every position-dependent quantity read from the device cursor ds_dev, so
// the same launch sequence (and the same captured CUDA graph) serves any token.
int moe_engine::enq_token() {
  cur_ds = ds_dev;
  EmbedParams ep{};
  ep.wte = wte;
  ep.wpe = wpe;
  ep.half = emb_half;
  ep.ds = ds_dev;
  ep.d = d;
  ep.x = x;
  ep.ln_g = ln1g[0];
  ep.ln_b = ln1b[0];
  ep.xn = xn;
  ep.site = 0;
  launch_embed(ep, s_comp, pdl && !prof);
  for (int l = 0; l < L; ++l) {
    enq_attention(l, 0, 0);
    enq_experts(l, 0);
  }
  enq_logits(0, logits);
  cur_ds = nullptr;
  return MOE_OK;
}

// n decode tokens: one graph launch per token when graphs are enabled (the
// graph is captured on first use), else the eager launch sequence.  One token
// is in flight at a time so the launch queue never fills while a kernel waits
// for the copy engine (the copier thread must always be able to submit).
int moe_engine::run_tokens(int n) {
  const bool graphs = use_graph && !prof && !debug && !serial_copies;
  if (!graphs) {
    const long long c0 = launch_count();
    for (int i = 0; i < n; ++i) enq_token();
    launches += launch_count() - c0;
    return MOE_OK;
  }
  if (!gexec) {
    const long long c0 = launch_count();
    CU(cudaStreamBeginCapture(s_comp, cudaStreamCaptureModeThreadLocal));
    capturing = true;
    enq_token();
    capturing = false;
    cudaGraph_t g = nullptr;
    CU(cudaStreamEndCapture(s_comp, &g));
    CU(cudaGraphInstantiate(&gexec, g, 0));
    CU(cudaGraphDestroy(g));
    graph_launches = launch_count() - c0;
  }
  for (int i = 0; i < n; ++i) {
    // one token in flight: a graph launch never waits for queue space while a
    // GEMV spins on a copy the copier thread still has to submit
    if (i >= 1) CU(cudaEventSynchronize(tok_ev[(i - 1) % 4]));
    CU(cudaGraphLaunch(gexec, s_comp));
    CU(cudaEventRecord(tok_ev[i % 4], s_comp));
    launches += graph_launches;
  }
  return MOE_OK;
}

int moe_engine::throttle() {
  if (capturing) return MOE_OK;
  while (units_issued - units_done >= ahead) {
    CU(cudaEventSynchronize(ring[units_done % ring.size()]));
    ++units_done;
  }
  return MOE_OK;
}

int moe_engine::unit_done() {
  if (capturing) return MOE_OK;
  CU(cudaEventRecord(ring[units_issued % ring.size()], s_comp));
  ++units_issued;
  return MOE_OK;
}

// MOE_DEBUG=1: synchronize and report after every launch group
int moe_engine::dbg(const char* what, int l, int p) {
  if (!debug) return MOE_OK;
  cudaError_t ce = cudaStreamSynchronize(s_comp);
  int ev = 0, fl = 0;
  cudaMemcpy(&fl, err, 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&ev, st.scalars + 3, 4, cudaMemcpyDeviceToHost);
  fprintf(stderr, "[moe] %-10s layer %3d pos %3d : %s err=0x%x nev=%d mailbox=%llu\n", what, l, p,
          cudaGetErrorString(ce), fl, ev, 0ull);
  fflush(stderr);
  return ce == cudaSuccess ? MOE_OK : fail(MOE_ERR_CUDA, cudaGetErrorString(ce));
}

int moe_engine::finish_call(bool want_logits) {
  // one stream synchronisation per call: the status words, the first chunk
  // of the event log and (optionally) the logits come back with async copies
  // into pinned memory queued behind the work
  CU(cudaEventRecord(t1, s_comp));
  CU(cudaMemcpyAsync(hstat->err, err, sizeof(hstat->err), cudaMemcpyDeviceToHost, s_comp));
  CU(cudaMemcpyAsync(&hstat->nev, st.scalars + 3, sizeof(int), cudaMemcpyDeviceToHost, s_comp));
  CU(cudaMemcpyAsync(hstat->ev, st.ev, sizeof(hstat->ev), cudaMemcpyDeviceToHost, s_comp));
  if (want_logits)
    CU(cudaMemcpyAsync(logits_h, logits, (size_t)V * 4, cudaMemcpyDeviceToHost, s_comp));
  CU(cudaStreamSynchronize(s_comp));
  units_done = units_issued;
  prof_collect();
  CU(cudaGetLastError());
  float ms = 0;
  cudaEventElapsedTime(&ms, t0, t1);
  last_ms = ms;
  const int e = hstat->err[0];
  const int nev = hstat->nev;
  if (nev > 0) {
    const size_t old = events.size();
    events.resize(old + nev);
    const int nh = std::min(nev, (int)MOE_HSTAT_EV);
    memcpy(events.data() + old, hstat->ev, nh * sizeof(moe_event));
    if (nev > nh)
      CU(cudaMemcpy(events.data() + old + nh, st.ev + nh, (nev - nh) * sizeof(moe_event),
                    cudaMemcpyDeviceToHost));
    CU(cudaMemsetAsync(st.scalars + 3, 0, sizeof(int), s_comp));
  }
  if (e) {
    // the first position whose gate input (err[6]) or logits (err[7]) were not
    // finite: tokens before it completed (the reference raises inside that
    // token's forward pass), so the caller advances by exactly those
    bad_pos = -1;
    for (int i = 6; i < 8; ++i)
      if (hstat->err[i] > 0 && (bad_pos < 0 || hstat->err[i] - 1 < bad_pos)) bad_pos = hstat->err[i] - 1;
    CU(cudaMemsetAsync(err, 0, sizeof(int), s_comp));
    CU(cudaMemsetAsync(err + 6, 0, 2 * sizeof(int), s_comp));
    if (bad_pos >= 0) {  // events of later tokens (decoded past the error) are dropped
      size_t keep = events.size();
      while (keep > 0 && events[keep - 1].token_pos > bad_pos) --keep;
      events.resize(keep);
    }
  }
  if (e & MOE_ERRF_TIMEOUT) {
    int diag[8] = {0};
    memcpy(diag, hstat->err, sizeof(diag));
    const int buf = (int)(((uintptr_t)diag[4] - ((uintptr_t)flags & 0x7fffffff)) / 4);
    cudaMemset(err, 0, sizeof(diag));
    return fail(MOE_ERR_TIMEOUT, "expert buffer never became ready (buffer " +
                                     std::to_string(buf) + " waiting for generation " +
                                     std::to_string(diag[2]) + ", flag " +
                                     std::to_string(diag[3]) + ")");
  }
  if (e & (MOE_ERRF_ALLOC | MOE_ERRF_EVENTS))
    return fail(MOE_ERR_RUNTIME, "device store overflow (buffers or event log)");
  if (e & MOE_ERRF_UNKNOWN) return fail(MOE_ERR_UNKNOWN_EXPERT, "no such expert");
  if (e & MOE_ERRF_NONFINITE_GATE) return fail(MOE_ERR_NONFINITE, "gate input is not finite");
  if (e & MOE_ERRF_NONFINITE_LOGITS) return fail(MOE_ERR_NONFINITE, "output logits are not finite");
  return MOE_OK;
}

// ====================================================================== C ABI
extern "C" {

const char* moe_last_error(void) { return g_err.c_str(); }
int moe_engine_fail(int code, const char* msg) { return fail(code, msg); }

int moe_create(const moe_model_desc* md, const moe_cache_cfg* cc, const moe_spec_cfg* sc,
               int32_t device, int32_t record_hidden, moe_engine** out) {
  if (!md || !cc || !sc || !out) return fail(MOE_ERR_VALUE, "null argument");
  const int dims[] = {md->vocab_size, md->d_model, md->n_layers, md->n_heads,
                      md->d_ffn,      md->n_experts, md->top_k,  md->max_seq_len};
  for (int v : dims)
    if (v < 1) return fail(MOE_ERR_VALUE, "all model dimensions must be >= 1");
  if (md->d_model % md->n_heads) return fail(MOE_ERR_VALUE, "d_model must be divisible by n_heads");
  if (md->top_k > md->n_experts) return fail(MOE_ERR_VALUE, "top_k_gate cannot exceed n_experts");
  if (md->top_k > MOE_MAX_TOPK || md->n_experts > 16)
    return fail(MOE_ERR_VALUE, "engine supports top_k <= 4 and n_experts <= 16");
  if (cc->k < 0 || cc->b < 0 || cc->expert_bytes <= 0)
    return fail(MOE_ERR_VALUE, "k and b must be >= 0 and expert_bytes positive");
  if (cc->k > md->n_experts)
    return fail(MOE_ERR_VALUE, "k=" + std::to_string(cc->k) + " exceeds experts per layer");
  if (sc->m < 0) return fail(MOE_ERR_VALUE, "m must be >= 0");
  if (sc->lookahead < 1) return fail(MOE_ERR_VALUE, "lookahead must be >= 1");
  if (sc->enabled && sc->m > cc->b)
    return fail(MOE_ERR_VALUE, "m=" + std::to_string(sc->m) + " exceeds b=" +
                                   std::to_string(cc->b) + " staging buffers");
  auto* e = new moe_engine();
  e->md = *md;
  e->cc = *cc;
  e->sc = *sc;
  // top-m of E gate logits is at most E experts (engine.py:60-68 argsort[:m])
  e->sc.m = std::min(sc->m, md->n_experts);
  e->dev = device;
  e->rec_hidden = record_hidden != 0;
  if (const char* dbgv = getenv("MOE_DEBUG")) e->debug = atoi(dbgv) != 0;
  // Under a kernel-serialising tool (ncu, compute-sanitizer: both inject a
  // library through CUDA_INJECTION64_PATH) a GEMV spinning on the copy
  // engine's flag would never see it: the host then drains the copies before
  // each expert GEMV instead.  MOE_SERIAL_COPIES=0/1 overrides.
  e->serial_copies = getenv("CUDA_INJECTION64_PATH") != nullptr ||
                     getenv("NV_COMPUTE_PROFILER_PERFWORKS_DIR") != nullptr;
  if (const char* sv = getenv("MOE_SERIAL_COPIES")) e->serial_copies = atoi(sv) != 0;
  if (const char* tv = getenv("MOE_COPY_TRACE")) e->trace_copies = atoi(tv) != 0;
  if (const char* pv = getenv("MOE_PDL")) e->pdl = atoi(pv) != 0;
  if (const char* gv = getenv("MOE_GRAPH")) e->use_graph = atoi(gv) != 0;
  if (const char* av = getenv("MOE_ATTN_FUSED")) e->attn_fused = atoi(av) != 0;
  if (const char* cp = getenv("MOE_COPY_PARK")) e->copy_park = atoi(cp) != 0;
  for (auto& ev : e->tok_ev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (const char* w = getenv("MOE_WAIT_TIMEOUT_MS")) e->wait_ns = 1000000ull * atoll(w);
  if (const char* a = getenv("MOE_AHEAD")) e->ahead = std::max(1, atoi(a));
  e->ring.resize(64);
  for (auto& ev : e->ring) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  e->d = md->d_model;
  e->f = md->d_ffn;
  e->V = md->vocab_size;
  e->L = md->n_layers;
  e->E = md->n_experts;
  e->H = md->n_heads;
  e->hd = md->d_model / md->n_heads;
  e->T = md->max_seq_len;
  e->topk = md->top_k;
  cudaError_t ce = cudaSetDevice(device);
  if (ce != cudaSuccess) {
    delete e;
    return fail(MOE_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(ce));
  }
  ce = preload_kernels();
  if (ce == cudaSuccess) ce = preload_tile_kernels();
  if (ce != cudaSuccess) {
    delete e;
    return fail(MOE_ERR_CUDA, std::string("kernel preload: ") + cudaGetErrorString(ce));
  }
  cudaStreamCreateWithFlags(&e->s_comp, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&e->s_copy, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&e->s_copy2, cudaStreamNonBlocking);
  cudaEventCreate(&e->t0);
  cudaEventCreate(&e->t1);
  const int L = e->L;
  e->wq.resize(L);
  e->wk.resize(L);
  e->wv.resize(L);
  e->wo.resize(L);
  e->ln1g.assign(L, nullptr);
  e->ln1b.assign(L, nullptr);
  e->ln2g.assign(L, nullptr);
  e->ln2b.assign(L, nullptr);
  e->gate.assign(L, nullptr);
  e->gate_h.assign(L, nullptr);
  e->loaded.assign((size_t)L * e->E, false);
  e->arena_idx.resize((size_t)L * e->E);
  for (size_t i = 0; i < e->arena_idx.size(); ++i) e->arena_idx[i] = (int)i;
  e->n_owned = L * e->E;
  *out = e;
  return MOE_OK;
}

static int load_dense_mat(moe_engine* e, const moe_matrix* m, DevMat* D, const char* nm) {
  Layout Lo;
  int rc = make_layout(m, &Lo, nm);
  if (rc) return rc;
  if (D->mem) cudaFree(D->mem);
  CU(cudaMalloc(&D->mem, Lo.total() + 64));  // + slack: 16-byte bulk copies of zmeta
  D->bytes = Lo.total();
  e->dev_bytes += Lo.total();
  rc = upload_and_tile(m, Lo, static_cast<uint8_t*>(D->mem), e->s_comp);
  if (rc) return rc;
  D->M = matdev_from(Lo, static_cast<uint8_t*>(D->mem));
  D->bits = Lo.bits;
  return MOE_OK;
}

static int load_vec(moe_engine* e, const moe_matrix* m, float** dst, int64_t n, const char* nm) {
  if ((int64_t)m->rows * m->cols != n) return fail(MOE_ERR_VALUE, std::string(nm) + ": wrong shape");
  std::vector<float> tmp(n);
  if (m->bits == 32) {
    memcpy(tmp.data(), m->codes, n * 4);
  } else if (m->bits == 16) {
    const uint16_t* hp = static_cast<const uint16_t*>(m->codes);
    for (int64_t i = 0; i < n; ++i) {
      __half_raw r;
      r.x = hp[i];
      tmp[i] = __half2float(__half(r));
    }
  } else {
    return fail(MOE_ERR_VALUE, std::string(nm) + ": must be fp16 or fp32");
  }
  if (!*dst) {
    CU(cudaMalloc(dst, n * 4));
    e->dev_bytes += n * 4;
  }
  CU(cudaMemcpy(*dst, tmp.data(), n * 4, cudaMemcpyHostToDevice));
  return MOE_OK;
}

int moe_load_tensor(moe_engine* e, const char* name, const moe_matrix* m) {
  if (!e || !name || !m) return fail(MOE_ERR_VALUE, "null argument");
  cudaSetDevice(e->dev);
  const std::string nm(name);
  const int d = e->d;
  if (nm == "wte" || nm == "wpe") {
    const int rows = nm == "wte" ? e->V : e->T;
    if (m->rows != rows || m->cols != d) return fail(MOE_ERR_VALUE, nm + ": wrong shape");
    if (m->bits != 16 && m->bits != 32) return fail(MOE_ERR_VALUE, nm + ": must be fp16 or fp32");
    const int half = m->bits == 16;
    if (e->emb_half >= 0 && e->emb_half != half)
      return fail(MOE_ERR_VALUE, "wte and wpe must share a dtype");
    e->emb_half = half;
    void** dst = nm == "wte" ? &e->wte : &e->wpe;
    const size_t bytes = (size_t)rows * d * (half ? 2 : 4);
    if (m->codes_len != (int64_t)bytes) return fail(MOE_ERR_FORMAT, nm + ": size mismatch");
    if (*dst) cudaFree(*dst);
    CU(cudaMalloc(dst, bytes));
    e->dev_bytes += bytes;
    CU(cudaMemcpy(*dst, m->codes, bytes, cudaMemcpyHostToDevice));
    return MOE_OK;
  }
  if (nm == "lm_head") {
    if (m->rows != d || m->cols != e->V) return fail(MOE_ERR_VALUE, "lm_head: wrong shape");
    if (m->bits != 16 && m->bits != 32) return fail(MOE_ERR_VALUE, "lm_head must be fp16/fp32");
    e->lm_bits = m->bits;
    return load_dense_mat(e, m, &e->lm_head, "lm_head");
  }
  if (nm == "ln_f.gamma") return load_vec(e, m, &e->lnfg, d, name);
  if (nm == "ln_f.beta") return load_vec(e, m, &e->lnfb, d, name);
  int l = -1;
  char rest[128] = {0};
  if (sscanf(name, "layers.%d.%127s", &l, rest) == 2 && l >= 0 && l < e->L) {
    const std::string r(rest);
    if (r == "ln1.gamma") return load_vec(e, m, &e->ln1g[l], d, name);
    if (r == "ln1.beta") return load_vec(e, m, &e->ln1b[l], d, name);
    if (r == "ln2.gamma") return load_vec(e, m, &e->ln2g[l], d, name);
    if (r == "ln2.beta") return load_vec(e, m, &e->ln2b[l], d, name);
    if (r == "gate") {
      if (m->rows != d || m->cols != e->E) return fail(MOE_ERR_VALUE, nm + ": wrong shape");
      const int64_t n = (int64_t)d * e->E;
      int rc = load_vec(e, m, &e->gate[l], n, name);
      if (rc) return rc;
      // fp16-passthrough role (quant.py:428): keep an exact fp16 copy for TMA staging
      std::vector<float> f(n);
      CU(cudaMemcpy(f.data(), e->gate[l], n * 4, cudaMemcpyDeviceToHost));
      std::vector<__half> hv(n);
      bool exact = true;
      for (int64_t i = 0; i < n && exact; ++i) {
        hv[i] = __float2half_rn(f[i]);
        exact = __half2float(hv[i]) == f[i];
      }
      if (e->gate_h[l]) cudaFree(e->gate_h[l]);
      e->gate_h[l] = nullptr;
      if (exact) {
        CU(cudaMalloc(&e->gate_h[l], n * 2));
        CU(cudaMemcpy(e->gate_h[l], hv.data(), n * 2, cudaMemcpyHostToDevice));
        e->dev_bytes += n * 2;
      }
      return MOE_OK;
    }
    DevMat* D = r == "attn.wq" ? &e->wq[l] : r == "attn.wk" ? &e->wk[l]
              : r == "attn.wv" ? &e->wv[l] : r == "attn.wo" ? &e->wo[l] : nullptr;
    if (D) {
      if (m->rows != d || m->cols != d) return fail(MOE_ERR_VALUE, nm + ": wrong shape");
      if (m->bits == 16) return fail(MOE_ERR_VALUE, nm + ": fp16 attention unsupported");
      if (e->attn_bits && e->attn_bits != m->bits)
        return fail(MOE_ERR_VALUE, "all attention projections must share one scheme");
      e->attn_bits = m->bits;
      return load_dense_mat(e, m, D, name);
    }
  }
  return fail(MOE_ERR_VALUE, "unknown tensor name " + nm);
}

static int set_expert_layout(moe_engine* e, const moe_matrix* ms[3]) {
  Layout lo[3];
  const char* nms[3] = {"w_gate_proj", "w_up_proj", "w_down_proj"};
  for (int i = 0; i < 3; ++i) {
    int rc = make_layout(ms[i], &lo[i], nms[i]);
    if (rc) return rc;
  }
  if (lo[0].K != e->d || lo[0].N != e->f || lo[1].K != e->d || lo[1].N != e->f ||
      lo[2].K != e->f || lo[2].N != e->d)
    return fail(MOE_ERR_VALUE, "expert matrices have the wrong shape");
  if (lo[0].bits != lo[1].bits || lo[0].bits != lo[2].bits || lo[0].bits == 16)
    return fail(MOE_ERR_VALUE, "expert matrices must share one scheme (2/3/4-bit or fp32)");
  if (e->xl_set) {
    for (int i = 0; i < 3; ++i)
      if (lo[i].bits != e->xl[i].bits || lo[i].g != e->xl[i].g || lo[i].sg != e->xl[i].sg)
        return fail(MOE_ERR_VALUE, "all experts must share one scheme");
    return MOE_OK;
  }
  size_t off = 0;
  for (int i = 0; i < 3; ++i) {
    e->xoff[i][0] = off;
    off += lo[i].rec;
  }
  for (int i = 0; i < 3; ++i) {
    e->xoff[i][1] = off;
    off += lo[i].scales;
  }
  for (int i = 0; i < 3; ++i) {
    e->xoff[i][2] = off;
    off += lo[i].zeros;
  }
  for (int i = 0; i < 3; ++i) {
    e->xoff[i][3] = off;
    off += lo[i].zmeta;
  }
  for (int i = 0; i < 3; ++i) e->xl[i] = lo[i];
  e->xbytes = off;
  e->slot_stride = (off + 255) & ~size_t(255);
  e->expert_bits = lo[0].bits;
  e->xl_set = true;
  const size_t arena = e->xbytes * (size_t)e->n_owned;
  CU(cudaHostAlloc(&e->arena, arena, cudaHostAllocPortable));
  return MOE_OK;
}

int moe_load_expert(moe_engine* e, int32_t layer, int32_t expert, const moe_matrix* w1,
                    const moe_matrix* w3, const moe_matrix* w2) {
  if (!e || !w1 || !w3 || !w2) return fail(MOE_ERR_VALUE, "null argument");
  if (layer < 0 || layer >= e->L || expert < 0 || expert >= e->E)
    return fail(MOE_ERR_VALUE, "payload key outside model dimensions");
  cudaSetDevice(e->dev);
  const moe_matrix* ms[3] = {w1, w3, w2};
  int rc = set_expert_layout(e, ms);
  if (rc) return rc;
  if (!e->owns(layer, expert)) return MOE_OK;  // expert parallel: another rank's expert
  uint8_t* tmp = nullptr;
  CU(cudaMalloc(&tmp, e->xbytes + 256));
  for (int i = 0; i < 3; ++i) {
    Layout lo;
    rc = make_layout(ms[i], &lo, "expert");
    if (rc) break;
    // tile each matrix into a contiguous scratch, then scatter its sections
    uint8_t* one = nullptr;
    CU(cudaMalloc(&one, lo.total() + 16));
    rc = upload_and_tile(ms[i], lo, one, e->s_comp);
    if (!rc) {
      const size_t secs[4] = {lo.rec, lo.scales, lo.zeros, lo.zmeta};
      size_t so = 0;
      for (int k = 0; k < 4; ++k) {
        if (secs[k]) CU(cudaMemcpy(tmp + e->xoff[i][k], one + so, secs[k], cudaMemcpyDeviceToDevice));
        so += secs[k];
      }
    }
    cudaFree(one);
    if (rc) break;
  }
  if (!rc) {
    CU(cudaMemcpy(e->arena + e->arena_off(layer, expert), tmp, e->xbytes,
                  cudaMemcpyDeviceToHost));
    e->loaded[(size_t)layer * e->E + expert] = true;
  }
  cudaFree(tmp);
  return rc;
}

int moe_finalize(moe_engine* e) {
  if (!e) return fail(MOE_ERR_VALUE, "null engine");
  if (e->finalized) return MOE_OK;
  cudaSetDevice(e->dev);
  const int L = e->L, E = e->E, d = e->d, f = e->f, V = e->V, T = e->T;
  if (!e->wte || !e->wpe || !e->lm_head.mem || !e->lnfg || !e->lnfb)
    return fail(MOE_ERR_VALUE, "missing embedding / lm_head / ln_f tensors");
  for (int l = 0; l < L; ++l)
    if (!e->wq[l].mem || !e->wk[l].mem || !e->wv[l].mem || !e->wo[l].mem || !e->ln1g[l] ||
        !e->ln1b[l] || !e->ln2g[l] || !e->ln2b[l] || !e->gate[l])
      return fail(MOE_ERR_VALUE, "missing tensors of layer " + std::to_string(l));
  for (size_t i = 0; i < e->loaded.size(); ++i)
    if (!e->loaded[i] && e->arena_idx[i] >= 0)
      return fail(MOE_ERR_UNKNOWN_EXPERT, "expert payload missing");
  const int k = e->cc.k, b = e->cc.b;
  e->nbuf = L * k + b + E + k + e->sc.m + 2;
  CU(cudaMalloc(&e->pool, e->slot_stride * (size_t)e->nbuf + 64));
  e->dev_bytes += e->slot_stride * (size_t)e->nbuf;
  int rc;
  if ((rc = e->dalloc(&e->flags, e->nbuf))) return rc;
  // activations
  if ((rc = e->dalloc(&e->x, (size_t)T * d))) return rc;
  if ((rc = e->dalloc(&e->h, (size_t)T * d))) return rc;
  if ((rc = e->dalloc(&e->xn, d))) return rc;
  if ((rc = e->dalloc(&e->ctx, d))) return rc;
  if ((rc = e->dalloc(&e->logits, (size_t)T * V))) return rc;
  // split planning in storage units (MatDev.nqp: quads, or k-steps for the
  // tensor-core layout) over column blocks (MatDev.ncb)
  // MOE_MG_WAVES="qkv,wo,up,down": resident waves per launch (experiment;
  // default one wave each)
  int waves_of[4] = {1, 1, 1, 1};
  if (const char* w = getenv("MOE_MG_WAVES"))
    sscanf(w, "%d,%d,%d,%d", &waves_of[0], &waves_of[1], &waves_of[2], &waves_of[3]);
  auto plan = [](int njobs, const MatDev& M, int* Q, int* S, int nw = 1) {
    *Q = plan_qps(njobs * M.ncb, M.nqp, gemv_qs(M.bits), M.mma != 0, std::max(nw, 1));
    *S = (M.nqp + *Q - 1) / *Q;
  };
  const MatDev xm0 = matdev_from(e->xl[0], nullptr), xm2 = matdev_from(e->xl[2], nullptr);
  plan(3, e->wq[0].M, &e->Q_qkv, &e->S_qkv, waves_of[0]);
  plan(1, e->wo[0].M, &e->Q_wo, &e->S_wo, waves_of[1]);
  plan(2 * e->topk, xm0, &e->Q_up, &e->S_up, waves_of[2]);
  plan(e->topk, xm2, &e->Q_dn, &e->S_dn, waves_of[3]);
  plan(1, e->lm_head.M, &e->Q_lm, &e->S_lm);
  if ((rc = e->dalloc(&e->qkv_part, (size_t)3 * e->S_qkv * d))) return rc;
  if ((rc = e->dalloc(&e->wo_part, (size_t)e->S_wo * d))) return rc;
  if ((rc = e->dalloc(&e->up_part, (size_t)2 * e->topk * e->S_up * f))) return rc;
  if ((rc = e->dalloc(&e->dn_part, (size_t)e->topk * e->S_dn * d))) return rc;
  if ((rc = e->dalloc(&e->wo_acc, (size_t)d))) return rc;
  if ((rc = e->dalloc(&e->qkv_acc, (size_t)3 * d))) return rc;
  if ((rc = e->dalloc(&e->dn_acc, (size_t)e->topk * d))) return rc;
  if ((rc = e->dalloc(&e->lm_part, (size_t)e->S_lm * V))) return rc;
  if ((rc = e->dalloc(&e->qkv_out, (size_t)3 * d))) return rc;
  if ((rc = e->dalloc(&e->wo_out, (size_t)d))) return rc;
  if ((rc = e->dalloc(&e->up_out, (size_t)2 * e->topk * f))) return rc;
  if ((rc = e->dalloc(&e->dn_out, (size_t)e->topk * d))) return rc;
  if ((rc = e->dalloc(&e->cnt, 4096))) return rc;
  if ((rc = e->dalloc(&e->kc, (size_t)L * T * d))) return rc;
  if ((rc = e->dalloc(&e->vc, (size_t)L * T * d))) return rc;
  if ((rc = e->dalloc(&e->route, T))) return rc;
  if ((rc = e->dalloc(&e->trace, (size_t)T * L))) return rc;
  if (e->rec_hidden && (rc = e->dalloc(&e->trace_hidden, (size_t)T * L * d))) return rc;
  if ((rc = e->dalloc(&e->tok_dev, 1))) return rc;
  if ((rc = e->dalloc(&e->tok_hist, T))) return rc;
  if ((rc = e->dalloc(&e->tok_in, T))) return rc;
  const int nblk = (V + 255) / 256;
  if ((rc = e->dalloc(&e->cand_val, nblk))) return rc;
  if ((rc = e->dalloc(&e->cand_idx, nblk))) return rc;
  if ((rc = e->dalloc(&e->counter, 1))) return rc;
  if ((rc = e->dalloc(&e->err, 8))) return rc;
  if ((rc = e->dalloc(&e->ds_dev, 1))) return rc;
  CU(cudaHostAlloc(&e->ds_host, sizeof(DecodeState), cudaHostAllocDefault));
  CU(cudaHostAlloc(&e->hstat, sizeof(HostStatus), cudaHostAllocDefault));
  CU(cudaHostAlloc(&e->logits_h, (size_t)V * 4, cudaHostAllocDefault));
  // device store state
  const int kk = std::max(k, 1);
  e->ev_cap = std::max(4096, T * L * (3 * e->topk + e->sc.m + 2) + L * E * 3);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 15) & ~size_t(15);
    return o;
  };
  const size_t o_lru = take((size_t)L * kk * 4), o_len = take((size_t)L * 4),
               o_res = take((size_t)L * E * 4), o_sl = take(std::max(b, 1) * 4),
               o_se = take(std::max(b, 1) * 4), o_ss = take(std::max(b, 1) * 4),
               o_sb = take(std::max(b, 1) * 4), o_sc = take(16), o_seq = take(16),
               o_free = take((size_t)e->nbuf * 4), o_pend = take((size_t)e->nbuf * 4),
               o_gen = take((size_t)e->nbuf * 4), o_ev = take((size_t)e->ev_cap * sizeof(DevEvent));
  CU(cudaMalloc(&e->st_mem, off));
  e->dev_bytes += off;
  CU(cudaMemset(e->st_mem, 0, off));
  uint8_t* sm = static_cast<uint8_t*>(e->st_mem);
  StoreDev& S = e->st;
  S.L = L;
  S.E = E;
  S.k = k;
  S.b = b;
  S.top_k = e->topk;
  S.nbuf = e->nbuf;
  S.expert_bytes = e->cc.expert_bytes;
  S.lru = reinterpret_cast<int*>(sm + o_lru);
  S.lru_len = reinterpret_cast<int*>(sm + o_len);
  S.res_buf = reinterpret_cast<int*>(sm + o_res);
  S.stg_layer = reinterpret_cast<int*>(sm + o_sl);
  S.stg_exp = reinterpret_cast<int*>(sm + o_se);
  S.stg_stamp = reinterpret_cast<int*>(sm + o_ss);
  S.stg_buf = reinterpret_cast<int*>(sm + o_sb);
  S.scalars = reinterpret_cast<int*>(sm + o_sc);
  S.seq = reinterpret_cast<long long*>(sm + o_seq);
  S.free_stack = reinterpret_cast<int*>(sm + o_free);
  S.pending = reinterpret_cast<int*>(sm + o_pend);
  S.gen = reinterpret_cast<uint32_t*>(sm + o_gen);
  S.ev = reinterpret_cast<DevEvent*>(sm + o_ev);
  S.state_base = reinterpret_cast<int*>(sm);  // everything before the event log
  S.state_ints = (int)(o_ev / 4);
  S.ev_cap = e->ev_cap;
  S.owned = nullptr;
  S.err = e->err;
  {
    std::vector<int> neg(std::max(b, 1), -1), fs(e->nbuf);
    CU(cudaMemcpy(S.stg_layer, neg.data(), neg.size() * 4, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(S.stg_exp, neg.data(), neg.size() * 4, cudaMemcpyHostToDevice));
    for (int i = 0; i < e->nbuf; ++i) fs[i] = e->nbuf - 1 - i;
    CU(cudaMemcpy(S.free_stack, fs.data(), fs.size() * 4, cudaMemcpyHostToDevice));
    const int sc4[4] = {0, e->nbuf, 0, 0};
    CU(cudaMemcpy(S.scalars, sc4, 16, cudaMemcpyHostToDevice));
  }
  if (e->ep_world > 1) {  // expert parallel: owned mask + exchange block
    std::vector<uint8_t> own((size_t)L * E);
    for (size_t i = 0; i < own.size(); ++i) own[i] = e->arena_idx[i] >= 0;
    CU(cudaMalloc(&e->owned_dev, own.size()));
    CU(cudaMemcpy(e->owned_dev, own.data(), own.size(), cudaMemcpyHostToDevice));
    S.owned = e->owned_dev;
    const size_t recv_bytes = (size_t)2 * e->topk * e->ep_world * d * sizeof(float);
    const size_t xbytes_all = recv_bytes + (size_t)(e->ep_world + 1) * 8;
    CU(cudaMalloc(&e->xch, xbytes_all));
    CU(cudaMemset(e->xch, 0, xbytes_all));
    e->dev_bytes += xbytes_all;
    e->xrecv = reinterpret_cast<float*>(e->xch);
    e->xflag = reinterpret_cast<unsigned long long*>(e->xch + recv_bytes);
    e->xseq = e->xflag + e->ep_world;
  }
  if (!write_value32()) return fail(MOE_ERR_CUDA, "cuStreamWriteValue32 unavailable");
  CU(cudaHostAlloc(&e->mb_host, sizeof(Mailbox), cudaHostAllocMapped));
  memset(e->mb_host, 0, sizeof(Mailbox));
  CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->mb_dev), e->mb_host, 0));
  S.mb = e->mb_dev;
  S.flags = e->flags;
  if (!e->sc.enabled) e->copy_chunk = e->xbytes;  // nothing to preempt: whole experts
  if (const char* cm = getenv("MOE_COPY_CHUNK_MB")) e->copy_chunk = (size_t)atoll(cm) << 20;
  CU(cudaDeviceSynchronize());
  e->copier = std::thread([e] { e->run_copier(); });
  e->finalized = true;
  return MOE_OK;
}

static int check_ready(moe_engine* e, bool need_peers = false) {
  if (!e) return fail(MOE_ERR_VALUE, "null engine");
  if (!e->finalized) return fail(MOE_ERR_RUNTIME, "engine not finalized (weights not loaded)");
  if (need_peers && e->ep_world > 1 && !e->ep_connected && !e->ep_nccl)
    return fail(MOE_ERR_RUNTIME, "expert parallel engine not connected to its peers");
  cudaSetDevice(e->dev);
  return MOE_OK;
}

int moe_reset_session(moe_engine* e) {
  int rc = check_ready(e);
  if (rc) return rc;
  e->pos = 0;
  e->has_logits = false;
  return MOE_OK;
}

int moe_prefill(moe_engine* e, const int32_t* tokens, int32_t n, float* logits_out) {
  NvtxRange nvtx("moe_prefill");
  int rc = check_ready(e, true);
  if (rc) return rc;
  e->pos = 0;  // reset_session (engine.py:149): KV and trace, not the store
  e->has_logits = false;
  e->launches = 0;
  if (n < 1) return fail(MOE_ERR_VALUE, "prompt must contain at least one token");
  for (int i = 0; i < n; ++i) {
    if (tokens[i] < 0 || tokens[i] >= e->V)
      return fail(MOE_ERR_VALUE, "token id " + std::to_string(tokens[i]) +
                                     " outside vocabulary of " + std::to_string(e->V));
    if (i >= e->T)
      return fail(MOE_ERR_VALUE, "position " + std::to_string(i) + " exceeds max_seq_len=" +
                                     std::to_string(e->T));
  }
  CU(cudaEventRecord(e->t0, e->s_comp));
  const long long c0 = launch_count();
  for (int p = 0; p < n; ++p) {
    EmbedParams ep{};
    ep.wte = e->wte;
    ep.wpe = e->wpe;
    ep.half = e->emb_half;
    ep.tok = tokens[p];
    ep.pos = p;
    ep.d = e->d;
    ep.x = e->x + (size_t)p * e->d;
    ep.site = 0;
    launch_embed(ep, e->s_comp, e->pdl);
  }
  if (e->batched_prefill_ok(n)) {
    rc = e->prefill_batched(n);
    if (rc) return rc;
  } else {
  for (int l = 0; l < e->L; ++l) {
    for (int p = 0; p < n; ++p) e->enq_attention(l, p, 1);
    PrefillBKParams pb{};
    pb.route = e->route;
    pb.st = e->st;
    pb.layer = l;
    pb.n = n;
    pb.top_k = e->topk;
    launch_prefill_bk(pb, e->s_comp);
    e->dbg("prefill_bk", l, n);
    for (int p = 0; p < n; ++p) e->enq_experts(l, p);
  }
  }
  for (int p = 0; p < n; ++p) e->enq_logits(p, e->logits + (size_t)p * e->V);
  e->launches = launch_count() - c0;
  CU(cudaGetLastError());
  rc = e->finish_call();
  if (rc) return rc;
  if (logits_out)
    CU(cudaMemcpy(logits_out, e->logits, (size_t)n * e->V * 4, cudaMemcpyDeviceToHost));
  if (n > 1)  // keep the last position's logits at slot 0 for decode
    CU(cudaMemcpy(e->logits, e->logits + (size_t)(n - 1) * e->V, (size_t)e->V * 4,
                  cudaMemcpyDeviceToDevice));
  e->pos = n;
  e->has_logits = true;
  return MOE_OK;
}

int moe_step(moe_engine* e, int32_t token, float* logits_out) {
  NvtxRange nvtx("moe_step");
  int rc = check_ready(e, true);
  if (rc) return rc;
  if (token < 0 || token >= e->V)
    return fail(MOE_ERR_VALUE, "token id " + std::to_string(token) + " outside vocabulary of " +
                                   std::to_string(e->V));
  if (e->pos >= e->T)
    return fail(MOE_ERR_VALUE, "position " + std::to_string(e->pos) + " exceeds max_seq_len=" +
                                   std::to_string(e->T));
  e->launches = 0;
  CU(cudaEventRecord(e->t0, e->s_comp));
  *e->ds_host = DecodeState{e->pos, 0, token, e->tok_seq};
  CU(cudaMemcpyAsync(e->ds_dev, e->ds_host, sizeof(DecodeState), cudaMemcpyHostToDevice,
                     e->s_comp));
  rc = e->run_tokens(1);
  if (rc) return rc;
  CU(cudaGetLastError());
  rc = e->finish_call(logits_out != nullptr);
  if (rc) return rc;
  e->pos += 1;
  e->tok_seq += 1;
  if (logits_out) memcpy(logits_out, e->logits_h, (size_t)e->V * 4);
  e->has_logits = true;
  return MOE_OK;
}

int moe_decode_greedy(moe_engine* e, int32_t n, int32_t* tokens_out, float* final_logits_out) {
  NvtxRange nvtx("moe_decode_greedy");
  int rc = check_ready(e, true);
  if (rc) return rc;
  if (n < 1) return fail(MOE_ERR_VALUE, "n_tokens must be >= 1");
  if (!e->has_logits) return fail(MOE_ERR_RUNTIME, "prefill must run before decoding");
  if (e->pos + n > e->T) {
    // the reference decodes token by token and raises in the first forward
    // pass past the cache (KVCache.append, model.py:265-268): the tokens that
    // fit are decoded (events, trace, KV and position advance), then it raises
    if (e->T > e->pos) {
      rc = moe_decode_greedy(e, e->T - e->pos, nullptr, nullptr);
      if (rc) return rc;
    }
    return fail(MOE_ERR_VALUE, "position " + std::to_string(e->T) + " exceeds max_seq_len=" +
                                   std::to_string(e->T));
  }
  e->launches = 0;
  CU(cudaEventRecord(e->t0, e->s_comp));
  // cursor: position from the host, first token = argmax of the last logits
  *e->ds_host = DecodeState{e->pos, 0, 0, e->tok_seq};
  CU(cudaMemcpyAsync(e->ds_dev, e->ds_host, sizeof(DecodeState), cudaMemcpyHostToDevice,
                     e->s_comp));
  CU(cudaMemcpyAsync(&e->ds_dev->tok, e->tok_dev, sizeof(int), cudaMemcpyDeviceToDevice,
                     e->s_comp));
  rc = e->run_tokens(n);
  if (rc) return rc;
  CU(cudaGetLastError());
  e->bad_pos = -1;
  rc = e->finish_call(final_logits_out != nullptr);
  if (rc) {
    if (e->bad_pos >= e->pos) {  // the tokens before the failing one completed
      e->tok_seq += (unsigned)(e->bad_pos - e->pos);
      e->pos = e->bad_pos;
    }
    return rc;
  }
  e->pos += n;
  e->tok_seq += (unsigned)n;
  if (tokens_out) CU(cudaMemcpy(tokens_out, e->tok_hist, (size_t)n * 4, cudaMemcpyDeviceToHost));
  if (final_logits_out) memcpy(final_logits_out, e->logits_h, (size_t)e->V * 4);
  return MOE_OK;
}

int64_t moe_num_events(moe_engine* e) { return e ? (int64_t)e->events.size() : 0; }

int moe_read_events(moe_engine* e, int64_t start, int64_t count, moe_event* out) {
  if (!e || start < 0 || count < 0 || start + count > (int64_t)e->events.size())
    return fail(MOE_ERR_VALUE, "event range out of bounds");
  if (count) memcpy(out, e->events.data() + start, count * sizeof(moe_event));
  return MOE_OK;
}

int64_t moe_num_trace(moe_engine* e) { return e ? (int64_t)e->pos * e->L : 0; }

int moe_read_trace(moe_engine* e, int64_t start, int64_t count, moe_trace_rec* out,
                   float* hidden_out) {
  int rc = check_ready(e);
  if (rc) return rc;
  if (start < 0 || count < 0 || start + count > (int64_t)e->pos * e->L)
    return fail(MOE_ERR_VALUE, "trace range out of bounds");
  if (!count) return MOE_OK;
  CU(cudaMemcpy(out, e->trace + start, count * sizeof(moe_trace_rec), cudaMemcpyDeviceToHost));
  if (hidden_out) {
    if (!e->rec_hidden) return fail(MOE_ERR_VALUE, "hidden states were not recorded");
    CU(cudaMemcpy(hidden_out, e->trace_hidden + start * e->d, count * e->d * 4,
                  cudaMemcpyDeviceToHost));
  }
  return MOE_OK;
}

int moe_device_state(moe_engine* e, int32_t* lru_out, int32_t* staged_out) {
  int rc = check_ready(e);
  if (rc) return rc;
  const int L = e->L, k = e->cc.k, kk = std::max(k, 1), b = e->cc.b;
  std::vector<int> lru((size_t)L * kk), len(L), sl(std::max(b, 1)), se(std::max(b, 1));
  CU(cudaMemcpy(lru.data(), e->st.lru, lru.size() * 4, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(len.data(), e->st.lru_len, L * 4, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(sl.data(), e->st.stg_layer, sl.size() * 4, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(se.data(), e->st.stg_exp, se.size() * 4, cudaMemcpyDeviceToHost));
  if (lru_out)
    for (int l = 0; l < L; ++l)
      for (int i = 0; i < k; ++i) lru_out[l * k + i] = i < len[l] ? lru[l * kk + i] : -1;
  if (staged_out)
    for (int i = 0; i < b; ++i) staged_out[i] = sl[i] >= 0 ? sl[i] * e->E + se[i] : -1;
  return MOE_OK;
}

int moe_measure_h2d(moe_engine* e, int32_t reps, double* best_gbs, double* median_gbs) {
  if (!e || !best_gbs || reps < 1) return fail(MOE_ERR_VALUE, "bad argument");
  if (!e->finalized || !e->arena || !e->pool || e->xbytes == 0)
    return fail(MOE_ERR_RUNTIME, "engine not finalized");
  cudaSetDevice(e->dev);
  CU(cudaStreamSynchronize(e->s_comp));
  CU(cudaStreamSynchronize(e->s_copy));
  CU(cudaStreamSynchronize(e->s_copy2));
  cudaEvent_t a, b;
  CU(cudaEventCreate(&a));
  CU(cudaEventCreate(&b));
  std::vector<double> g;
  // the last pool buffer: a transient slot the store never holds between calls
  uint8_t* dst = e->pool + (size_t)(e->nbuf - 1) * e->slot_stride;
  int x0 = 0;
  while (x0 < (int)e->arena_idx.size() && e->arena_idx[x0] < 0) ++x0;
  const uint8_t* src = e->arena + (size_t)e->arena_idx[x0] * e->xbytes;
  for (int r = 0; r < reps; ++r) {
    CU(cudaEventRecord(a, e->s_copy));
    CU(cudaMemcpyAsync(dst, src, e->xbytes, cudaMemcpyHostToDevice, e->s_copy));
    CU(cudaEventRecord(b, e->s_copy));
    CU(cudaEventSynchronize(b));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, a, b));
    if (ms > 0) g.push_back(e->xbytes / (ms * 1e6));
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (g.empty()) return fail(MOE_ERR_RUNTIME, "no timed copy");
  std::sort(g.begin(), g.end());
  *best_gbs = g.back();
  if (median_gbs) *median_gbs = g[g.size() / 2];
  return MOE_OK;
}

int moe_get_stats(moe_engine* e, moe_stats* out) {
  if (!e || !out) return fail(MOE_ERR_VALUE, "null argument");
  {
    std::lock_guard<std::mutex> g(e->cmu);
    std::vector<CopyRec> keep;
    for (auto& c : e->copies) {
      if (cudaEventQuery(c.b) != cudaSuccess) {
        keep.push_back(c);
        continue;
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, c.a, c.b);
      e->busy_ms += ms;
      e->n_copies += 1;
      e->copy_bytes += c.bytes;
      if (ms > 0) e->peak_gbs = std::max(e->peak_gbs, c.bytes / (ms * 1e6));
      e->free_events.push_back(c.a);
      e->free_events.push_back(c.b);
    }
    e->copies.swap(keep);
  }
  memset(out, 0, sizeof(*out));
  out->h2d_copies = e->n_copies;
  out->h2d_bytes = e->copy_bytes;
  out->h2d_busy_ms = e->busy_ms;
  out->h2d_peak_gbs = e->peak_gbs;
  out->n_buffers = e->nbuf;
  out->slot_bytes = (int64_t)e->slot_stride;
  out->device_bytes = (int64_t)e->dev_bytes;
  out->arena_bytes = (int64_t)(e->xbytes * (size_t)e->n_owned);
  out->kernel_launches = e->launches;
  out->last_call_ms = e->last_ms;
  return MOE_OK;
}

int moe_set_profiling(moe_engine* e, int32_t on) {
  if (!e) return fail(MOE_ERR_VALUE, "null engine");
  e->prof = on != 0;
  for (int i = 0; i < moe_engine::K_N; ++i) {
    e->prof_ms[i] = 0;
    e->prof_cnt[i] = 0;
  }
  return MOE_OK;
}

int moe_kernel_times(moe_engine* e, double* ms_out, int64_t* count_out) {
  if (!e) return fail(MOE_ERR_VALUE, "null engine");
  for (int i = 0; i < moe_engine::K_N; ++i) {
    if (ms_out) ms_out[i] = e->prof_ms[i];
    if (count_out) count_out[i] = e->prof_cnt[i];
  }
  return MOE_OK;
}

int moe_ep_configure(moe_engine* e, int32_t rank, int32_t world) {
  if (!e) return fail(MOE_ERR_VALUE, "null engine");
  if (e->finalized || e->xl_set)
    return fail(MOE_ERR_RUNTIME, "moe_ep_configure must precede expert loading");
  if (world < 1 || world > MOE_EP_MAX || rank < 0 || rank >= world || world > e->E)
    return fail(MOE_ERR_VALUE, "expert parallel: need 0 <= rank < world <= min(8, E)");
  e->ep_rank = rank;
  e->ep_world = world;
  e->n_owned = 0;
  for (int l = 0; l < e->L; ++l)
    for (int x = 0; x < e->E; ++x)  // expert_parallel.owner_of
      e->arena_idx[(size_t)l * e->E + x] = (x * world) / e->E == rank ? e->n_owned++ : -1;
  return MOE_OK;
}

int moe_ep_handle(moe_engine* e, void* out64) {
  if (!e || !out64) return fail(MOE_ERR_VALUE, "null argument");
  if (!e->xch) return fail(MOE_ERR_RUNTIME, "expert parallel not configured / not finalized");
  cudaSetDevice(e->dev);
  cudaIpcMemHandle_t h;
  CU(cudaIpcGetMemHandle(&h, e->xch));
  memcpy(out64, &h, sizeof(h));
  return MOE_OK;
}

int moe_ep_connect(moe_engine* e, const void* handles) {
  if (!e || !handles) return fail(MOE_ERR_VALUE, "null argument");
  if (!e->xch) return fail(MOE_ERR_RUNTIME, "expert parallel not configured / not finalized");
  cudaSetDevice(e->dev);
  const size_t recv_bytes = (size_t)2 * e->topk * e->ep_world * e->d * sizeof(float);
  for (int r = 0; r < e->ep_world; ++r) {
    uint8_t* base = e->xch;
    if (r != e->ep_rank) {
      cudaIpcMemHandle_t h;
      memcpy(&h, static_cast<const uint8_t*>(handles) + (size_t)r * sizeof(h), sizeof(h));
      void* p = nullptr;
      CU(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      e->ipc_opened.push_back(p);
      base = static_cast<uint8_t*>(p);
    }
    e->peer_recv[r] = reinterpret_cast<float*>(base);
    e->peer_flag[r] = reinterpret_cast<unsigned long long*>(base + recv_bytes);
  }
  e->ep_connected = true;
  return MOE_OK;
}

int moe_nccl_unique_id(void* out128) {
  if (!out128) return fail(MOE_ERR_VALUE, "null argument");
  const NcclApi& n = nccl_api();
  if (!n.why.empty()) return fail(MOE_ERR_RUNTIME, n.why);
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  const ncclResult_t r = n.unique_id(&id);
  if (r != ncclSuccess) return fail(MOE_ERR_CUDA, std::string("ncclGetUniqueId: ") + n.error_string(r));
  memcpy(out128, &id, sizeof(id));
  return MOE_OK;
}

int moe_ep_connect_nccl(moe_engine* e, const void* id128) {
  if (!e || !id128) return fail(MOE_ERR_VALUE, "null argument");
  if (!e->finalized) return fail(MOE_ERR_RUNTIME, "engine not finalized (weights not loaded)");
  if (e->ep_connected || e->ep_nccl) return fail(MOE_ERR_RUNTIME, "expert parallel already connected");
  if (e->gexec) return fail(MOE_ERR_RUNTIME, "connect before the first decode");
  const NcclApi& n = nccl_api();
  if (!n.why.empty()) return fail(MOE_ERR_RUNTIME, n.why);
  cudaSetDevice(e->dev);
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  const ncclResult_t r = n.init_rank(&e->nccl_comm, e->ep_world, id, e->ep_rank);
  if (r != ncclSuccess) {
    e->nccl_comm = nullptr;
    return fail(MOE_ERR_CUDA, std::string("ncclCommInitRank: ") + n.error_string(r));
  }
  const size_t bytes = (size_t)e->ep_world * e->topk * e->d * sizeof(float);
  CU(cudaMalloc(&e->nrecv, bytes));
  CU(cudaMemset(e->nrecv, 0, bytes));
  e->dev_bytes += bytes;
  e->ep_nccl = true;
  return MOE_OK;
}

int moe_timeline(moe_engine* e, int32_t on) {
  if (!e) return fail(MOE_ERR_VALUE, "null engine");
  cudaSetDevice(e->dev);
  const int n = 3 + 8 * e->L;
  const size_t bytes = n * sizeof(TimelineSlot) + (size_t)n * 8 * 8;  // spans + phase marks
  if (on) {
    if (!e->timeline) CU(cudaMalloc(&e->timeline, bytes));
    std::vector<TimelineSlot> init(n, TimelineSlot{~0ull, 0ull});
    CU(cudaMemset(e->timeline, 0, bytes));
    CU(cudaMemcpy(e->timeline, init.data(), n * sizeof(TimelineSlot), cudaMemcpyHostToDevice));
    CU(set_timeline(e->timeline, n));
  } else {
    CU(set_timeline(nullptr, 0));
  }
  return MOE_OK;
}

int moe_read_timeline(moe_engine* e, uint64_t* out, int32_t cap, int32_t* n_out) {
  if (!e || !e->timeline) return fail(MOE_ERR_VALUE, "timeline not enabled");
  const int n = 3 + 8 * e->L;
  if (n_out) *n_out = n;
  // out: 2*n span words, then 8*n phase marks (cap counts 64-bit words / 2)
  if (out && cap > 0)
    CU(cudaMemcpy(out, e->timeline,
                  std::min<size_t>((size_t)cap * 2, (size_t)n * 10) * sizeof(uint64_t),
                  cudaMemcpyDeviceToHost));
  return MOE_OK;
}

int moe_profiler_range(int32_t on) {
  CU(on ? cudaProfilerStart() : cudaProfilerStop());
  return MOE_OK;
}

int moe_destroy(moe_engine* e) {
  if (e) {
    cudaSetDevice(e->dev);
    delete e;
  }
  return MOE_OK;
}

}  // extern "C"

// ============================================================ synthesis path
namespace {

constexpr double kSynthIHStd = 37837.22700;  // oracle/model.py SYNTH_IHSTD

float synth_scale(double std) { return (float)(std / kSynthIHStd); }

struct QScratch {  // device scratch for generate -> quantize -> tile
  float* w = nullptr;
  uint8_t* codes = nullptr;
  uint8_t* zeros = nullptr;
  uint16_t *zs = nullptr, *zo = nullptr, *sc = nullptr;
  float *gmin = nullptr, *gscale = nullptr;
  uint8_t* tiled = nullptr;
  size_t cap = 0;
  void release() {
    void* p[] = {w, codes, zeros, zs, zo, sc, gmin, gscale, tiled};
    for (void* q : p)
      if (q) cudaFree(q);
  }
};

int qscratch_alloc(QScratch& Q, size_t nmax) {
  Q.cap = nmax;
  CU(cudaMalloc(&Q.w, nmax * 4));
  CU(cudaMalloc(&Q.codes, nmax / 2 + 64));
  CU(cudaMalloc(&Q.zeros, nmax / 16 + 64));
  CU(cudaMalloc(&Q.zs, nmax / 128 + 64));
  CU(cudaMalloc(&Q.zo, nmax / 128 + 64));
  CU(cudaMalloc(&Q.sc, nmax / 32 + 64));
  CU(cudaMalloc(&Q.gmin, nmax / 4 + 64));
  CU(cudaMalloc(&Q.gscale, nmax / 4 + 64));
  CU(cudaMalloc(&Q.tiled, nmax * 4 + 256));
  return MOE_OK;
}

// layout descriptor for a synthetic K x N matrix of `bits`
Layout synth_layout(int K, int N, int bits) {
  moe_matrix m{};
  m.bits = bits;
  m.rows = K;
  m.cols = N;
  m.meta_bits = 8;
  if (bits <= 4) {
    m.group_size = bits == 2 ? 16 : 64;
    m.scale_group_size = bits == 4 ? 256 : 128;
    const int64_t ng = (int64_t)K * N / m.group_size;
    m.codes_len = (int64_t)K * N * bits / 8;
    m.n_groups = ng;
    m.n_scales = (ng + m.scale_group_size / m.group_size - 1) / (m.scale_group_size / m.group_size);
    m.n_zruns = (ng + m.scale_group_size - 1) / m.scale_group_size;
  } else {
    m.codes_len = (int64_t)K * N * (bits / 8);
  }
  Layout L;
  make_layout(&m, &L, "synth");
  return L;
}

// generate (K x N) with id `tid`, quantize (or keep fp32 / round to fp16) and
// tile into Q.tiled.  Returns the layout.
int synth_matrix(QScratch& Q, uint64_t seed, uint64_t tid, int K, int N, double std, int bits,
                 int half_round, Layout* out, cudaStream_t s) {
  const int64_t n = (int64_t)K * N;
  launch_synth(seed, tid, n, synth_scale(std), half_round, Q.w, s);
  Layout L = synth_layout(K, N, bits);
  if (L.bits == 0) return fail(MOE_ERR_VALUE, "synthetic shape incompatible with the device layout");
  RefMat R = refmat_of(L);
  if (bits <= 4) {
    launch_quantize(Q.w, K, N, bits, L.g, L.sg, Q.codes, Q.zeros, Q.zs, Q.zo, Q.sc, Q.gmin,
                    Q.gscale, s);
    R.codes = Q.codes;
    R.zeros = Q.zeros;
    R.zs = Q.zs;
    R.zo = Q.zo;
    R.scales = Q.sc;
  } else if (bits == 16) {
    // reuse gscale region as the fp16 staging of the values
    std::vector<float> tmp;  // (device conversion below)
    R.codes = reinterpret_cast<const uint8_t*>(Q.w);
  } else {
    R.codes = reinterpret_cast<const uint8_t*>(Q.w);
  }
  int rc = tile_device(R, L, Q.tiled, s);
  if (rc) return rc;
  *out = L;
  return MOE_OK;
}

__global__ void k_f32_to_f16(const float* a, __half* b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = __float2half_rn(a[i]);
}

}  // namespace

extern "C" {

int moe_synth_model(moe_engine* e, uint64_t seed, int32_t attn_bits, int32_t expert_bits) {
  if (!e) return fail(MOE_ERR_VALUE, "null engine");
  if (!((attn_bits >= 2 && attn_bits <= 4) || attn_bits == 32) ||
      !((expert_bits >= 2 && expert_bits <= 4) || expert_bits == 32))
    return fail(MOE_ERR_VALUE, "synthetic bits must be 2/3/4 or 32");
  cudaSetDevice(e->dev);
  cudaStream_t s = e->s_comp;
  const int d = e->d, f = e->f, V = e->V, L = e->L, E = e->E, T = e->T;
  const bool mixed = attn_bits != 32 || expert_bits != 32;
  const int hr = mixed ? 1 : 0;  // fp16-passthrough roles (quant.py:428)
  const double sd = 1.0 / std::sqrt((double)d), sf = 1.0 / std::sqrt((double)f);
  QScratch Q;
  int rc = qscratch_alloc(Q, std::max(std::max((size_t)d * f, (size_t)V * d), (size_t)T * d));
  if (rc) {
    Q.release();
    return rc;
  }
  auto put_raw = [&](const char* name, uint64_t tid, int rows, int cols, double std) -> int {
    const int64_t n = (int64_t)rows * cols;
    launch_synth(seed, tid, n, synth_scale(std), hr, Q.w, s);
    moe_matrix m{};
    m.rows = rows;
    m.cols = cols;
    std::vector<uint8_t> host(n * (mixed ? 2 : 4));
    if (mixed) {
      k_f32_to_f16<<<1184, 256, 0, s>>>(Q.w, reinterpret_cast<__half*>(Q.tiled), n);
      CU(cudaMemcpyAsync(host.data(), Q.tiled, n * 2, cudaMemcpyDeviceToHost, s));
      m.bits = 16;
    } else {
      CU(cudaMemcpyAsync(host.data(), Q.w, n * 4, cudaMemcpyDeviceToHost, s));
      m.bits = 32;
    }
    CU(cudaStreamSynchronize(s));
    m.codes = host.data();
    m.codes_len = (int64_t)host.size();
    return moe_load_tensor(e, name, &m);
  };
  if ((rc = put_raw("wte", 1, V, d, 0.02)) || (rc = put_raw("wpe", 2, T, d, 0.02)) ||
      (rc = put_raw("lm_head", 3, d, V, 0.02))) {
    Q.release();
    return rc;
  }
  std::vector<float> ones(d, 1.f), zeros(d, 0.f);
  auto put_vec = [&](const std::string& name, std::vector<float>& v) {
    moe_matrix m{};
    m.bits = 32;
    m.rows = 1;
    m.cols = (int)v.size();
    m.codes = v.data();
    m.codes_len = (int64_t)v.size() * 4;
    return moe_load_tensor(e, name.c_str(), &m);
  };
  if ((rc = put_vec("ln_f.gamma", ones)) || (rc = put_vec("ln_f.beta", zeros))) {
    Q.release();
    return rc;
  }
  // experts share one layout; set it from the synthetic shapes
  Layout xl3[3] = {synth_layout(d, f, expert_bits), synth_layout(d, f, expert_bits),
                   synth_layout(f, d, expert_bits)};
  uint8_t* xtmp = nullptr;
  for (int l = 0; l < L && !rc; ++l) {
    const uint64_t base = 1000 + 100 * (uint64_t)l;
    const std::string pre = "layers." + std::to_string(l) + ".";
    rc = put_vec(pre + "ln1.gamma", ones);
    if (!rc) rc = put_vec(pre + "ln1.beta", zeros);
    if (!rc) rc = put_vec(pre + "ln2.gamma", ones);
    if (!rc) rc = put_vec(pre + "ln2.beta", zeros);
    for (int j = 0; j < 4 && !rc; ++j) {
      Layout lo;
      rc = synth_matrix(Q, seed, base + j, d, d, sd, attn_bits, 0, &lo, s);
      if (rc) break;
      DevMat& D = j == 0 ? e->wq[l] : j == 1 ? e->wk[l] : j == 2 ? e->wv[l] : e->wo[l];
      if (D.mem) cudaFree(D.mem);
      CU(cudaMalloc(&D.mem, lo.total() + 64));
      D.bytes = lo.total();
      e->dev_bytes += lo.total();
      CU(cudaMemcpyAsync(D.mem, Q.tiled, lo.total(), cudaMemcpyDeviceToDevice, s));
      D.M = matdev_from(lo, static_cast<uint8_t*>(D.mem));
      D.bits = lo.bits;
      e->attn_bits = lo.bits;
    }
    if (rc) break;
    {  // gate (fp16-rounded in mixed mode), kept as fp32 [d][E]
      launch_synth(seed, base + 4, (int64_t)d * E, synth_scale(sd), hr, Q.w, s);
      std::vector<float> g((size_t)d * E);
      CU(cudaMemcpyAsync(g.data(), Q.w, g.size() * 4, cudaMemcpyDeviceToHost, s));
      CU(cudaStreamSynchronize(s));
      moe_matrix m{};
      m.bits = 32;
      m.rows = d;
      m.cols = E;
      m.codes = g.data();
      m.codes_len = (int64_t)g.size() * 4;
      rc = moe_load_tensor(e, (pre + "gate").c_str(), &m);
      if (rc) break;
    }
    for (int x = 0; x < E && !rc; ++x) {
      if (!e->xl_set) {  // first expert defines the buffer layout + arena
        size_t off = 0;
        for (int i = 0; i < 3; ++i) { e->xoff[i][0] = off; off += xl3[i].rec; }
        for (int i = 0; i < 3; ++i) { e->xoff[i][1] = off; off += xl3[i].scales; }
        for (int i = 0; i < 3; ++i) { e->xoff[i][2] = off; off += xl3[i].zeros; }
        for (int i = 0; i < 3; ++i) { e->xoff[i][3] = off; off += xl3[i].zmeta; }
        for (int i = 0; i < 3; ++i) e->xl[i] = xl3[i];
        e->xbytes = off;
        e->slot_stride = (off + 255) & ~size_t(255);
        e->expert_bits = xl3[0].bits;
        e->xl_set = true;
        CU(cudaHostAlloc(&e->arena, e->xbytes * (size_t)e->n_owned, cudaHostAllocPortable));
        CU(cudaMalloc(&xtmp, e->slot_stride));
      }
      if (!e->owns(l, x)) continue;  // expert parallel: another rank's expert
      const int K3[3] = {d, d, f}, N3[3] = {f, f, d};
      const double sd3[3] = {sd, sd, sf};
      for (int i = 0; i < 3 && !rc; ++i) {
        Layout lo;
        rc = synth_matrix(Q, seed, base + 10 + 3 * x + i, K3[i], N3[i], sd3[i], expert_bits, 0, &lo,
                          s);
        if (rc) break;
        const size_t secs[4] = {lo.rec, lo.scales, lo.zeros, lo.zmeta};
        size_t so = 0;
        for (int k = 0; k < 4; ++k) {
          if (secs[k])
            CU(cudaMemcpyAsync(xtmp + e->xoff[i][k], Q.tiled + so, secs[k], cudaMemcpyDeviceToDevice, s));
          so += secs[k];
        }
      }
      if (rc) break;
      CU(cudaMemcpyAsync(e->arena + e->arena_off(l, x), xtmp, e->xbytes,
                         cudaMemcpyDeviceToHost, s));
      CU(cudaStreamSynchronize(s));
      e->loaded[(size_t)l * E + x] = true;
    }
  }
  CU(cudaStreamSynchronize(s));
  if (xtmp) cudaFree(xtmp);
  Q.release();
  return rc;
}

int moe_set_device(int32_t device) {
  CU(cudaSetDevice(device));
  return MOE_OK;
}

int moe_quantize_device(const float* w, int32_t rows, int32_t cols, int32_t bits,
                        int32_t group_size, int32_t scale_group_size, uint8_t* codes_out,
                        uint8_t* zeros_out, uint16_t* zscales_out, uint16_t* zoffsets_out,
                        uint16_t* scales_out) {
  if (bits < 2 || bits > 4) return fail(MOE_ERR_VALUE, "bits must be 2, 3 or 4");
  const int g = group_size, sg = scale_group_size;
  if (g < 1 || sg % g || cols % g || ((int64_t)g * bits) % 32)
    return fail(MOE_ERR_VALUE, "device quantizer needs cols % g == 0 and word-aligned groups");
  const int64_t n = (int64_t)rows * cols, ng = n / g, per = sg / g;
  const int64_t nsg = (ng + per - 1) / per, nruns = (ng + sg - 1) / sg;
  float *dw, *gmin, *gsc;
  uint8_t *dc, *dz;
  uint16_t *zs, *zo, *sc;
  CU(cudaMalloc(&dw, n * 4));
  CU(cudaMalloc(&gmin, ng * 4));
  CU(cudaMalloc(&gsc, ng * 4));
  CU(cudaMalloc(&dc, n * bits / 8 + 16));
  CU(cudaMalloc(&dz, ng));
  CU(cudaMalloc(&zs, nruns * 2));
  CU(cudaMalloc(&zo, nruns * 2));
  CU(cudaMalloc(&sc, nsg * 2));
  CU(cudaMemcpy(dw, w, n * 4, cudaMemcpyHostToDevice));
  launch_quantize(dw, rows, cols, bits, g, sg, dc, dz, zs, zo, sc, gmin, gsc, 0);
  CU(cudaGetLastError());
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(codes_out, dc, n * bits / 8, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(zeros_out, dz, ng, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(zscales_out, zs, nruns * 2, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(zoffsets_out, zo, nruns * 2, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(scales_out, sc, nsg * 2, cudaMemcpyDeviceToHost));
  void* ps[] = {dw, gmin, gsc, dc, dz, zs, zo, sc};
  for (void* p : ps) cudaFree(p);
  return MOE_OK;
}

int moe_gemv_device(const moe_matrix* m, const float* x, float* y) {
  CU(preload_kernels());
  Layout L;
  int rc = make_layout(m, &L, "gemv");
  if (rc) return rc;
  uint8_t* mem = nullptr;
  CU(cudaMalloc(&mem, L.total() + 16));
  rc = upload_and_tile(m, L, mem, 0);
  if (rc) {
    cudaFree(mem);
    return rc;
  }
  const MatDev M = matdev_from(L, mem);
  const int qps = plan_qps(M.ncb, M.nqp, gemv_qs(L.bits), M.mma != 0), S = (M.nqp + qps - 1) / qps;
  float *dx, *part, *dy;
  int* dcnt;
  CU(cudaMalloc(&dx, (size_t)L.K * 4));
  CU(cudaMalloc(&part, (size_t)S * L.N * 4));
  CU(cudaMalloc(&dy, (size_t)L.N * 4));
  CU(cudaMalloc(&dcnt, (size_t)M.ncb * 4));
  CU(cudaMemset(dcnt, 0, (size_t)M.ncb * 4));
  CU(cudaMemcpy(dx, x, (size_t)L.K * 4, cudaMemcpyHostToDevice));
  GLaunch P{};
  P.nj = 1;
  GJob& J = P.j[0];
  J.M = M;
  J.rel_slot = -1;
  J.xmode = X_PLAIN;
  J.x = dx;
  J.part = part;
  J.out = dy;
  J.reduce = 1;
  J.S = S;
  J.QPS = qps;
  J.blk0 = 0;
  P.cnt = dcnt;
  P.site = -1;
  finalize_launch(P);
  launch_gemv(L.bits, P, M.ncb * S, 0, false);
  CU(cudaGetLastError());
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(y, dy, (size_t)L.N * 4, cudaMemcpyDeviceToHost));
  cudaFree(mem);
  cudaFree(dx);
  cudaFree(part);
  cudaFree(dy);
  cudaFree(dcnt);
  return MOE_OK;
}

int moe_synth_tensor_device(uint64_t seed, uint64_t tensor_id, int64_t count, float scale,
                            float* out) {
  float* d = nullptr;
  CU(cudaMalloc(&d, count * 4));
  launch_synth(seed, tensor_id, count, scale, 0, d, 0);
  CU(cudaGetLastError());
  CU(cudaMemcpy(out, d, count * 4, cudaMemcpyDeviceToHost));
  cudaFree(d);
  return MOE_OK;
}

// GEMV microbenchmark: `njobs` independent K x N matrices of `bits` in one
// launch (like the expert up-projection), synthetic weights, weight sets
// rotated so the working set exceeds L2.  Returns the average device time per
// launch (back-to-back, PDL as requested) and the algorithmic GB/s.
int moe_bench_gemv(int32_t bits, int32_t K, int32_t N, int32_t njobs, int32_t iters, int32_t pdl,
                   double* us_out, double* gbs_out, double* detail_out) {
  if (njobs < 1 || njobs > MOE_GEMV_MAXJOBS || iters < 1) return fail(MOE_ERR_VALUE, "bad args");
  CU(preload_kernels());
  CU(preload_tile_kernels());
  const Layout L = synth_layout(K, N, bits);
  if (L.bits == 0) return fail(MOE_ERR_VALUE, "unsupported shape");
  const size_t mbytes = L.total();
  const size_t set_bytes = mbytes * njobs;
  const int nsets = (int)std::max<size_t>(2, (400ull << 20) / set_bytes + 1);
  QScratch Q;
  int rc = qscratch_alloc(Q, (size_t)K * N);
  if (rc) {
    Q.release();
    return rc;
  }
  std::vector<uint8_t*> mats((size_t)nsets * njobs, nullptr);
  cudaStream_t s;
  CU(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  for (size_t i = 0; i < mats.size(); ++i) {
    Layout lo;
    rc = synth_matrix(Q, 7, 100 + i % 8, K, N, 0.01, bits, 0, &lo, s);
    if (rc) break;
    CU(cudaMalloc(&mats[i], mbytes + 64));
    CU(cudaMemcpyAsync(mats[i], Q.tiled, mbytes, cudaMemcpyDeviceToDevice, s));
  }
  CU(cudaStreamSynchronize(s));
  CU(cudaGetLastError());
  if (rc) return rc;
  float *x, *part, *out;
  int* cnt;
  const MatDev M0 = matdev_from(L, nullptr);
  const int qps = plan_qps(M0.ncb * njobs, M0.nqp, gemv_qs(bits), M0.mma != 0),
            S = (M0.nqp + qps - 1) / qps;
  CU(cudaMalloc(&x, (size_t)K * 4));
  CU(cudaMalloc(&part, (size_t)njobs * S * N * 4));
  CU(cudaMalloc(&out, (size_t)njobs * N * 4));
  CU(cudaMalloc(&cnt, 4096 * 4));
  CU(cudaMemset(cnt, 0, 4096 * 4));
  // split-K as in decode: fixed-point sums (MOE_BENCH_REDUCE=1: last-CTA reduction)
  const int bred = getenv("MOE_BENCH_REDUCE") ? atoi(getenv("MOE_BENCH_REDUCE")) : 2;
  unsigned long long* bacc = nullptr;
  CU(cudaMalloc(&bacc, (size_t)njobs * N * 8));
  CU(cudaMemset(bacc, 0, (size_t)njobs * N * 8));
  launch_synth(9, 9, K, 1e-5f, 0, x, s);
  std::vector<GLaunch> P(nsets);
  int nblk = 0;
  for (int t = 0; t < nsets; ++t) {
    P[t] = GLaunch{};
    P[t].nj = njobs;
    P[t].cnt = cnt;
    P[t].site = -1;
    for (int j = 0; j < njobs; ++j) {
      GJob& J = P[t].j[j];
      J.M = matdev_from(L, mats[(size_t)t * njobs + j]);
      J.rel_slot = -1;
      J.xmode = X_PLAIN;
      J.x = x;
      J.part = part + (size_t)j * S * N;
      J.out = out + (size_t)j * N;
      J.reduce = bred;
      J.acc = bacc + (size_t)j * N;
      J.QPS = qps;
      J.S = S;
    }
    nblk = finalize_launch(P[t]);
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  CU(cudaStreamSynchronize(s));
  CU(cudaGetLastError());
  launch_gemv(bits, P[0], nblk, s, pdl != 0);
  {
    cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess)
      return fail(MOE_ERR_CUDA, std::string("gemv launch (grid ") + std::to_string(nblk) +
                                    "): " + cudaGetErrorString(le));
  }
  for (int w = 0; w < 3; ++w) launch_gemv(bits, P[w % nsets], nblk, s, pdl != 0);
  CU(cudaEventRecord(a, s));
  for (int i = 0; i < iters; ++i) launch_gemv(bits, P[i % nsets], nblk, s, pdl != 0);
  CU(cudaEventRecord(b, s));
  CU(cudaEventSynchronize(b));
  CU(cudaGetLastError());
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double us = 1e3 * ms / iters;
  // algorithmic bytes = reference payload bytes of the matrices
  const double alg = (double)njobs * ((double)K * N * bits / 8 +
                                      (bits <= 4 ? (double)K * N / L.g + 2.0 * K * N / L.sg +
                                                       4.0 * L.nruns
                                                 : 0.0));
  if (us_out) *us_out = us;
  if (gbs_out) *gbs_out = alg / (us * 1e-6) / 1e9;
  if (detail_out) {  // one more launch with the timeline: span + block-0 phase marks
    unsigned long long* ct = nullptr;
    CU(cudaMalloc(&ct, (size_t)nblk * 4 * 8));
    CU(cudaMemset(ct, 0, (size_t)nblk * 4 * 8));
    CU(set_cta_trace(ct));
    TimelineSlot* tl = nullptr;
    CU(cudaMalloc(&tl, sizeof(TimelineSlot) + 64));
    TimelineSlot init{~0ull, 0ull};
    CU(cudaMemset(tl, 0, sizeof(TimelineSlot) + 64));
    CU(cudaMemcpy(tl, &init, sizeof(init), cudaMemcpyHostToDevice));
    CU(set_timeline(tl, 1));
    GLaunch Q = P[0];
    Q.site = 0;
    CU(cudaStreamSynchronize(s));
    launch_gemv(bits, Q, nblk, s, false);
    CU(cudaStreamSynchronize(s));
    CU(set_timeline(nullptr, 0));
    unsigned long long h[10];
    CU(cudaMemcpy(h, tl, sizeof(h), cudaMemcpyDeviceToHost));
    cudaFree(tl);
    detail_out[0] = (h[1] - h[0]) / 1e3;  // span us
    for (int i = 0; i < 3; ++i) detail_out[1 + i] = h[2 + i] ? (double)(h[2 + i] - h[0]) / 1e3 : -1;
    CU(set_cta_trace(nullptr));
    std::vector<unsigned long long> cv((size_t)nblk * 4);
    CU(cudaMemcpy(cv.data(), ct, cv.size() * 8, cudaMemcpyDeviceToHost));
    cudaFree(ct);
    if (const char* dump = getenv("MOE_CTA_TRACE_FILE")) {
      FILE* fp = fopen(dump, "a");
      if (fp) {
        fprintf(fp, "# bits %d K %d N %d jobs %d grid %d\n", bits, K, N, njobs, nblk);
        for (int i = 0; i < nblk; ++i)
          fprintf(fp, "%d %llu %.3f %.3f %.3f\n", i, cv[i * 4 + 3],
                  (cv[i * 4 + 0] - h[0]) / 1e3, (cv[i * 4 + 1] - h[0]) / 1e3,
                  (cv[i * 4 + 2] - h[0]) / 1e3);
        fclose(fp);
      }
    }
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  for (auto p : mats)
    if (p) cudaFree(p);
  cudaFree(x);
  cudaFree(part);
  cudaFree(out);
  cudaFree(cnt);
  cudaFree(bacc);
  Q.release();
  cudaStreamDestroy(s);
  return rc;
}

}  // extern "C"
