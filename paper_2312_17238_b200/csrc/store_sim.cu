// Host execution of the device store (store_dev.cuh) for CPU tests and the
// expert-parallel ownership logic: the same store:: functions the k_tail /
// k_prefill_bk kernels run, on host memory, with the copy mailbox drained
// synchronously into a per-buffer "contents" table so tests can check that
// every routed buffer really holds the expert it was resolved for.
#include <cstring>
#include <string>
#include <vector>

#include "copy_sched.h"
#include "kernels.cuh"

struct moe_store_sim {
  StoreDev S{};
  std::vector<int> lru, lru_len, res_buf, stg_layer, stg_exp, stg_stamp, stg_buf, scalars,
      free_stack, pending;
  std::vector<long long> seq;
  std::vector<uint32_t> gen;
  std::vector<DevEvent> ev;
  std::vector<unsigned char> owned;
  std::vector<int> content;  // buffer -> layer*E + expert last copied into it
  std::vector<uint32_t> flag;  // buffer -> last published generation (ready flag)
  Mailbox* mb = nullptr;
  unsigned long long tail = 0;
  int err = 0;
  int64_t copies = 0, chunks = 0;
  // copy-engine simulation: the engine's CopySched policy; `progress` chunks
  // run after every bookkeeping call, then the consumer (the GEMVs) pulls
  // chunks until its buffers are ready.  A consumer that can never be
  // satisfied is a copy-engine deadlock.
  CopySched sched;
  int progress = 1 << 30;  // default: every request completes immediately
  void drain() {
    for (;;) {
      const CopyReq& r = mb->ring[tail % MOE_MAILBOX_CAP];
      if (__atomic_load_n(&r.stamp, __ATOMIC_ACQUIRE) != (uint32_t)(tail + 1)) break;
      const int kind = (r.layer >> 24) & 0xff, layer = r.layer & 0xffffff;
      sched.on_request(kind, req_buf(r), layer, req_expert(r), r.gen);
      if (kind != MOE_COPY_PROMOTE) ++copies;
      ++tail;
    }
  }
  bool step() {  // execute one chunk
    CopySched::Chunk c;
    if (!sched.next(&c)) return false;
    ++chunks;
    if (c.last) {
      content[c.buf] = c.layer * S.E + c.expert;
      flag[c.buf] = c.gen;
    }
    return true;
  }
  void run(int n) {
    for (int i = 0; i < n && step(); ++i) {
    }
  }
  bool consume(int buf, uint32_t gen) {  // GEMV wait on (buf, gen)
    while ((int)(flag[buf] - gen) < 0)
      if (!step()) return false;
    return true;
  }
  ~moe_store_sim() { delete mb; }
};

namespace {
thread_local std::string s_err;
int sfail(int code, const char* m) {
  s_err = m;
  return code;
}
int err_status(moe_store_sim* s) {
  const int e = s->err;
  s->err = 0;
  if (e & MOE_ERRF_UNKNOWN) return sfail(MOE_ERR_UNKNOWN_EXPERT, "no such expert");
  if (e & (MOE_ERRF_ALLOC | MOE_ERRF_EVENTS)) return sfail(MOE_ERR_RUNTIME, "store overflow");
  return MOE_OK;
}
}  // namespace

extern "C" {

int moe_store_sim_create(int32_t n_layers, int32_t n_experts, int32_t k, int32_t b,
                         int64_t expert_bytes, int32_t top_k, int32_t m,
                         const uint8_t* owned, moe_store_sim** out) {
  if (!out || n_layers < 1 || n_experts < 1 || n_experts > 64 || k < 0 || b < 0 ||
      top_k < 1 || top_k > MOE_MAX_TOPK || m < 0 || expert_bytes <= 0)
    return sfail(MOE_ERR_VALUE, "bad store geometry");
  if (k > n_experts) return sfail(MOE_ERR_VALUE, "k exceeds experts per layer");
  auto* s = new moe_store_sim();
  const int L = n_layers, E = n_experts, kk = k > 1 ? k : 1, bb = b > 1 ? b : 1;
  // same buffer budget as moe_finalize: L*k resident + b staged + transients
  const int nbuf = L * k + b + E + k + m + 2;
  s->lru.assign((size_t)L * kk, -1);
  s->lru_len.assign(L, 0);
  s->res_buf.assign((size_t)L * E, -1);
  s->stg_layer.assign(bb, -1);
  s->stg_exp.assign(bb, -1);
  s->stg_stamp.assign(bb, 0);
  s->stg_buf.assign(bb, -1);
  s->scalars.assign(4, 0);
  s->scalars[1] = nbuf;
  s->free_stack.resize(nbuf);
  for (int i = 0; i < nbuf; ++i) s->free_stack[i] = nbuf - 1 - i;
  s->pending.assign(nbuf, 0);
  s->seq.assign(2, 0);
  s->gen.assign(nbuf, 0);
  s->content.assign(nbuf, -1);
  s->flag.assign(nbuf, 0u);
  s->sched.init(nbuf, 1, 1);
  s->ev.resize(1 << 20);
  if (owned) s->owned.assign(owned, owned + (size_t)L * E);
  s->mb = new Mailbox();
  memset(s->mb, 0, sizeof(Mailbox));
  StoreDev& S = s->S;
  S.L = L;
  S.E = E;
  S.k = k;
  S.b = b;
  S.top_k = top_k;
  S.nbuf = nbuf;
  S.expert_bytes = expert_bytes;
  S.lru = s->lru.data();
  S.lru_len = s->lru_len.data();
  S.res_buf = s->res_buf.data();
  S.stg_layer = s->stg_layer.data();
  S.stg_exp = s->stg_exp.data();
  S.stg_stamp = s->stg_stamp.data();
  S.stg_buf = s->stg_buf.data();
  S.scalars = s->scalars.data();
  S.seq = s->seq.data();
  S.free_stack = s->free_stack.data();
  S.pending = s->pending.data();
  S.gen = s->gen.data();
  S.ev = s->ev.data();
  S.ev_cap = (int)s->ev.size();
  S.mb = s->mb;
  S.owned = owned ? s->owned.data() : nullptr;
  S.err = &s->err;
  S.flags = s->flag.data();
  *out = s;
  return MOE_OK;
}

int moe_store_sim_token(moe_store_sim* s, int32_t layer, int32_t pos, const int32_t* experts,
                        int32_t k, const int32_t* guesses, int32_t m, int32_t guess_layer,
                        int32_t* bufs_out) {
  if (!s || k < 0 || k > MOE_MAX_TOPK || m < 0 || m > 16)
    return sfail(MOE_ERR_VALUE, "bad arguments");
  if (m > s->S.b && guess_layer >= 0)
    return sfail(MOE_ERR_VALUE, "speculative keys exceed b buffers");
  int bufs[MOE_MAX_TOPK];
  uint32_t gens[MOE_MAX_TOPK];
  store::resolve_token(s->S, layer, experts, k, guesses, m, guess_layer, pos, bufs, gens);
  s->drain();
  s->run(s->progress);
  for (int j = 0; j < k; ++j)
    if (bufs[j] >= 0 && !s->consume(bufs[j], gens[j]))
      return sfail(MOE_ERR_TIMEOUT, "copy engine deadlock: routed buffer never published");
  if (bufs_out)
    for (int j = 0; j < k; ++j) bufs_out[j] = bufs[j];
  return err_status(s);
}

int moe_store_sim_prefill(moe_store_sim* s, int32_t layer, const int32_t* experts, int32_t n,
                          int32_t k, int32_t* bufs_out) {
  if (!s || n < 1 || k < 1 || k > MOE_MAX_TOPK) return sfail(MOE_ERR_VALUE, "bad arguments");
  std::vector<int> bb((size_t)n * k);
  std::vector<uint32_t> gg((size_t)n * k);
  store::resolve_prefill(
      s->S, layer, n, k, [&](int p, int j) { return (int)experts[p * k + j]; },
      [&](int p, int j, int b, uint32_t g) {
        bb[p * k + j] = b;
        gg[p * k + j] = g;
      });
  s->drain();
  s->run(s->progress);
  for (size_t i = 0; i < bb.size(); ++i)
    if (bb[i] >= 0 && !s->consume(bb[i], gg[i]))
      return sfail(MOE_ERR_TIMEOUT, "copy engine deadlock: routed buffer never published");
  if (bufs_out)
    for (size_t i = 0; i < bb.size(); ++i) bufs_out[i] = bb[i];
  return err_status(s);
}

int64_t moe_store_sim_num_events(moe_store_sim* s) { return s ? s->scalars[3] : 0; }

int moe_store_sim_events(moe_store_sim* s, moe_event* out, int64_t cap) {
  if (!s) return sfail(MOE_ERR_VALUE, "null store");
  const int64_t n = s->scalars[3] < cap ? s->scalars[3] : cap;
  if (n > 0) memcpy(out, s->ev.data(), (size_t)n * sizeof(moe_event));
  return MOE_OK;
}

// lru_out[l*k+i] (MRU first, -1 pad), staged_out[b] (layer*E+expert or -1),
// buf contents: content_out[nbuf] (layer*E+expert last copied, -1 never);
// res_buf_out[L*E] physical buffer of each resident key (-1 otherwise);
// stg_buf_out[b].  Any pointer may be NULL.
int moe_store_sim_state(moe_store_sim* s, int32_t* lru_out, int32_t* staged_out,
                        int32_t* content_out, int32_t* res_buf_out, int32_t* stg_buf_out,
                        int32_t* nbuf_out) {
  if (!s) return sfail(MOE_ERR_VALUE, "null store");
  const StoreDev& S = s->S;
  const int kk = S.k > 1 ? S.k : 1;
  if (lru_out)
    for (int l = 0; l < S.L; ++l)
      for (int i = 0; i < S.k; ++i)
        lru_out[l * S.k + i] = i < S.lru_len[l] ? S.lru[l * kk + i] : -1;
  for (int i = 0; i < S.b; ++i) {
    if (staged_out) staged_out[i] = S.stg_layer[i] >= 0 ? S.stg_layer[i] * S.E + S.stg_exp[i] : -1;
    if (stg_buf_out) stg_buf_out[i] = S.stg_layer[i] >= 0 ? S.stg_buf[i] : -1;
  }
  if (content_out)
    for (int i = 0; i < S.nbuf; ++i) content_out[i] = s->content[i];
  if (res_buf_out)
    for (int l = 0; l < S.L; ++l)
      for (int e = 0; e < S.E; ++e) {
        bool res = false;
        for (int i = 0; i < S.lru_len[l]; ++i) res |= S.lru[l * kk + i] == e;
        res_buf_out[l * S.E + e] = res ? S.res_buf[l * S.E + e] : -1;
      }
  if (nbuf_out) *nbuf_out = S.nbuf;
  return MOE_OK;
}

int64_t moe_store_sim_copies(moe_store_sim* s) { return s ? s->copies : 0; }

int moe_store_sim_copy_policy(moe_store_sim* s, int64_t job_bytes, int64_t chunk_bytes,
                              int32_t progress) {
  if (!s || job_bytes < 1 || chunk_bytes < 0 || progress < 0)
    return sfail(MOE_ERR_VALUE, "bad copy policy");
  s->sched.init(s->S.nbuf, (size_t)job_bytes, (size_t)chunk_bytes);
  s->progress = progress;
  return MOE_OK;
}

int64_t moe_store_sim_chunks(moe_store_sim* s) { return s ? s->chunks : 0; }

int64_t moe_store_sim_parked(moe_store_sim* s) { return s ? s->sched.n_parked : 0; }

int moe_store_sim_set_park(moe_store_sim* s, int32_t on) {
  if (!s) return sfail(MOE_ERR_VALUE, "null simulator");
  s->sched.park = on != 0;
  return MOE_OK;
}

const char* moe_store_sim_last_error(void) { return s_err.c_str(); }

int moe_store_sim_destroy(moe_store_sim* s) {
  delete s;
  return MOE_OK;
}

}  // extern "C"
