// Device-resident expert store: the exact semantics of the reference
// TieredExpertStore (store.py:76-220) executed by one thread on the GPU, plus
// the physical side the reference never sees: a pool of HBM expert buffers,
// per-buffer copy generations, and a copy-request mailbox in mapped pinned
// memory that the host copy engine drains (cudaMemcpyAsync + stream write of
// the buffer's ready flag).
//
// Logical state (must match the reference exactly): per-layer MRU-first LRU
// lists (<= k), b staging slots with stamps, the event sequence.
// Physical state: every resident / staged expert owns one buffer.  Buffers
// released during a bookkeeping call (evictions, k=0 transients, replaced
// staging entries) are only recycled at the next call, i.e. after the expert
// compute of the current layer has finished in stream order.
#pragma once
#include "common.cuh"
#include "../../include/moeb200.h"

#define MOE_ERRF_NONFINITE_GATE 1
#define MOE_ERRF_NONFINITE_LOGITS 2
#define MOE_ERRF_ALLOC 4
#define MOE_ERRF_EVENTS 8
#define MOE_ERRF_TIMEOUT 16
#define MOE_ERRF_UNKNOWN 32

#define MOE_MAX_TOPK 4
#define MOE_MAILBOX_CAP 65536

struct DevEvent {  // layout identical to moe_event
  long long seq;
  int kind, layer, expert, pos;
  long long bytes;
};

// copy request kinds (packed into CopyReq::layer bits 24..31)
#define MOE_COPY_DEMAND 0   // MISS_LOAD: the current layer waits for it
#define MOE_COPY_SPEC 1     // SPECULATIVE_LOAD: best effort, lowest priority
#define MOE_COPY_PROMOTE 2  // STAGING_HIT on a staged buffer whose copy may be pending

// One 16-byte mailbox entry, written by the device with a single vector store
// and validated by the host through its stamp (= entry index + 1): the host
// never relies on the ordering of separate PCIe writes.
struct CopyReq {
  int buf;        // bits 0..15 buffer, 16..31 expert
  int layer;      // bits 0..23 layer, 24..31 kind
  uint32_t gen;   // buffer generation
  uint32_t stamp; // (index + 1) mod 2^32
};
__host__ __device__ inline int req_buf(const CopyReq& r) { return r.buf & 0xffff; }
__host__ __device__ inline int req_expert(const CopyReq& r) { return (r.buf >> 16) & 0xffff; }

struct Mailbox {
  unsigned long long pad[16];
  CopyReq ring[MOE_MAILBOX_CAP];
};

struct RouteRec {  // per position: resolved experts of the current layer
  int e[MOE_MAX_TOPK];
  int buf[MOE_MAX_TOPK];
  uint32_t gen[MOE_MAX_TOPK];
  float w[MOE_MAX_TOPK];
  int ready[MOE_MAX_TOPK];  // decode: the tail saw flags[buf] >= gen (no flag wait needed)
};

struct TraceRecDev {  // layout identical to moe_trace_rec
  int pos, layer;
  int experts[8];
  float weights[8];
};

struct StoreDev {
  int L, E, k, b, top_k, nbuf;
  long long expert_bytes;
  int* lru;        // [L][max(k,1)] MRU first
  int* lru_len;    // [L]
  int* res_buf;    // [L][E]
  int* stg_layer;  // [b] (-1 = empty)
  int* stg_exp;
  int* stg_stamp;
  int* stg_buf;
  int* scalars;    // [0]=stamp [1]=nfree [2]=npending [3]=nev
  long long* seq;  // [0] event seq, [1] mailbox head (entries posted)
  int* free_stack;
  int* pending;
  uint32_t* gen;  // [nbuf]
  DevEvent* ev;
  int ev_cap;
  Mailbox* mb;    // device-mapped pointer
  const unsigned char* owned;  // [L][E] or null (expert parallel subset)
  int* err;
  const volatile uint32_t* flags;  // buffer ready generations (null: host simulator)
  int* state_base;  // contiguous block holding every array above except ev (device)
  int state_ints;
};

// Every store operation is __host__ __device__: the engine runs it on one GPU
// thread (k_tail / k_prefill_bk); the host simulator (store_sim.cu) runs the
// very same code on the CPU so the bookkeeping is testable without a GPU.
#define MOE_HD __host__ __device__ __forceinline__

namespace store {

MOE_HD void flag_err(StoreDev& S, int f) {
#ifdef __CUDA_ARCH__
  atomicOr(S.err, f);
#else
  __atomic_fetch_or(S.err, f, __ATOMIC_RELAXED);
#endif
}

MOE_HD void fence_system() {
#ifdef __CUDA_ARCH__
  fence_system();
#else
  __atomic_thread_fence(__ATOMIC_SEQ_CST);
#endif
}

MOE_HD void begin_call(StoreDev& S) {
  int nf = S.scalars[1];
  const int np = S.scalars[2];
  for (int i = 0; i < np; ++i) S.free_stack[nf++] = S.pending[i];
  S.scalars[1] = nf;
  S.scalars[2] = 0;
}

MOE_HD void emit(StoreDev& S, int kind, int l, int e, int pos, bool moved) {
  const long long sq = S.seq[0]++;
  const int n = S.scalars[3];
  if (n >= S.ev_cap) {
    flag_err(S, MOE_ERRF_EVENTS);
    return;
  }
  DevEvent ev;
  ev.seq = sq;
  ev.kind = kind;
  ev.layer = l;
  ev.expert = e;
  ev.pos = pos;
  ev.bytes = moved ? S.expert_bytes : 0;
  S.ev[n] = ev;
  S.scalars[3] = n + 1;
}

MOE_HD int alloc_buf(StoreDev& S) {
  const int nf = S.scalars[1];
  if (nf <= 0) {
    flag_err(S, MOE_ERRF_ALLOC);
    return 0;
  }
  S.scalars[1] = nf - 1;
  return S.free_stack[nf - 1];
}

MOE_HD void release(StoreDev& S, int buf) { S.pending[S.scalars[2]++] = buf; }

MOE_HD void post(StoreDev& S, int buf, int l, int e, uint32_t g, int kind) {
  const unsigned long long h = (unsigned long long)S.seq[1]++;  // device-side mailbox head
  CopyReq* slot = &S.mb->ring[h % MOE_MAILBOX_CAP];
  const uint32_t w0 = (uint32_t)(buf & 0xffff) | ((uint32_t)(e & 0xffff) << 16);
  const uint32_t w1 = (uint32_t)l | ((uint32_t)kind << 24);
  const uint32_t stamp = (uint32_t)(h + 1);
#ifdef __CUDA_ARCH__
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(slot), "r"(w0), "r"(w1),
               "r"(g), "r"(stamp)
               : "memory");
#else
  slot->buf = (int)w0;
  slot->layer = (int)w1;
  slot->gen = g;
  __atomic_store_n(&slot->stamp, stamp, __ATOMIC_RELEASE);
#endif
  // no system fence: the host validates each entry by its stamp, so nothing
  // depends on the order in which separate posted writes become visible
}

MOE_HD void issue_copy(StoreDev& S, int buf, int l, int e, int kind) {
  post(S, buf, l, e, ++S.gen[buf], kind);
}

MOE_HD int lru_find(const StoreDev& S, int l, int e) {
  const int* lst = S.lru + l * (S.k > 1 ? S.k : 1);
  const int n = S.lru_len[l];
  for (int i = 0; i < n; ++i)
    if (lst[i] == e) return i;
  return -1;
}

MOE_HD int staged_at(const StoreDev& S, int l, int e) {
  for (int i = 0; i < S.b; ++i)
    if (S.stg_layer[i] == l && S.stg_exp[i] == e) return i;
  return -1;
}

// store.py:148-153 _insert_resident
MOE_HD void make_resident(StoreDev& S, int l, int e, int buf, int pos) {
  int* lst = S.lru + l * (S.k > 1 ? S.k : 1);
  int n = S.lru_len[l];
  int evicted = -1;
  if (n == S.k) {  // list full: the LRU tail leaves after the insert
    evicted = lst[n - 1];
    --n;
  }
  for (int i = n; i > 0; --i) lst[i] = lst[i - 1];
  lst[0] = e;
  S.lru_len[l] = n + 1;
  S.res_buf[l * S.E + e] = buf;
  if (evicted >= 0) {
    emit(S, MOE_EV_EVICT_TO_HOST, l, evicted, pos, true);
    release(S, S.res_buf[l * S.E + evicted]);
  }
}

MOE_HD bool key_ok(const StoreDev& S, int l, int e) {
  if (l < 0 || l >= S.L || e < 0 || e >= S.E) return false;
  return S.owned == nullptr || S.owned[l * S.E + e];
}

// store.py:157-186 acquire; returns the physical buffer holding the expert
MOE_HD int acquire(StoreDev& S, int l, int e, int pos) {
  if (!key_ok(S, l, e)) {
    flag_err(S, MOE_ERRF_UNKNOWN);
    return 0;
  }
  const int idx = lru_find(S, l, e);
  if (idx >= 0) {
    int* lst = S.lru + l * (S.k > 1 ? S.k : 1);
    for (int i = idx; i > 0; --i) lst[i] = lst[i - 1];
    lst[0] = e;
    emit(S, MOE_EV_HIT, l, e, pos, false);
    return S.res_buf[l * S.E + e];
  }
  const int s = staged_at(S, l, e);
  if (s >= 0) {
    emit(S, MOE_EV_STAGING_HIT, l, e, pos, false);
    const int buf = S.stg_buf[s];
    // the speculative copy may still be queued behind demand copies: promote it
    if (S.flags == nullptr || (int)(S.flags[buf] - S.gen[buf]) < 0)
      post(S, buf, l, e, S.gen[buf], MOE_COPY_PROMOTE);
    S.stg_layer[s] = -1;
    S.stg_exp[s] = -1;
    if (S.k > 0) {
      emit(S, MOE_EV_PROMOTE_FROM_STAGING, l, e, pos, false);
      make_resident(S, l, e, buf, pos);
    } else {
      release(S, buf);
    }
    return buf;
  }
  emit(S, MOE_EV_MISS_LOAD, l, e, pos, true);
  const int buf = alloc_buf(S);
  issue_copy(S, buf, l, e, MOE_COPY_DEMAND);
  if (S.k > 0)
    make_resident(S, l, e, buf, pos);
  else
    release(S, buf);
  return buf;
}

// store.py:188-220 speculative_load (keys of one target layer)
MOE_HD void speculative_load(StoreDev& S, int tl, const int* es, int m, int pos, int cur_layer) {
  for (int j = 0; j < m; ++j) {
    const int e = es[j];
    if (!key_ok(S, tl, e)) continue;  // EP: other ranks own it
    if (lru_find(S, tl, e) >= 0 || staged_at(S, tl, e) >= 0) continue;
    int slot = -1;
    for (int i = 0; i < S.b; ++i)
      if (S.stg_layer[i] < 0) {
        slot = i;
        break;
      }
    if (slot < 0) {
      int best = 0x7fffffff;
      for (int i = 0; i < S.b; ++i)
        if (S.stg_layer[i] != cur_layer && S.stg_stamp[i] < best) {
          best = S.stg_stamp[i];
          slot = i;
        }
      if (slot < 0) continue;
      release(S, S.stg_buf[slot]);
    }
    const int buf = alloc_buf(S);
    issue_copy(S, buf, tl, e, MOE_COPY_SPEC);
    S.stg_layer[slot] = tl;
    S.stg_exp[slot] = e;
    S.stg_stamp[slot] = S.scalars[0]++;
    S.stg_buf[slot] = buf;
    emit(S, MOE_EV_SPECULATIVE_LOAD, tl, e, pos, true);
  }
}

// ---- shared-memory staging of the store state for the bookkeeping kernels:
// the single bookkeeping thread does a few hundred dependent accesses per
// layer; on shared memory they cost ~30 cycles instead of an L2 round trip.
MOE_HD int stage_ints(const StoreDev& S) { return S.state_ints; }

#ifdef __CUDACC__
// All the store arrays except the event log live in one contiguous block
// (state_base, state_ints); the bookkeeping kernels copy it to shared memory
// with one coalesced pass and rebase every pointer into the copy.
template <class T>
__device__ __forceinline__ T* rebase(T* p, const int* from, int* to) {
  return reinterpret_cast<T*>(reinterpret_cast<char*>(to) +
                              (reinterpret_cast<const char*>(p) -
                               reinterpret_cast<const char*>(from)));
}

// the store G with every state pointer rebased into the shared copy `sm`
__device__ __forceinline__ StoreDev stage_view(const StoreDev& G, int* sm) {
  StoreDev V = G;
  V.lru = rebase(G.lru, G.state_base, sm);
  V.lru_len = rebase(G.lru_len, G.state_base, sm);
  V.res_buf = rebase(G.res_buf, G.state_base, sm);
  V.stg_layer = rebase(G.stg_layer, G.state_base, sm);
  V.stg_exp = rebase(G.stg_exp, G.state_base, sm);
  V.stg_stamp = rebase(G.stg_stamp, G.state_base, sm);
  V.stg_buf = rebase(G.stg_buf, G.state_base, sm);
  V.scalars = rebase(G.scalars, G.state_base, sm);
  V.seq = rebase(G.seq, G.state_base, sm);
  V.free_stack = rebase(G.free_stack, G.state_base, sm);
  V.pending = rebase(G.pending, G.state_base, sm);
  V.gen = rebase(G.gen, G.state_base, sm);
  return V;
}

// all threads: copy the state of global store G to `sm` (16-byte aligned)
// and return the view backed by it (caller synchronizes before use)
__device__ __forceinline__ StoreDev stage_in(const StoreDev& G, int* sm) {
  const int n4 = G.state_ints >> 2;
  const int4* src = reinterpret_cast<const int4*>(G.state_base);
  int4* dst = reinterpret_cast<int4*>(sm);
  for (int i = threadIdx.x; i < n4; i += blockDim.x) dst[i] = __ldcg(src + i);
  for (int i = 4 * n4 + threadIdx.x; i < G.state_ints; i += blockDim.x)
    sm[i] = __ldcg(G.state_base + i);
  return stage_view(G, sm);
}

// all threads: write the staged state back
__device__ __forceinline__ void stage_out(const StoreDev& G, const int* sm) {
  const int n4 = G.state_ints >> 2;
  const int4* src = reinterpret_cast<const int4*>(sm);
  int4* dst = reinterpret_cast<int4*>(G.state_base);
  for (int i = threadIdx.x; i < n4; i += blockDim.x) dst[i] = src[i];
  for (int i = 4 * n4 + threadIdx.x; i < G.state_ints; i += blockDim.x) G.state_base[i] = sm[i];
}
#endif

// One decode layer's bookkeeping, in the order of OffloadEngine._resolve_token
// (engine.py:222-231): acquire the selected experts in descending-weight
// order, then speculative_load the top-m guesses for layer + lookahead.
// bufs/gens receive the physical buffer (and its copy generation) of each
// selected expert; -1 for experts another EP rank owns.
struct NoMark {
  MOE_HD void operator()(int) const {}
};

// mark(i) after each step (profiling: 1 begin_call, 2 + j acquire j, 6 speculation)
template <class Mark = NoMark>
MOE_HD void resolve_token(StoreDev& S, int layer, const int* sel, int k, const int* guesses,
                          int m, int guess_layer, int pos, int* bufs, uint32_t* gens,
                          Mark mark = Mark()) {
  begin_call(S);
  mark(1);
  for (int j = 0; j < k; ++j) {
    const bool in_range = layer >= 0 && layer < S.L && sel[j] >= 0 && sel[j] < S.E;
    // out of range -> UnknownExpertError; in range but another rank's -> -1
    bufs[j] = (!in_range || key_ok(S, layer, sel[j])) ? acquire(S, layer, sel[j], pos) : -1;
    mark(2 + (j < 3 ? j : 3));
  }
  if (guess_layer >= 0 && m > 0) speculative_load(S, guess_layer, guesses, m, pos, layer);
  for (int j = 0; j < k; ++j) gens[j] = bufs[j] >= 0 ? S.gen[bufs[j]] : 0u;
  mark(6);
}

// One prefill layer (engine.py:233-240): every distinct expert acquired once,
// first-use order over (position, descending weight), no speculation.
// get(p, j) -> routed expert id; put(p, j, buf, gen) receives the buffer.
#pragma nv_exec_check_disable
template <class Get, class Put>
MOE_HD void resolve_prefill(StoreDev& S, int layer, int n, int k, Get get, Put put) {
  begin_call(S);
  int table[64];
  for (int e = 0; e < 64; ++e) table[e] = -2;
  for (int p = 0; p < n; ++p)
    for (int j = 0; j < k; ++j) {
      const int e = get(p, j);
      if (e < 0 || table[e] != -2) continue;
      table[e] = key_ok(S, layer, e) ? acquire(S, layer, e, p) : -1;
    }
  for (int p = 0; p < n; ++p)
    for (int j = 0; j < k; ++j) {
      const int e = get(p, j);
      const int b = e >= 0 ? table[e] : -1;
      put(p, j, b, b >= 0 ? S.gen[b] : 0u);
    }
}

}  // namespace store
