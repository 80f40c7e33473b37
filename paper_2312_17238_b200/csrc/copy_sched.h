// Copy-engine scheduling policy (host side), shared by the engine's copier
// thread and the CPU store simulator so the policy is unit-testable.
//
// Requests come from the device store through the mailbox (store_dev.cuh):
//   DEMAND  (MISS_LOAD)         the current layer's GEMVs wait for it
//   SPEC    (SPECULATIVE_LOAD)  best effort
//   PROMOTE (STAGING_HIT)       a staged buffer is needed now
// Policy: demand jobs first (FIFO), then speculative jobs newest-first; a
// promoted speculative job joins the demand queue.  Speculative jobs are
// issued in small chunks so a demand copy waits at most one small chunk
// behind speculation; demand jobs go out whole (nothing may preempt them).
// A job whose buffer has since been re-requested with a newer generation is
// stale (its staging entry was replaced and the buffer reassigned) and is
// dropped.  A speculative job whose target layer has been passed (a later
// request comes from a later point of the decode: a demand for a later layer,
// a speculation issued at or after the target layer, or a new token) is
// parked: its remaining chunks are not copied unless a staging hit promotes
// it.  On a saturated host link, copies of guesses the token has already
// gone past only delay the demand copies that follow.
#pragma once
#include <cstddef>
#include <cstdint>
#include <deque>
#include <vector>

struct CopySched {
  struct Job {
    int buf, layer, expert;
    uint32_t gen;
    size_t off;
  };
  struct Chunk {
    int buf, layer, expert;
    uint32_t gen;
    size_t off, bytes;
    bool last;  // the job is complete after this chunk: publish `gen`
  };
  std::deque<Job> demand;
  std::vector<Job> spec;
  std::vector<Job> parked;  // speculative jobs whose target layer has passed
  std::vector<uint32_t> latest;
  size_t xbytes = 0, chunk = 0;
  int lookahead = 1;
  bool park = true;
  int64_t n_parked = 0;

  void init(int nbuf, size_t job_bytes, size_t chunk_bytes, int spec_lookahead = 1) {
    latest.assign(nbuf, 0u);
    xbytes = job_bytes;
    chunk = chunk_bytes ? chunk_bytes : job_bytes;
    lookahead = spec_lookahead > 0 ? spec_lookahead : 1;
    demand.clear();
    spec.clear();
    parked.clear();
  }

  // Does a new request (kind, layer) come from past speculative job j's target
  // layer?  Requests arrive in decode order: within a layer the acquires
  // (demand / promote of that layer) precede its speculation (for layer +
  // lookahead), layers ascend within a token and restart at the next token.
  bool passed(const Job& j, int kind, int layer) const {
    const int issue = kind == 1 ? layer - lookahead : layer;  // layer that posted it
    const int jissue = j.layer - lookahead;
    if (issue < jissue) return true;                   // a later token
    return kind == 1 ? issue >= j.layer : layer > j.layer;
  }

  // kind: 0 demand, 1 speculative, 2 promote (store_dev.cuh MOE_COPY_*)
  void on_request(int kind, int buf, int layer, int expert, uint32_t gen) {
    if (park)
      for (size_t i = 0; i < spec.size();) {
        if (passed(spec[i], kind, layer) && !(kind == 2 && spec[i].buf == buf)) {
          parked.push_back(spec[i]);
          spec.erase(spec.begin() + (long)i);
          ++n_parked;
        } else {
          ++i;
        }
      }
    if (kind == 2) {
      for (auto* q : {&spec, &parked})
        for (size_t i = 0; i < q->size(); ++i)
          if ((*q)[i].buf == buf && (*q)[i].gen == gen) {
            demand.push_back((*q)[i]);
            q->erase(q->begin() + (long)i);
            return;
          }
      return;
    }
    latest[buf] = gen;
    const Job j{buf, layer, expert, gen, 0};
    if (kind == 0)
      demand.push_back(j);
    else
      spec.push_back(j);
  }

  bool stale(const Job& j) const { return j.gen != latest[j.buf]; }

  bool empty() const { return demand.empty() && spec.empty(); }  // parked jobs wait

  void drop_stale() {
    while (!demand.empty() && stale(demand.front())) demand.pop_front();
    while (!spec.empty() && stale(spec.back())) spec.pop_back();
    for (size_t i = 0; i < parked.size();)
      if (stale(parked[i]))
        parked.erase(parked.begin() + (long)i);
      else
        ++i;
  }

  bool has_demand() {
    drop_stale();
    return !demand.empty();
  }

  // next chunk of the front demand job (whole remainder) or of the newest
  // speculative job (one `chunk`)
  bool next_demand(Chunk* c) {
    drop_stale();
    return !demand.empty() && take(&demand.front(), true, c);
  }
  bool next_spec(Chunk* c) {
    drop_stale();
    return !spec.empty() && take(&spec.back(), false, c);
  }

  // next chunk to issue under the single-stream policy, or false when idle
  bool next(Chunk* c) { return next_demand(c) || next_spec(c); }

 private:
  bool take(Job* j, bool from_demand, Chunk* c) {
    const size_t left = xbytes - j->off;
    const size_t n = from_demand ? left : (chunk < left ? chunk : left);
    *c = Chunk{j->buf, j->layer, j->expert, j->gen, j->off, n, j->off + n == xbytes};
    j->off += n;
    if (c->last) {
      if (from_demand)
        demand.pop_front();
      else
        spec.pop_back();
    }
    return true;
  }
};
