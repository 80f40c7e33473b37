"""Mixtral-width (2 layers) engine vs oracle: prefill hidden states, routing,
logits and decision margins (GPU debug aid)."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from oracle import cpu_bench  # noqa: E402
from oracle import engine as OE  # noqa: E402
from oracle import model as OM  # noqa: E402
from oracle.store import CacheConfig as OCache  # noqa: E402


def main(ebits=3, k=4, m=0, ntok=3, nprompt=3):
    from paper_2312_17238_b200 import CacheConfig, OffloadEngine, SpeculationConfig
    from paper_2312_17238_b200 import synthetic_model
    cfg_full = bench.cfg_obj(bench.MIXTRAL)
    dquant, dsynth = bench.device_helpers()
    model, pay = cpu_bench.build_sample(dquant, dsynth, cfg_full, 0, 4, ebits, n_layers_sample=2)
    cfg2 = model.config
    prompt = [int(t) for t in np.random.default_rng(0).integers(0, cfg2.vocab_size, nprompt)]
    ref = cpu_bench.ParallelOffloadEngine(model, OCache(k, 4), OE.SpeculationConfig(m > 0, max(m, 1)),
                                          payloads=pay, record_hidden=True)
    ref.pool = ThreadPoolExecutor(8)
    rpre = ref.prefill(prompt)
    eng = OffloadEngine(synthetic_model(cfg2, 0), CacheConfig(k=k, b=4),
                        SpeculationConfig(enabled=m > 0, m=max(m, 1)), record_hidden=True,
                        synth=(0, 4, ebits), expert_bytes=bench.expert_bytes(bench.MIXTRAL, ebits))
    gpre = eng.prefill(prompt)
    rrec = ref.sorted_records()
    grec = eng.trace().records
    for a, b in zip(rrec, grec):
        dh = float(np.abs(a.hidden - b.hidden).max())
        sc = float(np.abs(a.hidden).max())
        lg = a.hidden @ model.params[f"layers.{a.layer}.gate"]
        srt = np.sort(lg)[::-1]
        print(f"pos {a.token_pos} layer {a.layer}: ref {a.experts} got {b.experts} "
              f"|dh|={dh:.3e} (max|h| {sc:.3e}) gate top3 {srt[:3]} margin23 {srt[1]-srt[2]:.3e} "
              f"w ref {a.weights} got {b.weights}")
    for p in range(len(prompt)):
        d = float(np.abs(rpre[p] - gpre[p]).max())
        ra, ga = int(np.argmax(rpre[p])), int(np.argmax(gpre[p]))
        s = np.sort(rpre[p])[::-1]
        print(f"prefill logits pos {p}: max|d| {d:.3e} max|ref| {np.abs(rpre[p]).max():.3e} "
              f"argmax ref {ra} got {ga} top2 margin {s[0]-s[1]:.3e}")
    ev_r = ref.events
    ev_g = [(e.seq, e.kind, e.key.layer, e.key.expert, e.token_pos, e.bytes_moved) for e in eng.events]
    print("prefill events equal:", ev_r == ev_g, len(ev_r), len(ev_g))
    rt, rl = ref.decode(ntok)
    res = eng.decode(ntok)
    print("decode tokens ref", rt, "got", res.tokens)
    rrec = {(r.token_pos, r.layer): r for r in ref.sorted_records()}
    for b in res.trace.records:
        a = rrec.get((b.token_pos, b.layer))
        if a is None or b.token_pos < nprompt:
            continue
        nl = b.layer + 1
        if nl < cfg2.n_layers:
            G = model.params[f"layers.{nl}.gate"]
            la, lb = a.hidden @ G, b.hidden @ G
            ta, tb = OM.top_k(la, 3), OM.top_k(lb, 3)
            print(f"pos {b.token_pos} layer {b.layer}: guess ref {ta.tolist()} {np.sort(la)[::-1][:3]} "
                  f"got {tb.tolist()} {np.sort(lb)[::-1][:3]} |dh| {np.abs(a.hidden-b.hidden).max():.2e}")
    ev_r = ref.events
    ev_g = [(e.seq, e.kind, e.key.layer, e.key.expert, e.token_pos, e.bytes_moved) for e in eng.events]
    for i, (x, y) in enumerate(zip(ev_r, ev_g)):
        if x != y:
            print("first event diff at", i, "ref", x, "got", y)
            print("ref around:", ev_r[max(0, i - 4):i + 3])
            print("got around:", ev_g[max(0, i - 4):i + 3])
            break
    ref.pool.shutdown()


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
