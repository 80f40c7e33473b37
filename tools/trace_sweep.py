"""§8(f)2: trace-driven cache / speculation studies on GPU-recorded traces.

Records device traces (routing + hidden states, ``OffloadEngine.trace()``) of
the Mixtral-shape model with the reference init weights on the B200 engine,
for the five §8(d) prompts (default_rng(s), s = 0..4, 16 tokens, 32 greedy
tokens), then on each trace:

  * replays the reference store with the reference's own ``replay``
    (engine.py:263-313) over k = 0..8 x m = 0..2 -> hit rate, misses,
    speculative loads and H2D bytes per generated token, and the H2D floor
    per token at the measured pinned->HBM peak;
  * replays the same decisions through the engine's device store code
    (``DeviceStoreSim``: store_dev.cuh run on the host) and checks the event
    logs equal the reference replay's, point by point;
  * ``guess_recall`` (engine.py:316-338) at lookahead {1, 2, 10}, m {1, 2, 4};
  * for prompt 0 (first session of a fresh engine) checks the reference
    replay of the device trace equals the live device event log.

    python tools/trace_sweep.py [--config c3] [--tokens 32] [--out gpurun_out/trace_sweep]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--tokens", type=int, default=32)
    ap.add_argument("--prompts", type=int, default=5)
    ap.add_argument("--ks", default="0,1,2,3,4,5,6,7,8")
    ap.add_argument("--ms", default="0,1,2")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "trace_sweep"))
    a = ap.parse_args()
    import bench
    from paper_2312_17238_b200 import CacheConfig, OffloadEngine, SpeculationConfig, _lib, weights
    from moe_offload.engine import guess_recall, replay
    from paper_2312_17238_b200.store_sim import replay_device

    ab, xb, k0, m0 = bench.CONFIGS[a.config]
    eb = bench.expert_bytes(bench.MIXTRAL, xb)
    t0 = time.time()
    model, attn, experts = weights.mixtral_model(ab, xb)
    eng = OffloadEngine(model, CacheConfig(k=k0, b=4, expert_bytes=eb),
                        SpeculationConfig(enabled=m0 > 0, m=max(m0, 1)), payloads=experts,
                        attn_blocks=attn, expert_bytes=eb, record_hidden=True)
    import ctypes as C
    best, med = C.c_double(), C.c_double()
    _lib.check(_lib.lib().moe_measure_h2d(eng._h, 8, C.byref(best), C.byref(med)))
    h2d = best.value
    print(f"[trace_sweep] engine ready in {time.time() - t0:.0f}s, h2d peak {h2d:.2f} GB/s",
          flush=True)
    traces, live_check = [], None
    for s in range(a.prompts):
        e0 = len(eng.events)
        eng.prefill(bench.prompt_of(s, bench.MIXTRAL["vocab_size"]))
        eng.decode(a.tokens)
        tr = eng.trace()
        traces.append(tr)
        if s == 0:  # fresh store: the reference replay must reproduce the live log
            rep = replay(tr, CacheConfig(k=k0, b=4, expert_bytes=eb),
                         SpeculationConfig(enabled=m0 > 0, m=max(m0, 1)))
            live_check = {"config": a.config, "k": k0, "m": m0,
                          "events": len(rep.events),
                          "equal": rep.events == eng.events[e0:]}
            print(f"[trace_sweep] live vs replay: {live_check}", flush=True)
    eng.close()

    ks = [int(x) for x in a.ks.split(",")]
    ms = [int(x) for x in a.ms.split(",")]
    grid = []
    for k in ks:
        for m in ms:
            if m > 4:
                continue
            agg = {"k": k, "m": m, "acquires": 0, "hits": 0, "miss_loads": 0, "spec_loads": 0,
                   "staging_hits": 0, "gen_tokens": 0, "device_store_equal": True}
            for tr in traces:
                cache = CacheConfig(k=k, b=4, expert_bytes=eb)
                spec = SpeculationConfig(enabled=m > 0, m=max(m, 1))
                rep = replay(tr, cache, spec)
                dev = replay_device(tr, cache, spec).events
                agg["device_store_equal"] &= (dev == rep.events)
                gen = [e for e in rep.events if e.token_pos >= tr.prompt_len]
                acq = [e for e in gen if e.kind in ("hit", "staging_hit", "miss_load")]
                agg["acquires"] += len(acq)
                agg["hits"] += sum(1 for e in acq if e.kind in ("hit", "staging_hit"))
                agg["miss_loads"] += sum(1 for e in gen if e.kind == "miss_load")
                agg["spec_loads"] += sum(1 for e in gen if e.kind == "speculative_load")
                agg["staging_hits"] += sum(1 for e in gen if e.kind == "staging_hit")
                agg["gen_tokens"] += len({e.token_pos for e in gen}) or a.tokens
            n = agg["gen_tokens"]
            agg["hit_rate"] = round(agg["hits"] / max(agg["acquires"], 1), 4)
            agg["miss_per_tok"] = round(agg["miss_loads"] / n, 3)
            agg["spec_per_tok"] = round(agg["spec_loads"] / n, 3)
            agg["h2d_mb_per_tok"] = round((agg["miss_loads"] + agg["spec_loads"]) * eb / n / 1e6, 1)
            # copies the decisions require (a speculative copy is only needed
            # once it is consumed): misses + staging hits
            agg["h2d_floor_ms"] = round((agg["miss_loads"] + agg["staging_hits"]) * eb / n /
                                        (h2d * 1e9) * 1e3, 3)
            grid.append(agg)
            print(json.dumps(agg), flush=True)
    gr = []
    for la in (1, 2, 10):
        for m in (1, 2, 4):
            vals = [guess_recall(tr, la, m) for tr in traces]
            gr.append({"lookahead": la, "m": m, "guess_recall": round(float(np.mean(vals)), 4),
                       "per_prompt": [round(v, 4) for v in vals]})
            print(json.dumps(gr[-1]), flush=True)
    res = {"config": a.config, "expert_bytes": eb, "h2d_peak_gbs": round(h2d, 2),
           "prompts": a.prompts, "gen_tokens_per_prompt": a.tokens,
           "live_vs_replay": live_check, "grid": grid, "guess_recall": gr}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out + ".json", "w") as fh:
        json.dump(res, fh, indent=1)
    lines = [f"# Trace-driven sweep ({a.config}: {ab}-bit attention, {xb}-bit experts), "
             f"{a.prompts} prompts x {a.tokens} greedy tokens, reference init weights",
             "", f"Device traces recorded on B200; replayed with the reference `replay` "
             f"(engine.py:263-313) and with the engine's device store code. "
             f"Live device log vs reference replay of its own trace (prompt 0, k={k0}, m={m0}): "
             f"**{'equal' if live_check and live_check['equal'] else 'DIFFERENT'}** "
             f"({live_check['events'] if live_check else 0} events). H2D peak {h2d:.2f} GB/s (measured in this run).",
             "", "| k | m | hit rate | misses / tok | spec loads / tok | H2D MB / tok | H2D floor ms / tok | device store == reference |",
             "|---|---|---|---|---|---|---|---|"]
    for g in grid:
        lines.append(f"| {g['k']} | {g['m']} | {g['hit_rate']:.4f} | {g['miss_per_tok']:.2f} | "
                     f"{g['spec_per_tok']:.2f} | {g['h2d_mb_per_tok']:.0f} | {g['h2d_floor_ms']:.2f} | "
                     f"{'yes' if g['device_store_equal'] else 'NO'} |")
    lines += ["", "Speculative guess recall (`guess_recall`, engine.py:316-338), mean over prompts:", "",
              "| lookahead | m=1 | m=2 | m=4 |", "|---|---|---|---|"]
    for la in (1, 2, 10):
        row = {x["m"]: x["guess_recall"] for x in gr if x["lookahead"] == la}
        lines.append(f"| {la} | {row[1]:.4f} | {row[2]:.4f} | {row[4]:.4f} |")
    with open(a.out + ".md", "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
