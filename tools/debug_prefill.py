"""Debug aid: batched vs per-position prefill at Mixtral width, first
differing (position, layer) of the trace hidden states and logits."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2312_17238_b200 import CacheConfig, OffloadEngine, SpeculationConfig  # noqa: E402
from paper_2312_17238_b200 import synthetic_model  # noqa: E402


def run(bits, n, layers=2):
    cfg = dict(bench.MIXTRAL)
    cfg["n_layers"] = layers
    cobj = bench.cfg_obj(cfg)
    prompt = [int(t) for t in np.random.default_rng(5).integers(0, cobj.vocab_size, n)]
    outs = []
    for batch in ("1", "0"):
        os.environ["MOE_PREFILL_BATCH"] = batch
        eng = OffloadEngine(synthetic_model(cobj, 0), CacheConfig(k=2, b=4),
                            SpeculationConfig(enabled=False), record_hidden=True,
                            synth=(0, 4, bits), expert_bytes=bench.expert_bytes(bench.MIXTRAL, bits))
        lg = np.asarray(eng.prefill(prompt)).copy()
        tr = eng.trace()
        hid = {(r.token_pos, r.layer): r.hidden for r in tr.records}
        ex = {(r.token_pos, r.layer): r.experts for r in tr.records}
        outs.append((lg, hid, ex))
        eng.close()
    (la, ha, ea), (lb, hb, eb) = outs
    bad = [(p, l) for (p, l) in sorted(ha) if not np.array_equal(ha[(p, l)], hb[(p, l)])]
    badx = [(p, l) for (p, l) in sorted(ea) if ea[(p, l)] != eb[(p, l)]]
    badl = [p for p in range(n) if not np.array_equal(la[p], lb[p])]
    print(f"bits={bits} n={n}: hidden diffs {len(bad)} first {bad[:6]}; expert diffs {badx[:6]}; "
          f"logit rows differing {badl[:10]} (of {len(badl)})", flush=True)
    if bad:
        p, l = bad[0]
        d = np.abs(ha[(p, l)] - hb[(p, l)])
        print("  max |dh|", d.max(), "at", int(d.argmax()), flush=True)


if __name__ == "__main__":
    for bits, n in ((2, 70), (2, 9), (3, 70), (2, 64), (2, 65)):
        run(bits, n)
