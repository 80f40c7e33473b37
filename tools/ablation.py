"""§8(f)4: the paper's Table 2 ablation on real B200 timings (SPEC.md:306,
391-421): for 2-bit (C3 base) and 3-bit (C2 base) experts, Mixtral shape,
reference init weights, 4-bit attention, greedy decode of the §8(d) prompt:

  Full algorithm               LRU cache k + speculative pre-loading m = 2
  W/o expert pre-loading       LRU cache k, m = 0
  W/o LRU cache & pre-loading  k = 0, m = 0 (every use streams its expert)
  Naive offloading             load all E experts of a layer on every use:
                               closed form of SPEC.md:413 with this run's
                               measured constants -- all-hit compute per token
                               (k = E) + L * E * expert_bytes / measured H2D peak

Each measured row is one ``bench.py`` run (fresh engine, device-timed tokens/s,
CUDA events).  Writes a markdown table (and JSON next to it).

    python tools/ablation.py [--steps 16] [--out profiles/r2_ablation.md]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(config, k, m, steps):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", config, "--k", str(k),
           "--m", str(m), "--steps", str(steps), "--warmup", "4", "--no-cpu-baseline", "--no-e2e",
           "--no-prompts"]
    p = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=1500)
    try:
        return json.loads(p.stdout.strip().splitlines()[-1])
    except (IndexError, json.JSONDecodeError):
        print(f"{config} k={k} m={m}: failed\n{p.stderr[-3000:]}", file=sys.stderr)
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--configs", default="c3,c2")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "ablation.md"))
    a = ap.parse_args()
    sys.path.insert(0, ROOT)
    import bench
    L, E = bench.MIXTRAL["n_layers"], bench.MIXTRAL["n_experts"]
    out, lines = [], []
    for config in a.configs.split(","):
        ab, xb, k0, _ = bench.CONFIGS[config]
        kfull = 2 if xb == 2 else 4
        rows = [("Full algorithm", kfull, 2), ("W/o expert pre-loading", kfull, 0),
                ("W/o LRU cache & pre-loading", 0, 0), ("all experts resident (k = E)", E, 0)]
        res = {}
        for name, k, m in rows:
            d = run(config, k, m, a.steps)
            if d is None:
                continue
            res[name] = {"k": k, "m": m, "tok_s": d["value"], "ms_per_token": d["ms_per_step"],
                         "hit_rate": d["hit_rate"], "miss_per_tok": d["miss_loads_per_token"],
                         "spec_per_tok": d["spec_loads_per_token"],
                         "h2d_peak_gbs": d["roofline_e2e"]["h2d_peak_gbs"],
                         "expert_bytes": d["config"]["expert_bytes"]}
            print(json.dumps({config: {name: res[name]}}), flush=True)
        allhit = res.get("all experts resident (k = E)")
        if allhit:
            eb, peak = allhit["expert_bytes"], allhit["h2d_peak_gbs"]
            naive_ms = allhit["ms_per_token"] + L * E * eb / (peak * 1e9) * 1e3
            res["Naive offloading"] = {"k": 0, "m": 0, "tok_s": 1e3 / naive_ms,
                                       "ms_per_token": naive_ms, "modelled": True,
                                       "hit_rate": 0.0, "miss_per_tok": float(L * E),
                                       "spec_per_tok": 0.0}
        out.append({"config": config, "attn_bits": ab, "expert_bits": xb, "rows": res})
        lines += [f"## {xb}-bit experts, {ab}-bit attention ({config.upper()} base), Mixtral shape, 1x B200",
                  "", "| policy | k | m | tokens/s | ms / token | hit rate | MISS_LOAD / token | "
                  "SPECULATIVE_LOAD / token |", "|---|---|---|---|---|---|---|---|"]
        for name in ("Full algorithm", "W/o expert pre-loading", "W/o LRU cache & pre-loading",
                     "Naive offloading", "all experts resident (k = E)"):
            r = res.get(name)
            if not r:
                continue
            hr = "n/a" if r["hit_rate"] is None else f"{r['hit_rate']:.3f}"
            tag = " (closed form, measured constants)" if r.get("modelled") else ""
            lines.append(f"| {name}{tag} | {r['k']} | {r['m']} | {r['tok_s']:.2f} | "
                         f"{r['ms_per_token']:.2f} | {hr} | {r['miss_per_tok']:.2f} | "
                         f"{r['spec_per_tok']:.2f} |")
        lines.append("")
    txt = ("# Table 2 ablation on B200 (greedy decode, device-timed, fresh engine per row)\n\n"
           + "\n".join(lines))
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        fh.write(txt)
    with open(os.path.splitext(a.out)[0] + ".json", "w") as fh:
        json.dump(out, fh, indent=1)
    print(txt)


if __name__ == "__main__":
    main()
