"""C5: cache-size x prefetch-depth sweep on the Mixtral-shape model (BASELINE
configs[4]): hit rate, H2D GB/s and tokens/s per (k, m), one bench.py run per
point (fresh engine).  Writes a markdown table.

    python tools/sweep.py [--config c3] [--ks 0,1,2,4,8] [--ms 0,1,2] [--out FILE]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--ks", default="0,1,2,4,8")
    ap.add_argument("--ms", default="0,1,2")
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    for k in [int(x) for x in a.ks.split(",")]:
        for m in [int(x) for x in a.ms.split(",")]:
            cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", a.config, "--k", str(k),
                   "--m", str(m), "--steps", str(a.steps), "--warmup", "4", "--no-cpu-baseline",
                   "--no-e2e"]
            p = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=1200)
            try:
                d = json.loads(p.stdout.strip().splitlines()[-1])
            except (IndexError, json.JSONDecodeError):
                print(f"k={k} m={m}: failed\n{p.stderr[-2000:]}", file=sys.stderr)
                continue
            r = {"k": k, "m": m, "tok_s": d["value"], "hit_rate": d["hit_rate"],
                 "h2d_gbs": d["h2d_gbs"], "miss_per_tok": d["miss_loads_per_token"],
                 "spec_per_tok": d["spec_loads_per_token"],
                 "roofline_frac": d["roofline_e2e"]["frac"]}
            rows.append(r)
            print(json.dumps(r), flush=True)
    lines = [f"# C5 sweep ({a.config.upper()} base: Mixtral shape, {a.steps} greedy tokens per point, "
             "fresh engine per point, 1x B200)", "",
             "| k | m | tokens/s | hit rate | MISS_LOAD/token | SPECULATIVE_LOAD/token | H2D GB/s | "
             "roofline frac |", "|---|---|---|---|---|---|---|---|"]
    for r in rows:
        hr = "n/a" if r["hit_rate"] is None else f"{r['hit_rate']:.3f}"
        h2d = "n/a" if r["h2d_gbs"] is None else f"{r['h2d_gbs']:.1f}"
        lines.append(f"| {r['k']} | {r['m']} | {r['tok_s']:.2f} | {hr} | {r['miss_per_tok']:.2f} | "
                     f"{r['spec_per_tok']:.2f} | {h2d} | {r['roofline_frac']:.3f} |")
    txt = "\n".join(lines) + "\n"
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(txt)
    print(txt)


if __name__ == "__main__":
    main()
