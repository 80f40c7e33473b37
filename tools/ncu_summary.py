"""Markdown summary of an ncu launch list (--metrics gpu__time_duration.sum --csv)
and an ncu --set full report of one decode layer (tools/gpu_profile.sh).

    python tools/ncu_summary.py gpurun_out/launches.csv gpurun_out/prof.ncu-rep > out.md
"""
import collections
import csv
import subprocess
import sys


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
    agg = collections.OrderedDict()
    for r in data:
        try:
            v = float(r[vi].replace(",", ""))
        except (ValueError, IndexError):
            continue
        name = r[ki].split("(")[0].replace("void <unnamed>::", "").replace("<unnamed>::", "")
        agg.setdefault((name, r[gi]), []).append(v)
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | grid | launches | avg µs | share of kernel time |", "|---|---|---|---|---|"]
    for (name, grid), v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| {name} | {grid} | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | "
                   f"{100 * sum(v) / tot:.1f}% |")
    return out


def full_table(rep, names, alg):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h = rows[0]

    def f(x):
        try:
            return float(x.replace(",", ""))
        except ValueError:
            return 0.0
    out = ["| kernel | grid | regs | ncu µs (cold, serialised) | DRAM MB (read+write) | "
           "algorithmic MB | DRAM GB/s | SM-active µs | issue-active % | IMMA pipe % of SM-active |",
           "|---|---|---|---|---|---|---|---|---|---|"]
    for nm, r, a in zip(names, rows[2:], alg):
        d = dict(zip(h, r))
        g = lambda k: f(d.get(k, "0"))  # noqa: E731
        t = g("gpu__time_duration.sum")
        dr = g("dram__bytes_read.sum") + g("dram__bytes_write.sum")
        act = g("TPC.TriageCompute.sm__cycles_active.avg")
        imma = g("TPC.TriageCompute.sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg")
        out.append(f"| {nm} | {d.get('launch__grid_size')} | {d.get('launch__registers_per_thread')} "
                   f"| {t:.2f} | {dr:.2f} | {a if a else '-'} | {dr / t * 1e3:.0f} | "
                   f"{(f'{act / 1965:.2f}' if act else 'n/a')} | "
                   f"{g('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
                   f"{(f'{100 * imma / act:.1f}' if act else '-')} |")
    return out


if __name__ == "__main__":
    names = ["Q‖K‖V + fused combine/LN1 (`k_mgemv<4,1,1>`)",
             "Wo + fused attention (`k_mgemv<4,1,1>`, X_ATTN)", "tail (`k_tail<512>`)",
             "W1‖W3 (`k_mgemv<3,1,1>`)", "W2 + SwiGLU prologue (`k_mgemv<3,1,1>`)"]
    alg = [26.36, 8.79, None, 95.54, 47.77]
    print("## Launch list\n")
    print("\n".join(launch_table(sys.argv[1])))
    if len(sys.argv) > 2:
        print("\n## Full capture, one decode layer\n")
        print("\n".join(full_table(sys.argv[2], names, alg)))
