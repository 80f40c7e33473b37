"""Summarise a GEMV per-CTA trace (MOE_CTA_TRACE_FILE of moe_bench_gemv).

    python tools/cta_trace.py gpurun_out/cta_trace.txt
Columns per CTA: id, smid, start (after griddepcontrol.wait), loop end, end (us).
"""
import sys
from collections import Counter

import numpy as np


def main(path):
    for blk in open(path).read().split("#")[1:]:
        ls = blk.strip().split("\n")
        a = np.array([[float(x) for x in l.split()] for l in ls[1:] if l.strip()])
        sm = a[:, 1].astype(int)
        c = Counter(sm)
        print(ls[0], f"| {len(c)} SMs")
        for n in sorted(set(c.values())):
            idx = [i for i in range(len(a)) if c[sm[i]] == n]
            s = a[idx]
            print(f"  {n}-CTA SMs: {len(idx)} CTAs  start {s[:, 2].mean():.2f}  loop_end "
                  f"{s[:, 3].mean():.2f}  end {s[:, 4].mean():.2f}  (max end {s[:, 4].max():.2f})")
        print("  end pct 10/50/90/max:", np.round(np.percentile(a[:, 4], [10, 50, 90, 100]), 2),
              " start max:", round(a[:, 2].max(), 2))
        late = np.argsort(-a[:, 4])[:5]
        for i in late:
            print("   late:", a[i])


if __name__ == "__main__":
    main(sys.argv[1])
