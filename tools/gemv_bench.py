"""GEMV microbenchmark sweep on the GPU (profiling aid).

    python tools/gemv_bench.py   -> one line per (shape, bits)
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_17238_b200 import _lib  # noqa: E402

CASES = [  # name, bits, K, N, njobs
    ("expert_up_3b (2 experts x W1,W3)", 3, 4096, 14336, 4),
    ("expert_down_3b (2 experts)", 3, 14336, 4096, 2),
    ("expert_up_2b", 2, 4096, 14336, 4),
    ("expert_down_2b", 2, 14336, 4096, 2),
    ("attn_qkv_4b", 4, 4096, 4096, 3),
    ("attn_wo_4b", 4, 4096, 4096, 1),
    ("lm_head_f16", 16, 4096, 32000, 1),
]


def main():
    L = _lib.lib()
    out = []
    for name, bits, K, N, nj in CASES:
        for pdl in (0, 1):
            us, gbs = C.c_double(), C.c_double()
            det = (C.c_double * 4)()
            _lib.check(L.moe_bench_gemv(bits, K, N, nj, 50, pdl, C.byref(us), C.byref(gbs), det))
            out.append({"case": name, "pdl": pdl, "us": round(us.value, 2),
                        "gbs": round(gbs.value, 1),
                        "traced": {"span_us": round(det[0], 2), "blk0_prologue_us": round(det[1], 2),
                                   "blk0_loop_end_us": round(det[2], 2),
                                   "blk0_reduce_end_us": round(det[3], 2)}})
            print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
