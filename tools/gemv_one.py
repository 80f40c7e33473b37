"""Run one GEMV microbenchmark case (for ncu): python tools/gemv_one.py BITS K N NJOBS [ITERS]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_17238_b200 import _lib  # noqa: E402

bits, K, N, nj = (int(a) for a in sys.argv[1:5])
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 10
us, gbs = C.c_double(), C.c_double()
det = (C.c_double * 4)()
_lib.check(_lib.lib().moe_bench_gemv(bits, K, N, nj, iters, 1, C.byref(us), C.byref(gbs), det))
print(f"bits={bits} K={K} N={N} jobs={nj}: {us.value:.2f} us {gbs.value:.1f} GB/s")
