"""Time the c5 operator-term kernel (DMMA complex GEMM + fused Taylor epilogue).

    python tools/bench_zgemm.py [columns ...]      (default 64 128)
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_06200_b200 import _native  # noqa: E402

lib = _native.load()
out = {}
for c in ([int(a) for a in sys.argv[1:]] or [64, 128]):
    ms = C.c_double()
    _native.check(lib.lg_bench_zgemm(4096, c, 20, C.byref(ms)))
    out[f"lg_zgemm_4096x{c}_ms"] = ms.value
    out[f"lg_zgemm_4096x{c}_tflops"] = 8 * 4096 * 4096 * c / (ms.value / 1e3) / 1e12
print(json.dumps(out))
