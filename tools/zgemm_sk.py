"""Stream-K vs grid split-k for the c5 operator-term GEMM (LG_ZGEMM_SK read per launch), d = 4096:
ms per term and algorithmic / executed (3M) TFLOP/s per column count."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_06200_b200 import _native  # noqa: E402

lib = _native.load()
for sk in ("0", "1"):
    os.environ["LG_ZGEMM_SK"] = sk
    for c in (64, 128, 192, 256):
        ms = C.c_double()
        _native.check(lib.lg_bench_zgemm(4096, c, 20, C.byref(ms)))
        alg = 8 * 4096 * 4096 * c / (ms.value / 1e3) / 1e12
        print(json.dumps({"stream_k": sk, "C": c, "ms": round(ms.value, 4), "alg_tflops": round(alg, 2),
                          "exec_tflops": round(0.75 * alg, 2)}), flush=True)
