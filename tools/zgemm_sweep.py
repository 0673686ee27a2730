"""Sweep the c5 operator-term kernel over split-k and tile choices (LG_SPLITK / LG_ZGEMM_N32 are read
per launch), d = 4096, C = 64 / 128: ms per term and algorithmic / executed (3M) TFLOP/s."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_06200_b200 import _native  # noqa: E402

lib = _native.load()
rows = []
for n32 in ("64", "1", "0"):
    for ks in ("", "1", "2", "4", "8", "16"):
        os.environ["LG_ZGEMM_N32"] = n32
        if ks:
            os.environ["LG_SPLITK"] = ks
        else:
            os.environ.pop("LG_SPLITK", None)
        for c in (64, 128):
            ms = C.c_double()
            _native.check(lib.lg_bench_zgemm(4096, c, 20, C.byref(ms)))
            alg = 8 * 4096 * 4096 * c / (ms.value / 1e3) / 1e12
            rows.append({"n32_from": n32, "splitk": ks or "auto", "C": c, "ms": round(ms.value, 4),
                         "alg_tflops": round(alg, 2), "exec_tflops": round(0.75 * alg, 2)})
            print(json.dumps(rows[-1]), flush=True)
