"""Summarise the ws-cluster backward's per-step clock64 traces (LG_TRACE) for one config.

    python tools/ws_trace.py [c2] [n_steps|full]

Slot 7 = psi-recovery rank, slots 6, 5 = costate ranks 0, 1, slots 0.. = derivative workers.
Prints medians (cycles) of each phase; comparisons are within one CTA (one SM clock).
"""
import os
import subprocess
import sys

import numpy as np

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = sys.argv[2] if len(sys.argv) > 2 else "full"
path = "/tmp/lg_trace.bin"
env = dict(os.environ, LG_TRACE=path)
here = os.path.dirname(os.path.abspath(__file__))
subprocess.run([sys.executable, os.path.join(here, "run_eval.py"), name, n, "1"], env=env, check=True)
t = np.fromfile(path, np.int64)
N = 2000 if n == "full" else int(n)
t = t.reshape(-1, 8, N, 4)[0].astype(np.float64)
med = lambda x: float(np.median(x))
P = t[7]
print(f"P  : step {med(np.diff(P[:, 0])):.0f}  chain {med(P[:, 1] - P[:, 0]):.0f}  slot waits {med(P[:, 2] - P[:, 1]):.0f}")
for s, slot in enumerate((6, 5)):
    L = t[slot]
    if not L[:, 0].any():
        continue
    print(f"L{s} : step {med(np.diff(L[:-1, 0])):.0f}  lempty wait {med(L[:-1, 1] - L[:-1, 0]):.0f}  "
          f"push+load+chain {med(L[:-1, 2] - L[:-1, 1]):.0f}  source wait+add {med(L[:-1, 3] - L[:-1, 2]):.0f}")
for w in range(6):
    X = t[w]
    rows = X[X[:, 0] != 0]
    if not len(rows):
        continue
    print(f"X{w} : period {med(np.diff(rows[:, 0])):.0f}  psi wait {med(rows[:, 1] - rows[:, 0]):.0f}  "
          f"chain {med(rows[:, 2] - rows[:, 1]):.0f}  hand-off {med(rows[:, 3] - rows[:, 2]):.0f}")
