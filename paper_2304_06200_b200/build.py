"""Build the sm_100a shared library in-tree (nvcc; no torch JIT, no CPU fallback).

    python -m paper_2304_06200_b200.build

Output: paper_2304_06200_b200/_lib/libleangrape_b200.so (git-ignored; it
travels to the GPU box with the repo snapshot).
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib" + ("_debug" if os.environ.get("LG_DEBUG") else ""))
LIB = os.path.join(OUT, "libleangrape_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-ffp-contract=off", "-Xptxas", "-v"]

# per-unit flags: the step-preparation/planner and host units must round like
# numpy / CPython (no FMA contraction); the sweep engine may contract.
UNITS = {
    "lg_prep.cu": ["-fmad=false"],
    "lg_api.cu": ["-fmad=false"],
    "lg_host.cu": ["-fmad=false"],
    "lg_configure.cu": ["-fmad=false"],
    "lg_dense_host.cu": ["-fmad=false"],
    "lg_engine.cu": [],
    "lg_sweep_cta.cu": ["-DLG_DEBUG"] if os.environ.get("LG_DEBUG") else [],
    "lg_dense.cu": [],
    "lg_sweep_ws.cu": [],
    "lg_sweep_cl.cu": [],
    **{f"lg_sweep_cl_w{w}.cu": [] for w in range(3, 10)},
    "lg_diag.cu": [],
}


def _sources():
    return [os.path.join(SRC, f) for f in os.listdir(SRC) if f.endswith((".cu", ".cuh", ".h"))] + [
        os.path.join(os.path.dirname(HERE), "include", "leangrape_b200.h")
    ]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in _sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(OUT, exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor

    def newest_dep(path, seen=None):
        """mtime of `path` and of every local header it includes (recursively)."""
        seen = set() if seen is None else seen
        if path in seen or not os.path.exists(path):
            return 0.0
        seen.add(path)
        t = os.path.getmtime(path)
        with open(path) as fh:
            for line in fh:
                line = line.strip()
                if line.startswith("#include \""):
                    inc = line.split('"')[1]
                    for base in (os.path.dirname(path), os.path.join(os.path.dirname(HERE), "include")):
                        cand = os.path.normpath(os.path.join(base, inc))
                        if os.path.exists(cand):
                            t = max(t, newest_dep(cand, seen))
                            break
        return t

    def compile_unit(item):
        unit, flags = item
        obj = os.path.join(OUT, unit.replace(".cu", ".o"))
        src = os.path.join(SRC, unit)
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) >= newest_dep(src)):
            return unit, obj, None
        cmd = [NVCC, *COMMON, *flags, "-c", os.path.join(SRC, unit), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        with open(os.path.join(OUT, unit + ".ptxas.log"), "w") as fh:
            # resource usage per kernel (registers, spills, stack); compile times dropped so the
            # committed logs only change when the code does
            fh.write("".join(l for l in r.stderr.splitlines(True) if "Compile time" not in l))
        return unit, obj, r

    objs = []
    with ThreadPoolExecutor(max_workers=len(UNITS)) as ex:
        for unit, obj, r in ex.map(compile_unit, UNITS.items()):
            if r is None:  # up to date
                objs.append(obj)
                continue
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed for {unit}")
            if verbose:
                sys.stderr.write(r.stderr)
            objs.append(obj)
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-lcublas", "-lcusolver"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
