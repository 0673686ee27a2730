"""Summarise an ncu report's SASS source page: stall reasons, per-opcode shares, hottest instructions.

    python tools/ncu_sass_summary.py report.ncu-rep [n_hot]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n_hot = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
print(rows[0][:2])
h = rows[1]
data = [r for r in rows[2:] if len(r) >= len(h)]
ix = {k: i for i, k in enumerate(h)}


def num(r, k):
    try:
        return int(r[ix[k]] or 0)
    except ValueError:
        return 0


st = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = {k: sum(num(r, k) for r in data) for k in st}
T = sum(tot.values()) or 1
print("stalls %:", {k[6:]: round(100 * v / T, 1) for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v > 0.005 * T})
agg = collections.defaultdict(lambda: [0, 0])
S = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
I = sum(num(r, "Instructions Executed") for r in data) or 1
for r in data:
    toks = r[ix["Source"]].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    agg[op][0] += num(r, "Warp Stall Sampling (All Samples)")
    agg[op][1] += num(r, "Instructions Executed")
print("opcode  stall% inst%")
for op, a in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
    print(f"  {op:14s} {100 * a[0] / S:5.1f} {100 * a[1] / I:5.1f}")
data.sort(key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))
print("hottest:")
for r in data[:n_hot]:
    top = sorted(((num(r, k), k[6:]) for k in st), reverse=True)[:2]
    print(f"  {r[ix['Address']][-5:]} {r[ix['Source']][:56]:56s} {num(r, 'Warp Stall Sampling (All Samples)'):7d} {top}")
