"""Markdown summary of every kernel in an ncu --set full report: duration, DRAM traffic, shared-memory
wavefronts (and their share of the pipe), FP64 pipe, issue activity, occupancy and the top stall
reasons (per issued instruction).  Used for profiles/r02_*.md.

    python tools/ncu_kernels_md.py report.ncu-rep
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ix = {k: i for i, k in enumerate(h)}


def g(r, k):
    return r[ix[k]] if k in ix else ""


stalls = [k for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
print("| kernel | ms | DRAM read MB | DRAM write MB | smem wavefronts | smem pipe % (elapsed) | smem ld bank-conflict wavefronts | FP64 pipe % (active) | issue % (active) | warps/SM | registers | top stalls (warps per issue) |")
print("|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---|")
for r in rows[2:]:
    st = sorted(((float(g(r, k) or 0), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")])
                 for k in stalls), reverse=True)[:4]
    print(f"| `{g(r, 'Kernel Name')}` | {float(g(r, 'gpu__time_duration.sum')):.3f} | {g(r, 'dram__bytes_read.sum')} | "
          f"{g(r, 'dram__bytes_write.sum')} | {g(r, 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum')} | "
          f"{float(g(r, 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed') or 0):.1f} | "
          f"{g(r, 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum')} | "
          f"{float(g(r, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active') or 0):.1f} | "
          f"{float(g(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active') or 0):.1f} | "
          f"{float(g(r, 'sm__warps_active.avg.per_cycle_active') or 0):.1f} | {g(r, 'launch__registers_per_thread')} | "
          + ", ".join(f"{n} {v:.2f}" for v, n in st) + " |")
