"""One-kernel summary of an ncu --set full report (key throughput / memory / occupancy counters,
DRAM traffic per launch, stall breakdown).  Used to write profiles/*.md.

    python tools/ncu_summary.py report.ncu-rep
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate", "Registers Per Thread", "Block Size", "Grid Size",
        "Cluster Size", "Dynamic Shared Memory Per Block", "Achieved Occupancy", "Theoretical Occupancy",
        "Max Active Clusters", "Waves Per SM", "Warp Cycles Per Issued Instruction"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    res = {"kernel": rows[1][ix["Kernel Name"]]}
    for r in rows[1:]:
        name = r[ix["Metric Name"]]
        if name in KEYS and name not in res:
            res[name] = f"{r[ix['Metric Value']]} {r[ix['Metric Unit']]}".strip()
    return res


def raw_metric(rep, names):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    res = {}
    for n in names:
        if n in h:
            i = h.index(n)
            res[n] = (v[i], u[i])
    return res


if __name__ == "__main__":
    rep = sys.argv[1]
    d = details(rep)
    raw = raw_metric(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
                           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
                           "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "gpu__time_duration.sum"])
    print(json.dumps({"details": d, "raw": raw}, indent=1))
