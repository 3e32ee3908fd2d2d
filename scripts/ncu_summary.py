"""Summarise an ncu report: key SOL / scheduler / memory metrics (+ optional JSON out)."""
import csv
import io
import json
import subprocess
import sys

WANT = ['Duration', 'Elapsed Cycles', 'SM Frequency', 'Compute (SM) Throughput', 'Memory Throughput',
        'L1/TEX Cache Throughput', 'L2 Cache Throughput', 'DRAM Throughput', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'Executed Ipc Active', 'Issue Slots Busy',
        'L1/TEX Hit Rate', 'L2 Hit Rate', 'Mem Busy', 'Max Bandwidth', 'No Eligible',
        'Active Warps Per Scheduler', 'Eligible Warps Per Scheduler', 'Warp Cycles Per Issued Instruction',
        'Executed Instructions', 'Dynamic Shared Memory Per Block', 'Block Limit Registers',
        'Block Limit Shared Mem', 'Grid Size', 'Block Size']


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(io.StringIO(out))
    h = next(r)
    res = {}
    for row in r:
        name = row[h.index("Metric Name")]
        if name in WANT:
            res[name] = (row[h.index("Metric Value")], row[h.index("Metric Unit")])
        if "Kernel Name" in h:
            res["kernel"] = (row[h.index("Kernel Name")][:90], "")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) >= 3:
        hdr, units, vals = rr[0], rr[1], rr[2]
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed.sum",
                    "smsp__inst_executed.sum", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
                    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                    "sm__inst_executed_pipe_tex.avg.pct_of_peak_sustained_active",
                    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                    "l1tex__t_requests_pipe_tex_mem_texture.sum",
                    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active"):
            if key in hdr:
                i = hdr.index(key)
                res[key] = (vals[i], units[i])
    return res


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        if rep.endswith(".json"):
            continue
        s = summary(rep)
        print("==", rep)
        for k, (v, u) in s.items():
            print(f"  {k:60s} {v:>18s} {u}")
