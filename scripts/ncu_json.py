"""Summary JSON (the fields bench.py reads for roofline.traffic / ncu_pipes) from an `ncu --page raw --csv` file.
Usage: python scripts/ncu_json.py RAW.csv KERNEL_DESC SOURCE_NOTE > profiles/ncu_<workload>_summary.json"""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
d = dict(zip(rows[0], rows[2]))
unit = dict(zip(rows[0], rows[1]))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "nsecond": 1e-6, "us": 1e-3,
         "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def f(k, scale=1.0):
    """Value of metric k in base units (bytes, ms), times scale."""
    try:
        return float(d[k].replace(",", "")) * SCALE.get(unit.get(k, ""), 1.0) * scale
    except (KeyError, ValueError):
        return None


rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
print(json.dumps({
    "round": 2,
    "kernel": sys.argv[2],
    "source": sys.argv[3],
    "duration_ms": f("gpu__time_duration.sum"),
    "dram_bytes_read": rd, "dram_bytes_write": wr,
    "dram_bytes_per_launch": (rd or 0) + (wr or 0),
    "executed_warp_instructions": f("smsp__inst_executed.sum"),
    "issue_slots_busy_pct": f("sm__inst_issued.avg.pct_of_peak_sustained_active"),
    "l1tex_throughput_pct": f("l1tex__throughput.avg.pct_of_peak_sustained_active"),
    "l2_hit_rate_pct": f("lts__t_sector_hit_rate.pct"),
    "achieved_occupancy_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": f("launch__registers_per_thread"),
    "fma_pipe_active_pct": f("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
}, indent=1))
