"""Development tool: key metrics of every kernel in an `ncu --set full` report (.ncu-rep), as JSON lines.
usage: ncu_summary.py report.ncu-rep"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.per_cycle_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_active.avg",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
for r in rows[2:]:
    d = {"kernel": r[h.index("Kernel Name")]}
    for k in KEYS:
        if k in h:
            v = r[h.index(k)].replace(",", "")
            try:
                v = float(v)
            except ValueError:
                pass
            d[k] = v
            u = units[h.index(k)]
            if u == "Kbyte":
                d[k] = v * 1e3
            elif u == "Mbyte":
                d[k] = v * 1e6
            elif u == "Gbyte":
                d[k] = v * 1e9
            elif u == "byte":
                d[k] = v
            elif u in ("ms", "msecond"):
                d[k] = v * 1e-3
            elif u in ("us", "usecond"):
                d[k] = v * 1e-6
            elif u in ("ns", "nsecond"):
                d[k] = v * 1e-9
    print(json.dumps(d))
