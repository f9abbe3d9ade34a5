"""Compact text summary of ncu reports (ncu -i ... --page raw --csv), one
block per captured launch: duration, DRAM bytes, FP64 / DMMA pipe use,
occupancy, issue activity, top warp-stall reasons, shared-memory bank
conflicts.

    python tools/ncu_summary.py a.ncu-rep [b.ncu-rep ...] > profiles/x.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("duration_us", "gpu__time_duration.sum", "time"),
    ("dram_read_MB", "dram__bytes_read.sum", "bytes"),
    ("dram_write_MB", "dram__bytes_write.sum", "bytes"),
    ("dram_pct_peak", "dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("fp64_pipe_pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1),
    ("dmma_pipe_pct", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", 1),
    ("issue_active_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
    ("achieved_occupancy_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct", 1),
    ("smem_bank_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    ("registers", "launch__registers_per_thread", 1),
    ("grid", "launch__grid_size", 1),
]


TIME = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
BYTES = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


for path in sys.argv[1:]:
    h, units, data = rows(path)
    unit = dict(zip(h, units))
    for v in data:
        d = dict(zip(h, v))
        name = d.get("Kernel Name", "?")
        print(f"== {path.split('/')[-1]}: {name[:110]}")
        parts = []
        for label, key, scale in KEYS:
            x = num(d.get(key, ""))
            if x is not None:
                if scale == "time":
                    x *= TIME.get(unit.get(key, ""), float("nan"))
                elif scale == "bytes":
                    x *= BYTES.get(unit.get(key, ""), float("nan"))
                else:
                    x *= scale
                parts.append(f"{label}={x:.4g}")
        print("   " + "  ".join(parts))
        stalls = []
        for k, x in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                y = num(x)
                if y is not None:
                    stalls.append((y, k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        stalls.sort(reverse=True)
        print("   stalls (warps per issue): " + ", ".join(f"{n} {y:.2f}" for y, n in stalls[:5]))
