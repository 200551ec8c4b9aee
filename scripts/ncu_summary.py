"""Summarise ncu output for profiles/: launch-list shares and key metrics of a --set full capture."""
import csv
import subprocess
import sys
from collections import defaultdict

SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[i], rows[i + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in data:
        us = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    out = [f"# launch list: {path} (ncu --metrics gpu__time_duration.sum --clock-control none; cold, serialised)",
           f"{'launches':>8} {'total_us':>14} {'share':>7}  kernel"]
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{c:8d} {v:14.1f} {100 * v / tot:6.2f}%  {k}")
    return "\n".join(out)


KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit", "launch__shared_mem_per_block", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__t_bytes.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warp_latency_issue_stalled"]


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h, u = r[0], r[1]
    out = [f"# ncu --set full: {path}"]
    for row in r[2:]:
        kn = row[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        out.append(f"## {kn.split('(')[0]}")
        for i, name in enumerate(h):
            if any(name.startswith(k) for k in KEYS) and not name.endswith("_bucket"):
                out.append(f"{name} = {row[i]} {u[i]}")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launches(path) if kind == "launches" else full(path))
