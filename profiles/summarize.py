"""Summarise ncu captures into profiles/ (run here, on the CPU box).

  python profiles/summarize.py gpurun_out/prof_x.ncu-rep ... > profiles/rNN_x.txt
  python profiles/summarize.py --launches gpurun_out/launches.csv > profiles/rNN_launches.txt
"""
import collections
import csv
import re
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed",
    "derived__l1tex__lsu_writeback_bytes_mem_lgds.sum.per_second",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"== {path}: {re.sub(r'[(].*', '', name)}")
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                print(f"  {m:78s} {r[i]:>18s} {units[i]}")


def launches(path):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.OrderedDict()
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[1:]:
        if "swg::" not in r[ki]:  # bench scaffolding: the spin before a step, L2 flush fills
            continue
        name = re.sub(r"[(].*", "", r[ki]).replace("swg::<unnamed>::", "")
        us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        n, t = tot.get(name, (0, 0.0))
        tot[name] = (n + 1, t + us)
    all_us = sum(t for _, t in tot.values())
    print("# libswg kernels only (the bench's spin kernel and L2-flush fills excluded)")
    print(f"{'kernel':70s} {'launches':>8s} {'total us':>12s} {'share':>7s}")
    for k, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:70s} {n:8d} {t:12.1f} {100 * t / all_us:6.1f}%")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        for p in sys.argv[1:]:
            rep(p)
