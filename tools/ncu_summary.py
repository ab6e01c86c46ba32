"""Summarise an ncu launch list (gpu__time_duration.sum CSV) per kernel, and
optionally the key metrics of a --set full report.

  python tools/ncu_summary.py launches.csv [--full rep.ncu-rep]
"""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    out = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        out.append((r[ki].split("(")[0], float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)))
    return out


def per_kernel(seq):
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, ms in seq:
        agg[n][0] += 1
        agg[n][1] += ms
    tot = sum(v[1] for v in agg.values())
    lines = [f"{'kernel':70s} {'launches':>8s} {'total ms':>9s} {'avg ms':>8s} {'share':>6s}"]
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{n[:70]:70s} {c:8d} {t:9.3f} {t / c:8.4f} {100 * t / tot:5.1f}%")
    return "\n".join(lines)


KEYS = ("Duration", "Elapsed Cycles", "SM Active Cycles", "Compute (SM) Throughput",
        "Memory Throughput", "DRAM Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Achieved Active Warps Per SM", "Executed Instructions",
        "Warp Cycles Per Issued Instruction", "L2 Hit Rate", "Grid Size", "Block Size")


def full(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h = rows[0]
    out = []
    for row in rows[1:]:
        d = dict(zip(h, row))
        if d.get("Metric Name") in KEYS:
            out.append(f"{d['Kernel Name'][:40]:40s} {d['Metric Name']:40s} {d['Metric Value']:>16s} "
                       f"{d['Metric Unit']}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,"
                          "sm__pipe_tmem_cycles_active.avg.pct_of_peak_sustained_active,"
                          "sm__inst_executed_pipe_uma.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    return "\n".join(out) + "\n\nraw:\n" + raw


if __name__ == "__main__":
    print(per_kernel(launches(sys.argv[1])))
    if "--full" in sys.argv:
        print()
        print(full(sys.argv[sys.argv.index("--full") + 1]))
