"""Summarise ncu captures into text for profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py gpurun_out/launches.csv gpurun_out/prof_*.ncu-rep > profiles/rNN_ncu.txt
"""
import collections
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":    # launch lists may carry DRAM metrics too
            continue
        name = r[ki].split("(")[0].replace("void ", "")[:64]
        v = float(r[vi].replace(",", ""))
        v *= {"usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"== launch list {path}: {sum(v[0] for v in agg.values())} launches, {tot/1e6:.3f} ms "
          "(ncu, serialised, cold cache: compare shares)")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {k:64s} n={n:5d} total={t/1e6:8.3f} ms share={t/tot*100:5.1f}% avg={t/n/1e3:9.1f} us")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return
    h = rows[0]
    print(f"== {path}")
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"  kernel: {name[:100]}")
        for k in KEYS:
            if k in h:
                print(f"    {k:70s} {r[h.index(k)]}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        if p.endswith(".csv"):
            launches(p)
        else:
            report(p)
