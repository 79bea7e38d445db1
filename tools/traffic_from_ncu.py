"""Per-launch DRAM traffic from an ncu launch list of ONE timed bench step.

    ZO_NVTX=1 ncu --nvtx --nvtx-include zo_step/ --clock-control none --csv \
        --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --log-file gpurun_out/step_traffic.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e
    python tools/traffic_from_ncu.py gpurun_out/step_traffic.csv > profiles/ncu_traffic.json

bench.py copies `perturb_bytes_per_launch` and `gemm_bytes_per_step` into
its roofline objects' `traffic` fields.
"""
import collections
import csv
import json
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ii, ki, mi, vi, ui = (h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                          h.index("Metric Unit"))
    launches = collections.defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        launches[r[ii]][r[mi]] = v
        names[r[ii]] = r[ki].split("(")[0].replace("void ", "")
    per_kernel = collections.defaultdict(lambda: {"n": 0, "bytes": 0.0, "s": 0.0})
    for lid, m in launches.items():
        k = per_kernel[names[lid]]
        k["n"] += 1
        k["bytes"] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        k["s"] += m.get("gpu__time_duration.sum", 0)
    pert = [v for k, v in per_kernel.items() if "perturb_update_kernel" in k]
    gemm = [v for k, v in per_kernel.items() if "gemm_tcgen05" in k]
    out = {
        "source": path,
        "launches": len(launches),
        "perturb_bytes_per_launch": (sum(v["bytes"] for v in pert) / max(1, sum(v["n"] for v in pert))) if pert else None,
        # the fill plan splits the pass into one launch per block: the step's total is the comparable figure
        "perturb_bytes_per_step": sum(v["bytes"] for v in pert) if pert else None,
        "perturb_launches_per_step": sum(v["n"] for v in pert),
        "gemm_bytes_per_step": sum(v["bytes"] for v in gemm) if gemm else None,
        "gemm_launches_per_step": sum(v["n"] for v in gemm),
        "kernels": {k: {"n": v["n"], "dram_bytes": v["bytes"], "ncu_time_ms": v["s"] * 1e3}
                    for k, v in sorted(per_kernel.items(), key=lambda kv: -kv[1]["s"])},
    }
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])
