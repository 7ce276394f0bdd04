"""Summarise tools/ncu_configs.sh CSVs: per kernel, launches, mean duration,
DRAM bytes per launch, fp64-pipe and l1tex utilisation (duration-weighted).
With --write, also store the whole evaluation's totals (the CSV holds exactly
one evaluation) as profiles/kernel_metrics.json["workload:<cfg>"], which
bench.py attaches to the c1-c4 lines (DRAM GB/s and fp64 pipe
per config).  Usage: python tools/ncu_config_summary.py [--write] gpurun_out/ncu_c*.csv"""
import collections
import csv
import json
import os
import re
import sys

write = "--write" in sys.argv
paths = [a for a in sys.argv[1:] if a != "--write"]
store = {}
for path in paths:
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    iI, iN, iM, iV, iU = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    launches = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) <= iV:
            continue
        m = re.search(r"([A-Za-z_][A-Za-z0-9_]*)(<[^()]*>)?\(", r[iN])
        name = m.group(1) if m else r[iN][:30]
        d = launches.setdefault(r[iI], {"name": name})
        v = float(r[iV].replace(",", "")) if r[iV] not in ("", "n/a") else 0.0
        unit = r[iU]
        if r[iM] == "gpu__time_duration.sum":
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        if r[iM].startswith("dram__bytes"):
            v *= {"byte": 1, "B": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}.get(unit, 1.0)
        d[r[iM]] = v
    agg = collections.OrderedDict()
    for d in launches.values():
        a = agg.setdefault(d["name"], [0, 0.0, 0.0, 0.0, 0.0])
        t = d.get("gpu__time_duration.sum", 0.0)
        a[0] += 1
        a[1] += t
        a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        a[3] += t * d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0)
        a[4] += t * d.get("l1tex__throughput.avg.pct_of_peak_sustained_active", 0)
    print(f"== {path}")
    print(f"{'kernel':24s} {'launches':>8s} {'mean_us':>9s} {'dram_MB/launch':>15s} {'fp64%':>6s} {'l1tex%':>7s}")
    for k, a in agg.items():
        n, t = a[0], a[1]
        print(f"{k:24s} {n:8d} {t / n:9.2f} {a[2] / n / 1e6:15.3f} {a[3] / max(t, 1e-9):6.1f} {a[4] / max(t, 1e-9):7.1f}")
    T = sum(a[1] for a in agg.values())
    tot = {"eval_kernel_us": T, "launches": sum(a[0] for a in agg.values()),
           "dram_bytes_per_eval": sum(a[2] for a in agg.values()),
           "fp64_pipe_pct": sum(a[3] for a in agg.values()) / max(T, 1e-9),
           "l1tex_pct": sum(a[4] for a in agg.values()) / max(T, 1e-9)}
    print(f"{'evaluation':24s} {tot['launches']:8d} {T:9.2f} {tot['dram_bytes_per_eval'] / 1e6:15.3f} "
          f"{tot['fp64_pipe_pct']:6.1f} {tot['l1tex_pct']:7.1f}")
    m = re.search(r"ncu_(c[1-5])", path)
    if m:
        tot["source"] = (f"ncu --metrics (gpu__time_duration, dram__bytes_read/write, sm__pipe_fp64_cycles_active, "
                         f"l1tex__throughput) of every kernel of one {m.group(1)} evaluation after warm-up "
                         f"(tools/ncu_configs.sh), duration-weighted; profiles/r02/config_kernels_ncu.txt")
        store["workload:" + m.group(1)] = tot
if write and store:
    kp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "kernel_metrics.json")
    km = json.load(open(kp)) if os.path.exists(kp) else {}
    km.update(store)
    json.dump(km, open(kp, "w"), indent=1)
    print("wrote", ", ".join(store), "to", kp)
