"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel."""
import collections
import csv
import re
import sys


def main(path, out=None, title=""):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    iN, iM, iV, iU = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) <= iV or r[iM] != "gpu__time_duration.sum":
            continue
        m = re.search(r"([A-Za-z_][A-Za-z0-9_]*)(<[^()]*>)?\(", r[iN])
        name = m.group(1) if m else r[iN][:40]
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[iU], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[iV].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    lines = [title, f"{'kernel':28s} {'launches':>8s} {'total_us':>14s} {'avg_us':>12s} {'share':>7s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k:28s} {n:8d} {t:14.1f} {t / n:12.1f} {100 * t / tot:6.2f}%")
    text = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(text)
    print(text)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None, sys.argv[3] if len(sys.argv) > 3 else "")
