"""Per-source-line shared-memory wavefronts (actual vs ideal) of an ncu report."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = {}
cur = None
hdr = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or len(r) != len(hdr):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    def g(name):
        try:
            return float(r[hdr.index(name)] or 0)
        except (ValueError, IndexError):
            return 0.0
    a = agg.setdefault(ln, [0.0, 0.0, 0.0, r[1].strip()[:90]])
    a[0] += g("L1 Wavefronts Shared")
    a[1] += g("L1 Wavefronts Shared Ideal")
    a[2] += g("L2 Theoretical Sectors Global")
tot = sum(v[0] for v in agg.values()) or 1
print(f"total shared wavefronts {tot:.3e}")
for ln, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100 * v[0] / tot:5.1f}%  wf={v[0]:.3e} ideal={v[1]:.3e} l2sec={v[2]:.3e}  {ln}: {v[3]}")
