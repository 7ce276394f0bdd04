"""Per-source-line stall reasons (samples) for selected lines of an ncu report."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
want = set(int(x) for x in sys.argv[2].split(",")) if len(sys.argv) > 2 and sys.argv[2] else None
hdr = None
agg = {}
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    if want and ln not in want:
        continue
    a = agg.setdefault(ln, {"src": r[1].strip()[:70]})
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                a[h] = a.get(h, 0.0) + float(r[i] or 0)
            except ValueError:
                pass
order = sorted(agg.items())
if len(sys.argv) > 3 and sys.argv[3] == "top":  # heaviest lines first
    order = sorted(agg.items(), key=lambda kv: -sum(v for k, v in kv[1].items() if k != "src"))[:40]
grand = sum(v for _, a in agg.items() for k, v in a.items() if k != "src") or 1
for ln, a in order:
    allv = sum(v for k, v in a.items() if k != "src")
    st = sorted(((v, k) for k, v in a.items() if k != "src" and v > 0), reverse=True)[:6]
    tot = sum(v for v, _ in st) or 1
    print(f"{ln}: [{100 * allv / grand:.1f}% of samples] {a['src']}")
    print("    " + ", ".join(f"{k[6:]}={100 * v / tot:.0f}%" for v, k in st))
