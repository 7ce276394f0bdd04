"""Per-source-line warp-stall sample shares of an ncu report (needs -lineinfo)."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res = []
for i, r in enumerate(rows):
    if r and r[0] == "Line No" and "Warp Stall Sampling (All Samples)" in r:
        hdr = r
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        fname = rows[i - 2][1] if i >= 2 else "?"
        for rr in rows[i + 1:]:
            if not rr or rr[0] in ("File Path", "File Name"):
                break
            try:
                res.append((int(rr[iS]), fname.split("/")[-1], int(rr[0]), rr[1].strip()[:100]))
            except (ValueError, IndexError):
                pass
tot = sum(x[0] for x in res) or 1
res.sort(reverse=True)
for s, f, l, src in res[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{100 * s / tot:5.1f}%  {f}:{l}: {src}")
