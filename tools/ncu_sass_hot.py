"""Hottest SASS instructions of an ncu report (stall samples), with the ones
before them: python tools/ncu_sass_hot.py report.ncu-rep [N] [context]"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
body = [r for r in rows[2:] if len(r) == len(hdr)]
iS = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[iS] or 0) for r in body) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 3
idx = sorted(range(len(body)), key=lambda i: -float(body[i][iS] or 0))[:n]
for i in sorted(idx):
    print("-----")
    for j in range(max(0, i - ctx), i + 1):
        r = body[j]
        print(f"{100 * float(r[iS] or 0) / tot:5.1f}%  {r[0][-5:]}  {r[1].strip()[:90]}")
