"""Table 1 / Fig. 2 analog of the paper with libdvm:
E_1 after one TVD-RK2 step of dt = 0.01 from the BKW datum for N = 8..128 and
N̄ in {1, 3, 7, 14, 28} (N̄ <= Ñ) on the paper's boxes, and E_1(t) for N = 32
and 64 up to t = 4.  Operator: the Carleman weights a(k) = h^2/(π gcd k)
(c = 1, reading R24); then the printed weights h^3|k|/gcd k scaled
by the fitted constant for comparison.
Usage: python tools/bkw_table.py > profiles/r02/bkw_table.txt"""
import sys

sys.path.insert(0, ".")
from paper_1201_3986_b200 import bkw  # noqa: E402
from paper_1201_3986_b200 import Plan  # noqa: E402

nbars = [1, 3, 7, 14, 28]
for weights in ("carleman", "printed"):
    c = 1.0 if weights == "carleman" else bkw.calibrate(weights="printed")
    print(f"== weights {weights}: a(k) = " + ("h^2/(pi gcd k), c = 1" if weights == "carleman"
                                              else f"h^3|k|/gcd k, fitted c = {c:.6f}"))
    print("E_1 after one step, dt = 0.01 (rows N, columns N̄; x = N̄ > Ñ)")
    print("   N  Ñ   " + "  ".join(f"N̄={nb:<8d}" for nb in nbars))
    for N in (8, 16, 32, 64, 128):
        if weights == "carleman" and N < 16:
            continue  # general weights run on the spectral path, N >= 16
        Nt = Plan(2, N, 1, L=bkw.PAPER_BOX[N]).Ntilde
        row = []
        for nb in nbars:
            row.append(f"{bkw.run(N, nb, c, weights=weights)[0]:.4e}" if nb <= Nt else "    x     ")
        print(f"{N:4d} {Nt:3d}   " + "  ".join(row), flush=True)
    print()
    print("E_1(t), N̄ = 3 and N̄ = Ñ, dt = 0.01 (Fig. 2 analog)")
    for N in (32, 64):
        Nt = Plan(2, N, 1, L=bkw.PAPER_BOX[N]).Ntilde
        for nb in (3, Nt):
            _, hist = bkw.run(N, nb, c, nsteps=400, record_every=25, weights=weights)
            print(f"N={N} N̄={nb}: " + ", ".join(f"t={t:.2f}:{e:.3e}" for t, e in hist), flush=True)
    print()
