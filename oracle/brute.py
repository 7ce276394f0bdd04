"""O0: tiny-grid brute force of the periodized DVM, in NumPy (independent of the C oracle).

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py).  Used solely to cross-check
oracle/dvm_oracle.c on tiny grids (pin P3).  It does not build a pair list:
it loops over every (k, l) in the box squared and tests the conditions of
eq:DR + line truncation inline, and it
applies each term to the whole grid at once with periodic np.roll, so its
summation order and index arithmetic differ from the C oracle's.
"""
from __future__ import annotations

import itertools
import math

import numpy as np


def _line_order(k):
    g = 0
    for c in k:
        g = math.gcd(g, abs(c))
    return max(abs(c) // g for c in k), g


def collide(f: np.ndarray, Nbar: int, Ntilde: int, h: float, a_box=None, b_box=None):
    """f has shape [N]*d.  Returns Q with the same shape.  a_box, b_box:
    optional decoupled weights a(k), b(l) (eq:decoup) as
    arrays of shape [2Ñ+1]*d indexed by k + Ñ."""
    f = np.asarray(f, dtype=np.float64)
    d = f.ndim
    rng = range(-Ntilde, Ntilde + 1)
    Q = np.zeros_like(f)
    axes = tuple(range(d))

    def shifted(o):  # g(i) = f(i + o), periodic
        return np.roll(f, shift=tuple(-c for c in o), axis=axes)

    for k in itertools.product(rng, repeat=d):
        if not any(k):
            continue
        order, g = _line_order(k)
        if order > Nbar:
            continue
        a = h ** (d + 1) * math.sqrt(sum(c * c for c in k)) / g
        if a_box is not None:
            a = float(a_box[tuple(c + Ntilde for c in k)])
        fk = shifted(k)
        for l in itertools.product(rng, repeat=d):
            if sum(x * y for x, y in zip(k, l)) != 0:
                continue
            kl = tuple(x + y for x, y in zip(k, l))
            w = a if b_box is None else a * float(b_box[tuple(c + Ntilde for c in l)])
            Q += w * (fk * shifted(l) - f * shifted(kl))
    return Q
