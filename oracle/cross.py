"""Cross-oracles for tiny grids (TEST INFRASTRUCTURE ONLY: imported by tests/,
never by the product path).  Independent routes to the operators of the paper,
used to pin oracle/dvm_oracle.c from outside its own formulation.

dense_beta_Q  the pseudo-spectral form of the periodized DVM (PAPER.md
              eq:sysDiff, eq:betaKL, lines 520-556): with the involution
              f~_I = (1/n^d) Σ_i f_i e_{-I}(i), f_i = Σ_I f~_I e_I(i),
              ∂_t f~_I = Σ_{K+L ≡ I} β~(K, L) f~_K f~_L,
              β~(K, L) = β(K, L) − β(L, L),
              β(K, L) = Σ_{k,l} Γ~_{k,l} e_K(k) e_L(l),
              over the same truncated pair set as the oracle (k on the lines of
              order <= N̄, |k|, |l| <= Ñ, k.l = 0; Γ~ = a(k), reading R5).
              O(n^{2d}): for n^d <= a few hundred nodes.
D_tr          the box-truncated operator of PAPER.md:371-381:
              D^tr_i = Σ_{k,l : i+k, i+l, i+k+l in the box} Γ~_{k,l} [f_{i+k} f_{i+l} − f_i f_{i+k+l}]
              (no periodization); completely conservative, not translation
              invariant.
Both build the truncated pair set from its definition here (no code shared
with oracle/dvm_oracle.c): k ≠ 0 in [-Ñ,Ñ]^d on a line of order <= N̄
(|k / gcd(k)|_inf <= N̄), l in [-Ñ,Ñ]^d with k.l = 0, Γ~_{k,l} = a(k) =
h^{d+1} |k| / gcd(k) (readings R4, R5, R8, R9), or
Γ~_{k,l} = a(k) b(l) from caller weight tables (eq:decoup).
"""
from __future__ import annotations

import itertools
import math

import numpy as np


def _pairs(d, N, Nbar, Ntilde, L, a_box=None, b_box=None):
    h = 2.0 * L / N
    box = list(itertools.product(range(-Ntilde, Ntilde + 1), repeat=d))
    K, Lp, A = [], [], []
    for k in box:
        if not any(k):
            continue
        g = 0
        for c in k:
            g = math.gcd(g, abs(c))
        if max(abs(c) for c in k) // g > Nbar:
            continue
        a = h ** (d + 1) * math.sqrt(sum(c * c for c in k)) / g
        if a_box is not None:  # eq:decoup with caller weights: Γ~ = a(k) b(l)
            a = float(a_box[tuple(c + Ntilde for c in k)])
        for l in box:
            if sum(x * y for x, y in zip(k, l)) == 0:
                K.append(k)
                Lp.append(l)
                A.append(a if b_box is None else a * float(b_box[tuple(c + Ntilde for c in l)]))
    return np.array(K, dtype=np.int64), np.array(Lp, dtype=np.int64), np.array(A, dtype=np.float64)


def dense_beta_Q(f, d, N, Nbar, Ntilde, L=8.0, a_box=None, b_box=None):
    """Q by the pseudo-spectral route (complex128), real part returned.
    a_box, b_box: optional decoupled weights (eq:decoup), [2Ñ+1]*d arrays."""
    k, l, a = _pairs(d, N, Nbar, Ntilde, L, a_box, b_box)
    grid = np.array(list(itertools.product(range(N), repeat=d)))  # mode index K (row-major)
    n = grid.shape[0]
    # E_k[p, K] = e_K(k_p) = exp(2πi K.k_p / N)
    Ek = np.exp(2j * np.pi * (k @ grid.T) / N)
    El = np.exp(2j * np.pi * (l @ grid.T) / N)
    beta = (Ek * a[:, None]).T @ El  # β(K, L), [n, n]
    diag = np.diag(beta).copy()  # β(L, L)
    bt = beta - diag[None, :]  # β~(K, L)
    fg = np.asarray(f, dtype=np.float64).reshape((N,) * d)
    ft = np.fft.fftn(fg) / n  # f~_I = (1/n) Σ_i f_i e_{-I}(i)
    fv = ft.reshape(-1)
    # index of K + L (mod N) in row-major order
    idx = np.zeros((n, n), dtype=np.int64)
    s = (grid[:, None, :] + grid[None, :, :]) % N
    for j in range(d):
        idx = idx * N + s[:, :, j]
    rhs = np.zeros(n, dtype=np.complex128)
    np.add.at(rhs, idx.reshape(-1), (bt * fv[:, None] * fv[None, :]).reshape(-1))
    Qg = np.fft.ifftn(rhs.reshape((N,) * d)) * n  # f_i = Σ_I f~_I e_I(i)
    return Qg.real.reshape(-1), np.abs(Qg.imag).max()


def D_tr(f, d, N, Nbar, Ntilde, L=8.0):
    """The box-truncated (non-periodized) operator on the N^d box."""
    k, l, a = _pairs(d, N, Nbar, Ntilde, L)
    fg = np.asarray(f, dtype=np.float64).reshape((N,) * d)
    Q = np.zeros_like(fg)
    for i in itertools.product(range(N), repeat=d):
        ii = np.array(i)
        acc = 0.0
        for kk, ll, aa in zip(k, l, a):
            ik, il, ikl = ii + kk, ii + ll, ii + kk + ll
            if (ik.min() < 0 or ik.max() >= N or il.min() < 0 or il.max() >= N or ikl.min() < 0
                    or ikl.max() >= N):
                continue
            acc += aa * (fg[tuple(ik)] * fg[tuple(il)] - fg[i] * fg[tuple(ikl)])
        Q[i] = acc
    return Q.reshape(-1)
