"""The regroupings the GPU paths evaluate, checked against the oracle's separate
gain (G) and loss (Lo) outputs on small grids (CPU, NumPy; `-m "not gpu"`).

R21  loss:  Σ_e a_e f U_e = f · (λ ⊛ f),  λ(j) = Σ_e a_e #{(m, l): 1<=|m|<=M_e,
     l ∈ P_e, me + l ≡ j}  (β̃ = β − β(L,L))
     -> dvm_loss.cu
gain per direction: G = Σ_e a_e S_e T_e, S_e = Σ_{m≠0} f(.+me), T_e = Σ_{P_e} f(.+l)
     (eq:decD) -> dvm_gain3d.cu
2D pairs: P_e = {n e⊥ : |n| <= M_e} and e⊥ is a direction with the same M_e, a_e,
     so G = Σ_{pairs} a_e [(W_e − f) W_e⊥ + (W_e⊥ − f) W_e]  -> dvm_pair2d.cu
These are identities of finite sums, so they hold to rounding.
"""
import itertools

import numpy as np
import pytest

from oracle import oracle


def _dirs(d, Nbar):
    return [tuple(int(c) for c in e) for e in oracle.directions(d, Nbar)]


def _perp_set(e, Nt):
    d = len(e)
    return [l for l in itertools.product(range(-Nt, Nt + 1), repeat=d) if sum(a * b for a, b in zip(l, e)) == 0]


def _shift(f, v):
    """g(x) = f(x + v) on the periodic grid."""
    return np.roll(f, shift=tuple(-c for c in v), axis=tuple(range(f.ndim)))


def _lam(d, N, Nbar, Nt, h):
    lam = np.zeros((N,) * d)
    for e in _dirs(d, Nbar):
        M = Nt // max(abs(c) for c in e)
        a = h ** (d + 1) * float(np.sqrt(sum(c * c for c in e)))
        P = _perp_set(e, Nt)
        for m in list(range(-M, 0)) + list(range(1, M + 1)):
            for l in P:
                j = tuple((m * ec + lc) % N for ec, lc in zip(e, l))
                lam[j] += a
    return lam


@pytest.mark.parametrize("d,N,Nbar,Nt", [(2, 16, 3, 4), (2, 12, 2, 5), (3, 8, 1, 3), (3, 10, 2, 3)])
def test_r21_loss_is_one_convolution(d, N, Nbar, Nt):
    L = 8.0
    h = 2 * L / N
    f = np.random.default_rng(N * d + Nbar).uniform(0.0, 1.0, size=(N,) * d)
    lam = _lam(d, N, Nbar, Nt, h)
    # λ is even: λ(-j) = λ(j) (m -> -m, l -> -l), so λ̂ is real
    neg = lam[tuple(np.ix_(*[(-np.arange(N)) % N] * d))]
    assert np.array_equal(lam, neg)
    Lam = np.real(np.fft.ifftn(np.fft.fftn(lam) * np.fft.fftn(f)))
    _, _, Lo = oracle.collide(f.reshape(-1), d, N, Nbar, Nt, L)
    Lo = Lo.reshape((N,) * d)
    np.testing.assert_allclose(f * Lam, Lo, rtol=0, atol=1e-13 * np.abs(Lo).max())


@pytest.mark.parametrize("d,N,Nbar,Nt", [(2, 16, 3, 4), (3, 8, 1, 3), (3, 10, 2, 3)])
def test_gain_is_sum_of_line_times_plane(d, N, Nbar, Nt):
    L = 8.0
    h = 2 * L / N
    f = np.random.default_rng(7 + N).uniform(0.0, 1.0, size=(N,) * d)
    G = np.zeros_like(f)
    for e in _dirs(d, Nbar):
        M = Nt // max(abs(c) for c in e)
        a = h ** (d + 1) * float(np.sqrt(sum(c * c for c in e)))
        S = sum(_shift(f, tuple(m * c for c in e)) for m in list(range(-M, 0)) + list(range(1, M + 1)))
        T = sum(_shift(f, l) for l in _perp_set(e, Nt))
        G += a * S * T
    _, Go, _ = oracle.collide(f.reshape(-1), d, N, Nbar, Nt, L)
    np.testing.assert_allclose(G, Go.reshape((N,) * d), rtol=0, atol=1e-13 * np.abs(Go).max())


@pytest.mark.parametrize("N,Nbar,Nt", [(16, 4, 4), (16, 3, 7), (20, 5, 6)])
def test_2d_gain_direction_pairs(N, Nbar, Nt):
    L = 8.0
    h = 2 * L / N
    f = np.random.default_rng(N + Nbar).uniform(0.0, 1.0, size=(N, N))
    dset = set(_dirs(2, Nbar))

    def canon(v):
        return v if (v[0] > 0 or (v[0] == 0 and v[1] > 0)) else (-v[0], -v[1])

    pairs = set()
    for e in dset:
        ep = canon((-e[1], e[0]))
        assert ep in dset  # the table is closed under e -> e⊥
        pairs.add(tuple(sorted((e, ep))))
    assert 2 * len(pairs) == len(dset)
    G = np.zeros_like(f)
    for e, ep in pairs:
        M = Nt // max(abs(e[0]), abs(e[1]))
        assert M == Nt // max(abs(ep[0]), abs(ep[1]))
        a = h ** 3 * float(np.hypot(*e))
        We = sum(_shift(f, (m * e[0], m * e[1])) for m in range(-M, M + 1))
        Wp = sum(_shift(f, (m * ep[0], m * ep[1])) for m in range(-M, M + 1))
        G += a * ((We - f) * Wp + (Wp - f) * We)
    _, Go, _ = oracle.collide(f.reshape(-1), 2, N, Nbar, Nt, L)
    np.testing.assert_allclose(G, Go.reshape(N, N), rtol=0, atol=1e-13 * np.abs(Go).max())
