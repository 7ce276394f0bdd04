"""Pins for the CPU oracle (oracle/dvm_oracle.c) against what the paper and the
mathematics fix -- never against itself.  CPU only (`-m "not gpu"`).

P1  hand-worked two-delta collisions (tests/golden/two_delta.txt) + the general
    Thales-circle rule on random, wrapping configurations
P2  N̄ = Ñ  =>  plain eq:DR over every orthogonal pair of the box
P3  C oracle == independent NumPy brute force (oracle/brute.py) on tiny grids
P4  exact mass conservation
P5  f = const  =>  Q = 0 exactly (bracket of eq:DR vanishes)
P6  no-aliasing support  =>  momentum and energy conserved (eq:weakpe)
P7  translation / reflection / axis-permutation equivariance; even f => even Q
P8  lattice Maxwellian is an equilibrium up to wrap-around
P9  Q(cf) = c^2 Q(f) and Q ∝ h^{d+1} at fixed nodal data (eq:DR + PAPER.md:582-587)
P10 gain coefficients non-negative: G >= 0 for f >= 0
P11 direction counts: Fig. 1 (16 lines), A^1 = 4(|F^1|-1) with |F^1| by its
    definition, Möbius closed form in 2D/3D, partition property;
    Ñ rule values 1,3,7,14
P12 the pseudo-spectral route (eq:sysDiff, eq:betaKL): the
    dense β(K,L) evaluation (oracle/cross.py, its own pair set) equals the oracle
P13 the box-truncated D^tr (oracle/cross.py) conserves mass,
    momentum and energy for any f, and equals the periodized operator when no
    collision of supp f leaves the box
P14 general decoupled weights Γ̃_{k,l} = a(k) b(l) (eq:decoup, PAPER.md:575-579;
    SURVEY §8(f) row 2): the weighted oracle equals the weighted brute force and
    the weighted dense-β route; mass is conserved for even a and any b, and
    broken by an odd a; f = const gives 0; a cosine mode cos(2πK.i/N) gives the
    spatially constant Q = Σ_{(k,l)} a(k) b(l) sin(2πK.k/N) sin(2πK.l/N)
    (the e_{±2K} terms of the bracket cancel; non-zero only when neither a nor b is even); the default tables reproduce the
    built-in weights bit for bit
"""
import itertools
import math
import os

import numpy as np
import pytest

from oracle import brute, oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "two_delta.txt")


def _idx(coords, N):
    i = 0
    for c in coords:
        i = i * N + (c % N)
    return i


def _rep(c, N):
    """Representative of c mod N in [-N/2, N/2)."""
    c %= N
    return c - N if c >= N - N // 2 else c


# ---------------------------------------------------------------- P1
def _parse_golden():
    groups = {}
    with open(GOLDEN) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            head, a, b, rest = [s.strip() for s in line.split("|")]
            d, N, L, Nt, Nb = head.split()
            node, expr = [s.strip() for s in rest.split(":")]
            val = eval(expr, {"s2": math.sqrt(2.0), "s5": math.sqrt(5.0)})
            key = (int(d), int(N), float(L), int(Nt), int(Nb),
                   tuple(map(int, a.split(","))), tuple(map(int, b.split(","))))
            groups.setdefault(key, []).append((tuple(map(int, node.split(","))), val))
    return groups


@pytest.mark.parametrize("key", list(_parse_golden().keys()), ids=str)
def test_p1_two_delta_golden(key):
    d, N, L, Nt, Nb, a, b = key
    expect = _parse_golden()[key]
    base = tuple(3 + j for j in range(d))  # place node a away from the origin
    f = np.zeros(N ** d)
    pa = tuple(x + y for x, y in zip(base, a))
    pb = tuple(x + y for x, y in zip(base, b))
    f[_idx(pa, N)] += 1.0
    f[_idx(pb, N)] += 1.0
    Q, G, Lo = oracle.collide(f, d, N, Nb, Nt, L)
    Q = Q[0]
    want = np.zeros(N ** d)
    for node, val in expect:
        want[_idx(tuple(x + y for x, y in zip(base, node)), N)] = val
    np.testing.assert_allclose(Q, want, rtol=0, atol=1e-13)


def _thales_rule(d, N, Nt, Nb, h, pa, pb):
    """Independent closed form of Q for f = δ_pa + δ_pb (pa != pb)."""
    def allowed(k):
        g = 0
        for c in k:
            g = math.gcd(g, abs(c))
        return g > 0 and max(abs(c) // g for c in k) <= Nb

    def weight(k):
        g = 0
        for c in k:
            g = math.gcd(g, abs(c))
        return h ** (d + 1) * math.sqrt(sum(c * c for c in k)) / g

    inbox = lambda v: max(abs(c) for c in v) <= Nt
    Q = np.zeros(N ** d)
    for i in itertools.product(range(N), repeat=d):
        gain = 0.0
        for p, q in ((pa, pb), (pb, pa)):
            k = tuple(_rep(x - y, N) for x, y in zip(p, i))
            l = tuple(_rep(x - y, N) for x, y in zip(q, i))
            if inbox(k) and inbox(l) and allowed(k) and sum(x * y for x, y in zip(k, l)) == 0:
                gain += weight(k)
        loss = 0.0
        if tuple(i) in (pa, pb):
            j = pb if tuple(i) == pa else pa
            for k in itertools.product(range(-Nt, Nt + 1), repeat=d):
                if not allowed(k):
                    continue
                # l must satisfy i + k + l ≡ j (mod N) with l in the box
                for l in itertools.product(range(-Nt, Nt + 1), repeat=d):
                    if all((ii + kk + ll - jj) % N == 0 for ii, kk, ll, jj in zip(i, k, l, j)) \
                            and sum(x * y for x, y in zip(k, l)) == 0:
                        loss += weight(k)
        Q[_idx(i, N)] = gain - loss
    return Q


@pytest.mark.parametrize("seed", range(6))
def test_p1_two_delta_rule_random(seed):
    rng = np.random.default_rng(100 + seed)
    d = 2
    N = int(rng.choice([9, 10, 12]))
    Nt = int(rng.integers(1, (N - 1) // 2 + 1))
    Nb = int(rng.integers(1, Nt + 1))
    L = float(rng.uniform(1.0, 6.0))
    h = 2 * L / N
    pa = tuple(int(x) for x in rng.integers(0, N, size=d))
    while True:
        pb = tuple(int(x) for x in rng.integers(0, N, size=d))
        if pb != pa:
            break
    f = np.zeros(N ** d)
    f[_idx(pa, N)] = 1.0
    f[_idx(pb, N)] = 1.0
    Q = oracle.collide(f, d, N, Nb, Nt, L)[0][0]
    want = _thales_rule(d, N, Nt, Nb, h, pa, pb)
    np.testing.assert_allclose(Q, want, rtol=0, atol=1e-12 * max(1.0, np.abs(want).max()))


def test_p1_two_delta_rule_3d():
    d, N, Nt, Nb, L = 3, 7, 2, 1, 2.0
    h = 2 * L / N
    pa, pb = (1, 5, 2), (2, 6, 2)
    f = np.zeros(N ** d)
    f[_idx(pa, N)] = 1.0
    f[_idx(pb, N)] = 1.0
    Q = oracle.collide(f, d, N, Nb, Nt, L)[0][0]
    want = _thales_rule(d, N, Nt, Nb, h, pa, pb)
    np.testing.assert_allclose(Q, want, rtol=0, atol=1e-12 * np.abs(want).max())


# ---------------------------------------------------------------- P2
def _plain_eq_dr(f, Nt, h):
    """eq:DR with no line truncation at all: every orthogonal (k,l) of the box."""
    d = f.ndim
    Q = np.zeros_like(f)
    axes = tuple(range(d))
    sh = lambda o: np.roll(f, tuple(-c for c in o), axes)
    for k in itertools.product(range(-Nt, Nt + 1), repeat=d):
        if not any(k):
            continue
        g = 0
        for c in k:
            g = math.gcd(g, abs(c))
        a = h ** (d + 1) * math.sqrt(sum(c * c for c in k)) / g
        for l in itertools.product(range(-Nt, Nt + 1), repeat=d):
            if sum(x * y for x, y in zip(k, l)) == 0:
                Q += a * (sh(k) * sh(l) - f * sh(tuple(x + y for x, y in zip(k, l))))
    return Q


@pytest.mark.parametrize("d,N,Nt", [(2, 9, 4), (2, 12, 3), (3, 6, 2), (3, 7, 3)])
def test_p2_full_directions_equal_eq_dr(d, N, Nt):
    f = np.random.default_rng(7).uniform(0, 1, size=(N,) * d)
    L = 3.0
    Q = oracle.collide(f, d, N, Nt, Nt, L)[0][0].reshape(f.shape)
    want = _plain_eq_dr(f, Nt, 2 * L / N)
    np.testing.assert_allclose(Q, want, rtol=0, atol=1e-13 * np.abs(want).max())


def test_p2_pair_counts_full():
    # With N̄ = Ñ the pair list is every (k != 0, l) orthogonal pair of the box.
    for d, Nt in [(2, 4), (2, 7), (3, 3)]:
        box = list(itertools.product(range(-Nt, Nt + 1), repeat=d))
        cnt = sum(1 for k in box if any(k) for l in box if sum(x * y for x, y in zip(k, l)) == 0)
        k, l, a = oracle.pairs(d, Nt, Nt, 1.0)
        assert len(a) == cnt


# ---------------------------------------------------------------- P3
@pytest.mark.parametrize("case", range(10))
def test_p3_brute_force_tiny(case):
    rng = np.random.default_rng(1000 + case)
    d = 2 if case < 6 else 3
    N = int(rng.choice([6, 7, 8, 10])) if d == 2 else int(rng.choice([5, 6, 7]))
    Nt = int(rng.integers(1, (N - 1) // 2 + 1))
    Nb = int(rng.integers(1, Nt + 1))
    L = float(rng.uniform(0.5, 5.0))
    f = rng.uniform(-1, 1, size=(N,) * d)
    Q = oracle.collide(f, d, N, Nb, Nt, L)[0][0].reshape(f.shape)
    want = brute.collide(f, Nb, Nt, 2 * L / N)
    np.testing.assert_allclose(Q, want, rtol=0, atol=1e-13 * max(np.abs(want).max(), 1e-300))


def test_points_variant_matches_full():
    f = np.random.default_rng(3).uniform(0, 1, size=(2, 8 ** 3))
    Q, G, Lo = oracle.collide(f, 3, 8, 2, 3, 4.0)
    pts = np.array([0, 7, 100, 511, 256])
    Qp, Gp, Lp = oracle.collide(f, 3, 8, 2, 3, 4.0, points=pts)
    assert np.array_equal(Qp, Q[:, pts]) and np.array_equal(Gp, G[:, pts]) and np.array_equal(Lp, Lo[:, pts])


# ---------------------------------------------------------------- P4, P5, P10
@pytest.mark.parametrize("d,N,Nb,Nt", [(2, 16, 4, 4), (2, 16, 2, 5), (2, 20, 3, 6), (3, 10, 1, 3), (3, 12, 2, 3)])
def test_p4_mass_p10_gain_nonneg(d, N, Nb, Nt):
    f = np.random.default_rng(11).uniform(0, 1, size=N ** d)
    Q, G, Lo = oracle.collide(f, d, N, Nb, Nt, 8.0)
    assert abs(Q.sum()) <= 1e-13 * G.sum()
    assert (G >= 0).all() and (Lo >= 0).all()
    np.testing.assert_allclose(Q, G - Lo, rtol=0, atol=1e-13 * G.max())


@pytest.mark.parametrize("c", [1.0, 0.3, 2.5])
def test_p5_constant_is_exact_zero(c):
    for d, N, Nb, Nt in [(2, 16, 3, 4), (3, 8, 2, 3)]:
        Q, G, _ = oracle.collide(np.full(N ** d, c), d, N, Nb, Nt, 8.0)
        assert np.all(Q == 0.0) and G.min() > 0


# ---------------------------------------------------------------- P6
@pytest.mark.parametrize("d,N,Nt,Nb", [(2, 16, 4, 2), (2, 16, 4, 4), (3, 12, 3, 2)])
def test_p6_no_alias_conservation(d, N, Nt, Nb):
    s = N // 2 - 1 - Nt  # support half-width allowed by the no-aliasing condition
    L = 4.0
    h = 2 * L / N
    rng = np.random.default_rng(5)
    f = np.zeros((N,) * d)
    sl = tuple(slice(N // 2 - s, N // 2 + s + 1) for _ in range(d))
    f[sl] = rng.uniform(0.1, 1.0, size=f[sl].shape)
    Q, G, _ = oracle.collide(f, d, N, Nb, Nt, L)
    Q = Q[0].reshape(f.shape)
    v = [((np.arange(N) - N // 2) * h).reshape([N if j == a else 1 for j in range(d)]) for a in range(d)]
    scale = (G.sum()) * (N // 2 * h) ** 2
    assert abs(Q.sum()) <= 1e-13 * G.sum()
    for a in range(d):
        assert abs((v[a] * Q).sum()) <= 1e-13 * scale
    assert abs((sum(x * x for x in v) * Q).sum()) <= 1e-13 * scale
    # one node wider breaks it (the condition is sharp)
    s2 = s + 2
    f2 = np.zeros((N,) * d)
    sl2 = tuple(slice(N // 2 - s2, N // 2 + s2 + 1) for _ in range(d))
    f2[sl2] = rng.uniform(0.1, 1.0, size=f2[sl2].shape)
    Q2, G2, _ = oracle.collide(f2, d, N, Nb, Nt, L)
    Q2 = Q2[0].reshape(f2.shape)
    assert abs((sum(x * x for x in v) * Q2).sum()) > 1e-6 * G2.sum() * (N // 2 * h) ** 2


# ---------------------------------------------------------------- P7
def test_p7_equivariance():
    d, N, Nb, Nt = 3, 9, 2, 3
    f = np.random.default_rng(9).uniform(0, 1, size=(N,) * d)
    run = lambda g: oracle.collide(g, d, N, Nb, Nt, 3.0)[0][0].reshape(g.shape)
    Q = run(f)
    sc = np.abs(Q).max()
    # translation (bitwise: same per-node summation order)
    t = (2, -3, 4)
    assert np.array_equal(run(np.roll(f, t, (0, 1, 2))), np.roll(Q, t, (0, 1, 2)))
    # axis permutation and reflection
    perm = (2, 0, 1)
    np.testing.assert_allclose(run(np.transpose(f, perm)), np.transpose(Q, perm), rtol=0, atol=1e-14 * sc)
    refl = lambda g: np.roll(np.flip(g, 1), 1, 1)  # j -> N - j (mod N) on axis 1
    np.testing.assert_allclose(run(refl(f)), refl(Q), rtol=0, atol=1e-14 * sc)


def test_p7_even_f_even_q_zero_momentum():
    d, N, Nb, Nt, L = 2, 16, 3, 4, 8.0
    f = np.random.default_rng(4).uniform(0, 1, size=(N, N))
    refl = lambda g: np.roll(np.flip(g, (0, 1)), (1, 1), (0, 1))  # v -> -v on the node-centred grid
    fe = f + refl(f)
    Q = oracle.collide(fe, d, N, Nb, Nt, L)[0][0].reshape(N, N)
    sc = np.abs(Q).max()
    np.testing.assert_allclose(Q, refl(Q), rtol=0, atol=1e-14 * sc)
    # Zero global momentum: on the periodic node-centred grid the
    # node x_j = 0 (v = -L) is its own mirror image, so it is left out of the sum.
    h = 2 * L / N
    v = (np.arange(N) - N // 2) * h
    v[0] = 0.0
    assert abs((v[:, None] * Q).sum()) <= 1e-13 * sc * N * N * L
    assert abs((v[None, :] * Q).sum()) <= 1e-13 * sc * N * N * L


# ---------------------------------------------------------------- P8
def test_p8_lattice_maxwellian_equilibrium():
    d, N, Nb, Nt, L = 2, 32, 3, 7, 8.0
    h = 2 * L / N
    v = (np.arange(N) - N // 2) * h
    ratios = []
    for T in (2.0, 1.0, 0.5):
        f = np.exp(-((v[:, None] - 0.3) ** 2 + (v[None, :] + 0.2) ** 2) / (2 * T))
        Q, G, _ = oracle.collide(f, d, N, Nb, Nt, L)
        ratios.append(np.abs(Q).max() / G.max())
    # a non-equilibrium datum of the same scale is far from zero
    g = np.exp(-((v[:, None] - 1.5) ** 2 + v[None, :] ** 2) / 2) + np.exp(-((v[:, None] + 1.5) ** 2 + v[None, :] ** 2) / 2)
    Qg, Gg, _ = oracle.collide(g, d, N, Nb, Nt, L)
    assert np.abs(Qg).max() / Gg.max() > 1e-2
    assert ratios[0] > ratios[1] > ratios[2]  # residual is wrap-around only: shrinks with the tail mass
    assert ratios[2] < 1e-9


# ---------------------------------------------------------------- P9
def test_p9_scaling():
    d, N, Nb, Nt = 3, 8, 2, 3
    f = np.random.default_rng(2).uniform(0, 1, size=N ** d)
    Q1 = oracle.collide(f, d, N, Nb, Nt, 4.0)[0]        # h = 1
    Q2 = oracle.collide(f, d, N, Nb, Nt, 8.0)[0]        # h = 2: exactly 2^{d+1} times
    assert np.array_equal(Q2, Q1 * 2.0 ** (d + 1))
    Qc = oracle.collide(3.0 * f, d, N, Nb, Nt, 4.0)[0]
    np.testing.assert_allclose(Qc, 9.0 * Q1, rtol=0, atol=1e-13 * np.abs(Qc).max())


# ---------------------------------------------------------------- P11
def _mobius(n):
    mu, m, p = 1, n, 2
    while p * p <= m:
        if m % p == 0:
            m //= p
            if m % p == 0:
                return 0
            mu = -mu
        p += 1
    return -mu if m > 1 else mu


def test_p11_direction_counts():
    # PAPER.md Fig. 1 (N=7, N̄=3): 16 lines through 0.
    assert len(oracle.directions(2, 3)) == 16
    for Nb in range(1, 21):
        # |F^1| straight from its definition
        F1 = sum(1 for q in range(1, Nb + 1) for p in range(0, q + 1) if math.gcd(p, q) == 1)
        A = len(oracle.directions(2, Nb))
        assert A == 4 * (F1 - 1)
        assert A == sum(_mobius(t) * ((2 * (Nb // t) + 1) ** 2 - 1) for t in range(1, Nb + 1)) // 2
    for Nb in range(1, 10):
        A3 = len(oracle.directions(3, Nb))
        assert A3 == sum(_mobius(t) * ((2 * (Nb // t) + 1) ** 3 - 1) for t in range(1, Nb + 1)) // 2
    assert [len(oracle.directions(3, n)) for n in (1, 2, 3, 4, 8)] == [13, 49, 145, 289, 2017]


def test_p11_partition_property():
    for d, Nb, Nt in [(2, 4, 7), (3, 3, 5)]:
        dirs = [tuple(e) for e in oracle.directions(d, Nb)]
        for k in itertools.product(range(-Nt, Nt + 1), repeat=d):
            if not any(k):
                continue
            g = 0
            for c in k:
                g = math.gcd(g, abs(c))
            hits = [e for e in dirs if any(all(m * x == y for x, y in zip(e, k)) for m in range(-Nt, Nt + 1) if m)]
            assert len(hits) == (1 if max(abs(c) // g for c in k) <= Nb else 0)


def test_ntilde_rule_paper_values():
    # PAPER.md:978-980 (and N̄ = 28 <= Ñ at N = 128 in Table 2)
    assert [oracle.ntilde_rule(N, 1) for N in (8, 16, 32, 64, 128)] == [1, 3, 7, 14, 28]
    # BASELINE configs (reading R2): c1 raises Ñ to N̄ = 4
    assert [oracle.ntilde_rule(N, Nb) for N, Nb in ((16, 4), (64, 8), (256, 16), (32, 4), (64, 8))] == [4, 14, 57, 7, 14]


# ---------------------------------------------------------------- P12, P13: cross-oracles
@pytest.mark.parametrize("d,N,Nb,Nt", [(2, 8, 1, 3), (2, 9, 2, 4), (2, 12, 3, 5), (3, 5, 1, 2), (3, 6, 2, 2)])
def test_p12_pseudo_spectral_route(d, N, Nb, Nt):
    from oracle import cross
    f = np.random.default_rng(N * 10 + d).uniform(0.0, 1.0, N ** d)
    Qo = oracle.collide(f, d, N, Nb, Nt, 8.0)[0].reshape(-1)
    Qb, imag = cross.dense_beta_Q(f, d, N, Nb, Nt, 8.0)
    scale = np.abs(Qo).max()
    assert np.abs(Qb - Qo).max() <= 1e-13 * scale
    assert imag <= 1e-13 * scale  # real f: the spectral sum is real


@pytest.mark.parametrize("d,N,Nb,Nt", [(2, 12, 2, 3), (3, 7, 1, 2)])
def test_p13_truncated_operator_conserves_and_matches_interior(d, N, Nb, Nt):
    from oracle import cross
    L = 8.0
    h = 2 * L / N
    v = (np.arange(N) - N // 2) * h
    V = np.stack(np.meshgrid(*([v] * d), indexing="ij"), axis=-1).reshape(-1, d)
    f = np.random.default_rng(2 + d).uniform(0.0, 1.0, N ** d)
    Dt = cross.D_tr(f, d, N, Nb, Nt, L)
    scale = np.abs(Dt).sum() * (1 + np.abs(V).max() ** 2)
    assert abs(Dt.sum()) <= 1e-14 * scale
    for j in range(d):
        assert abs((Dt * V[:, j]).sum()) <= 1e-14 * scale
    assert abs((Dt * (V ** 2).sum(1)).sum()) <= 1e-14 * scale
    # the periodized operator is not conservative for this f (it wraps) ...
    Qo = oracle.collide(f, d, N, Nb, Nt, L)[0].reshape(-1)
    assert abs((Qo * (V ** 2).sum(1)).sum()) > 1e-6 * scale
    # ... but equals D^tr when every collision of supp f stays in the box
    g = np.zeros((N,) * d)
    lo, hi = N // 2 - 1, N // 2 + 1
    sl = tuple(slice(lo, hi) for _ in range(d))
    g[sl] = np.random.default_rng(5).uniform(0.5, 1.0, g[sl].shape)
    Qg = oracle.collide(g.reshape(-1), d, N, Nb, Nt, L)[0].reshape(-1)
    Dg = cross.D_tr(g.reshape(-1), d, N, Nb, Nt, L)
    assert np.abs(Dg - Qg).max() <= 1e-13 * np.abs(Qg).max()


# ---------------------------------------------------------------- P14: general weights a(k) b(l)
def _even_table(d, Nt, seed, lo=0.5, hi=1.5):
    r = np.random.default_rng(seed).uniform(lo, hi, size=(2 * Nt + 1,) * d)
    return 0.5 * (r + np.flip(r))  # w(-k) = w(k)


@pytest.mark.parametrize("d,N,Nb,Nt", [(2, 8, 2, 3), (2, 10, 3, 4), (3, 6, 1, 2), (3, 7, 2, 3)])
def test_p14_weighted_oracle_vs_brute_and_dense_beta(d, N, Nb, Nt):
    from oracle import cross
    a = _even_table(d, Nt, 100 + N)
    b = _even_table(d, Nt, 200 + N)
    L = 4.0
    f = np.random.default_rng(N + d).uniform(0.0, 1.0, size=(N,) * d)
    Qo = oracle.collide(f, d, N, Nb, Nt, L, a_box=a, b_box=b)[0].reshape(f.shape)
    Qb = brute.collide(f, Nb, Nt, 2 * L / N, a_box=a, b_box=b)
    scale = np.abs(Qb).max()
    np.testing.assert_allclose(Qo, Qb, rtol=0, atol=1e-13 * scale)
    Qs, imag = cross.dense_beta_Q(f.reshape(-1), d, N, Nb, Nt, L, a_box=a, b_box=b)
    assert np.abs(Qs - Qo.reshape(-1)).max() <= 1e-13 * scale and imag <= 1e-13 * scale
    # the weights enter: the unweighted operator differs
    assert np.abs(oracle.collide(f, d, N, Nb, Nt, L)[0].reshape(f.shape) - Qo).max() > 1e-3 * scale


@pytest.mark.parametrize("d,N,Nb,Nt", [(2, 16, 3, 5), (3, 8, 2, 3)])
def test_p14_weighted_mass_and_constant(d, N, Nb, Nt):
    a = _even_table(d, Nt, 7)
    b = np.random.default_rng(8).uniform(0.0, 2.0, size=(2 * Nt + 1,) * d)  # b need not be even
    f = np.random.default_rng(9).uniform(0.0, 1.0, N ** d)
    Q, G, _ = oracle.collide(f, d, N, Nb, Nt, 8.0, a_box=a, b_box=b)
    assert abs(Q.sum()) <= 1e-13 * G.sum()
    # an odd part in a breaks the k -> -k pairing that conserves mass
    a_odd = a * (1.0 + 0.5 * np.sign(np.arange(a.size).reshape(a.shape) - a.size // 2))
    Q2, G2, _ = oracle.collide(f, d, N, Nb, Nt, 8.0, a_box=a_odd, b_box=b)
    assert abs(Q2.sum()) > 1e-6 * G2.sum()
    Qc, Gc, _ = oracle.collide(np.full(N ** d, 0.7), d, N, Nb, Nt, 8.0, a_box=a, b_box=b)
    assert np.all(Qc == 0.0) and Gc.min() > 0


@pytest.mark.parametrize("d,N,Nb,Nt,K", [(2, 16, 3, 5, (1, 2)), (2, 12, 2, 4, (3, 0)), (3, 8, 2, 3, (1, 0, 2))])
def test_p14_cosine_mode_closed_form(d, N, Nb, Nt, K):
    from oracle import cross
    # neither table even: for even a (b) the k -> -k (l -> -l) pairing makes the sum vanish
    a = np.random.default_rng(30 + d).uniform(0.5, 1.5, size=(2 * Nt + 1,) * d)
    b = np.random.default_rng(40 + d).uniform(0.5, 1.5, size=(2 * Nt + 1,) * d)
    grid = np.stack(np.meshgrid(*([np.arange(N)] * d), indexing="ij"), axis=-1).reshape(-1, d)
    th = 2 * np.pi * np.asarray(K, dtype=np.float64) / N
    f = np.cos(grid @ th)
    Q = oracle.collide(f, d, N, Nb, Nt, 8.0, a_box=a, b_box=b)[0].reshape(-1)
    k, l, _ = cross._pairs(d, N, Nb, Nt, 8.0)
    w = np.array([a[tuple(kk + Nt)] * b[tuple(ll + Nt)] for kk, ll in zip(k, l)])
    want = float((w * np.sin(k @ th) * np.sin(l @ th)).sum())
    assert abs(want) > 1e-3
    np.testing.assert_allclose(Q, want, rtol=0, atol=1e-12 * np.abs(w).sum())


@pytest.mark.parametrize("d,N,Nb,Nt", [(2, 16, 4, 4), (3, 8, 2, 3)])
def test_p14_default_tables_reproduce_builtin(d, N, Nb, Nt):
    L = 8.0
    h = 2 * L / N
    a = np.zeros((2 * Nt + 1,) * d)
    for k in itertools.product(range(-Nt, Nt + 1), repeat=d):
        if any(k):
            g = 0
            for c in k:
                g = math.gcd(g, abs(c))
            a[tuple(c + Nt for c in k)] = h ** (d + 1) * math.sqrt(sum(c * c for c in k)) / g
    f = np.random.default_rng(4).uniform(0.0, 1.0, N ** d)
    Q0 = oracle.collide(f, d, N, Nb, Nt, L)[0]
    Q1 = oracle.collide(f, d, N, Nb, Nt, L, a_box=a, b_box=np.ones_like(a))[0]
    assert np.array_equal(Q0, Q1)
