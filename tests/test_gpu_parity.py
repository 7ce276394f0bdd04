"""GPU parity: libdvm (through the C ABI) against the CPU oracle, element by
element on the same seeded inputs.  Bar (BASELINE.json north_star):
max|Q_gpu - Q_oracle| <= 1e-11 * max|Q_oracle| in fp64.

Full grids where the oracle finishes in seconds; at BASELINE full sizes
c3 and c4 on every node, c5 in bench.py's launch configuration (128 nodes in
each of the 512 cells plus one whole cell), plus invariants that hold at any
size.  Every tolerance scale is max|Q_oracle| over the compared nodes.
"""
import itertools
import os
import math

import numpy as np
import pytest

import dvm_inputs
from oracle import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-11


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _plan(d, N, Nbar, **kw):
    from paper_1201_3986_b200 import Plan
    return Plan(d, N, Nbar, **kw)


def _gpu(plan, f_np):
    f = torch.from_numpy(np.ascontiguousarray(f_np, dtype=np.float64)).cuda()
    q = plan.collide(f)
    torch.cuda.synchronize()
    return q.cpu().numpy()


def _assert_parity(Qg, Qo, what):
    """The bar of BASELINE.json north_star; the scale is always the oracle's."""
    scale = np.abs(Qo).max()
    err = np.abs(Qg - Qo).max()
    assert err <= TOL * scale, f"{what}: max err {err:.3e} > {TOL:g} * {scale:.3e} (rel {err / scale:.2e})"
    return err / scale


def _sample_points(f_cell, d, N, n_uniform, seed):
    arg = int(np.argmax(f_cell))
    c = []
    r = arg
    for _ in range(d):
        c.append(r % N)
        r //= N
    c = c[::-1]
    pts = set()
    for off in itertools.product((-1, 0, 1), repeat=d):
        idx = 0
        for j in range(d):
            idx = idx * N + (c[j] + off[j]) % N
        pts.add(idx)
    rng = np.random.default_rng(seed)
    pts.update(int(x) for x in rng.integers(0, N ** d, size=n_uniform))
    return np.array(sorted(pts), dtype=np.int64)


# ---------------------------------------------------------------- plan tables
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_direction_table_matches_definition(name):
    cfg = dvm_inputs.CONFIGS[name]
    p = _plan(cfg.d, cfg.N, cfg.Nbar)
    dirs, M, a, loc = p.directions()
    assert np.array_equal(dirs, oracle.directions(cfg.d, cfg.Nbar))
    assert p.Ntilde == oracle.ntilde_rule(cfg.N, cfg.Nbar)
    inf = np.abs(dirs).max(axis=1)
    assert np.array_equal(M, p.Ntilde // inf)
    np.testing.assert_allclose(a, p.h ** (cfg.d + 1) * np.sqrt((dirs.astype(float) ** 2).sum(1)), rtol=1e-15)
    assert loc.all()


@pytest.mark.parametrize("name", ["c2", "c4", "c5"])
def test_perp_rows_equal_perp_set(name):
    """The rows {αu+βw : lo<=α<=hi} of every direction are exactly
    P_e = {l in [-Ñ,Ñ]^d : l.e = 0}, each point once."""
    cfg = dvm_inputs.CONFIGS[name]
    p = _plan(cfg.d, cfg.N, cfg.Nbar)
    Nt = p.Ntilde
    dirs = p.directions()[0]
    box = np.array(list(itertools.product(range(-Nt, Nt + 1), repeat=cfg.d)))
    for i, e in enumerate(dirs):
        u, w, rows = p.geometry(i)
        if cfg.d == 3:
            assert np.array_equal(np.cross(u, w), e)  # basis of e^⊥ ∩ Z^3
        pts = []
        for b, lo, hi in rows:
            for al in range(lo, hi + 1):
                pts.append(tuple(al * u + b * w))
        want = {tuple(l) for l in box[box @ e == 0]}
        assert len(pts) == len(set(pts)) == len(want) and set(pts) == want, (i, e)


def test_lpt_sharding_matches_host_logic():
    from paper_1201_3986_b200 import parallel
    cfg = dvm_inputs.CONFIGS["c4"]
    full = _plan(3, cfg.N, cfg.Nbar)
    costs = [4 * len(full.geometry(i)[2]) + 8 for i in range(full.A)]
    for world in (2, 3, 8):
        owner = parallel.lpt_assign(costs, world)
        for r in range(world):
            loc = _plan(3, cfg.N, cfg.Nbar, shard_rank=r, shard_world=world).directions()[3]
            assert np.array_equal(loc, owner == r)


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_2d_shards_are_pair_units_matching_host_logic(name):
    """2D direction sharding assigns whole pair units {e, e⊥},
    exactly as paper_1201_3986_b200.parallel.owners_2d mirrors it."""
    from paper_1201_3986_b200 import parallel
    cfg = dvm_inputs.CONFIGS[name]
    full = _plan(2, cfg.N, cfg.Nbar)
    dirs, M, _, _ = full.directions()
    for world in (2, 3, 8):
        owner = parallel.owners_2d(dirs, M, world)
        for r in range(world):
            loc = _plan(2, cfg.N, cfg.Nbar, shard_rank=r, shard_world=world).directions()[3]
            assert np.array_equal(loc, owner == r), (world, r)


# ---------------------------------------------------------------- parity, full grids
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_parity_full_2d(name):
    cfg = dvm_inputs.CONFIGS[name]
    f = dvm_inputs.make(name)
    p = _plan(cfg.d, cfg.N, cfg.Nbar)
    Qg = _gpu(p, f)
    Qo, G, _ = oracle.collide(f, cfg.d, cfg.N, cfg.Nbar, p.Ntilde, cfg.L)
    _assert_parity(Qg, Qo, name)
    assert abs(Qg.sum()) <= 1e-13 * G.sum()


@pytest.mark.parametrize("d,N,Nbar,Nt", [(3, 16, 3, 3), (3, 16, 2, 7), (3, 8, 1, 3), (2, 32, 5, 7),
                                         (2, 8, 1, 3), (2, 4, 1, 1),
                                         # N = 32: the 3D frame-plane gain kernel + FFT loss, every node
                                         (3, 32, 1, 3), (3, 32, 2, 4), (3, 32, 3, 3)])
def test_parity_full_small(d, N, Nbar, Nt):
    f = dvm_inputs.two_bumps(d, N, 8.0, 1.5, 0.01, 3).reshape(-1)
    p = _plan(d, N, Nbar, Ntilde=Nt)
    Qg = _gpu(p, f)
    Qo, _, _ = oracle.collide(f, d, N, Nbar, Nt, 8.0)
    _assert_parity(Qg, Qo, f"d={d} N={N} Nbar={Nbar} Nt={Nt}")


@pytest.mark.parametrize("seed", range(8))
def test_parity_fuzz(seed):
    rng = np.random.default_rng(50 + seed)
    d = 2 if seed % 2 == 0 else 3
    N = int(rng.choice([8, 16, 32])) if d == 2 else int(rng.choice([8, 16]))
    Ntmax = (N - 1) // 2
    Nt = int(rng.integers(1, Ntmax + 1))
    Nbar = int(rng.integers(1, Nt + 1))
    L = float(rng.uniform(1.0, 10.0))
    cells = int(rng.integers(1, 4))
    f = rng.uniform(0.0, 1.0, size=(cells, N ** d))
    p = _plan(d, N, Nbar, Ntilde=Nt, L=L)
    Qg = _gpu(p, f)
    Qo, _, _ = oracle.collide(f, d, N, Nbar, Nt, L)
    for c in range(cells):
        _assert_parity(Qg[c], Qo[c], f"fuzz seed={seed} cell={c}")


# ---------------------------------------------------------------- parity, BASELINE sizes (sampled)
@pytest.mark.parametrize("name", ["c4", "c3"])
def test_parity_full_grid_3d_and_c3(name):
    """c4 (32^3) and c3 (256^2) on every node against the full direct oracle
    (3.4e9 / 8.1e9 pair evaluations on the host cores: seconds), default path."""
    cfg = dvm_inputs.CONFIGS[name]
    f = dvm_inputs.make(name)
    p = _plan(cfg.d, cfg.N, cfg.Nbar)
    Qg = _gpu(p, f)[0]
    Qo, _, _ = oracle.collide(f, cfg.d, cfg.N, cfg.Nbar, p.Ntilde, cfg.L)
    _assert_parity(Qg, Qo[0], f"{name} full grid")


@pytest.mark.parametrize("name,npts", [("c3", 1500), ("c4", 3000)])
def test_parity_sampled_single_grid(name, npts):
    cfg = dvm_inputs.CONFIGS[name]
    f = dvm_inputs.make(name)
    p = _plan(cfg.d, cfg.N, cfg.Nbar)
    Qg = _gpu(p, f)[0]
    pts = _sample_points(f[0], cfg.d, cfg.N, npts, 7)
    Qo, G, _ = oracle.collide(f, cfg.d, cfg.N, cfg.Nbar, p.Ntilde, cfg.L, points=pts)
    _assert_parity(Qg[pts], Qo[0], name)
    # invariants at full size: exact mass conservation
    assert abs(Qg.sum()) <= 1e-12 * np.abs(Qg).sum()


def _c5_points(f_cell, seed):
    """the 27 nodes around the argmax of f plus 101 seeded uniform
    nodes (distinct; topped up to 128 when the uniform draw repeats one)."""
    pts = list(_sample_points(f_cell, 3, 64, 101, seed))
    rng = np.random.default_rng(10_000 + seed)
    have = set(pts)
    while len(pts) < 128:
        x = int(rng.integers(0, 64 ** 3))
        if x not in have:
            have.add(x)
            pts.append(x)
    return np.array(sorted(pts[:128]), dtype=np.int64)


def test_parity_c5_all_cells_and_one_full_cell():
    """c5 exactly as bench.py launches it (512 cells, one batched call through
    the C ABI, k_fg2 with direction chunks), against the direct oracle:
    128 nodes in EVERY one of the 512 cells (27 around argmax f + 101 seeded;
    1.05e11 pair evaluations) and all 64^3 nodes of the last cell (4.2e11).
    Scale per cell: max |Q_oracle| over that cell's compared nodes."""
    cfg = dvm_inputs.CONFIGS["c5"]
    f = dvm_inputs.make("c5")
    p = _plan(3, cfg.N, cfg.Nbar)
    Qg = _gpu(p, f)
    assert Qg.shape == (512, 64 ** 3)
    pts = np.stack([_c5_points(f[c], 100 + c) for c in range(512)])
    Qo, _, _ = oracle.collide(f, 3, cfg.N, cfg.Nbar, p.Ntilde, cfg.L, points=pts, diagnostics=False)
    worst = 0.0
    for c in range(512):
        worst = max(worst, _assert_parity(Qg[c][pts[c]], Qo[c], f"c5 cell {c}"))
    print(f"c5: 512 cells x 128 nodes, worst max|dQ|/max|Q_oracle| = {worst:.3e}")
    c = 511
    Qf, _, _ = oracle.collide(f[c], 3, cfg.N, cfg.Nbar, p.Ntilde, cfg.L, diagnostics=False)
    rel = _assert_parity(Qg[c], Qf[0], "c5 cell 511, all nodes")
    print(f"c5 cell 511, all 262144 nodes: max|dQ|/max|Q_oracle| = {rel:.3e}")
    # invariant at full size: exact mass conservation in every cell
    sums = Qg.sum(axis=1)
    assert np.all(np.abs(sums) <= 1e-12 * np.abs(Qg).sum(axis=1))


# ---------------------------------------------------------------- trajectories, invariants
def test_c2_euler_trajectory():
    """c2: 100 explicit Euler steps dt = 0.01 (reading R11); Q parity on the GPU
    state at steps 0, 50, 100; mass drift at round-off."""
    cfg = dvm_inputs.CONFIGS["c2"]
    p = _plan(2, 64, 8)
    f0 = dvm_inputs.make("c2")[0]
    f = torch.from_numpy(f0.copy()).cuda()
    moms = []
    for step in (0, 50, 100):
        if step:
            moms.append(p.euler(f, 0.01, 50))
        fs = f.cpu().numpy()
        assert fs.min() >= 0.0  # positivity
        Qg = _gpu(p, fs).reshape(-1)
        Qo, _, _ = oracle.collide(fs, 2, 64, 8, p.Ntilde, 8.0)
        _assert_parity(Qg, Qo[0], f"c2 step {step}")
    m = np.concatenate([moms[0], moms[1][1:]])
    assert m.shape == (101, 4)
    assert abs(m[-1, 0] - m[0, 0]) <= 1e-12 * m[0, 0]
    # and the moments agree with a host recomputation
    h = p.h
    v = (np.arange(64) - 32) * h
    fs = f.cpu().numpy().reshape(64, 64)
    np.testing.assert_allclose(m[-1, 0], h * h * fs.sum(), rtol=1e-13)
    np.testing.assert_allclose(m[-1, 3], h * h * ((v[:, None] ** 2 + v[None, :] ** 2) * fs).sum(), rtol=1e-12)


@pytest.mark.parametrize("d,N,Nbar", [(2, 64, 8), (3, 32, 4)])
def test_constant_field(d, N, Nbar):
    p = _plan(d, N, Nbar)
    p.set_path(2)  # the FFT-loss path
    Q1 = _gpu(p, np.ones(N ** d))
    # the loss is an FFT convolution: exact only up to rounding (reading R18) ...
    _, G1, _ = oracle.collide(np.ones(N ** d), d, N, Nbar, p.Ntilde, 8.0, points=np.arange(4))
    assert np.abs(Q1).max() <= 1e-13 * G1.max()
    # ... while the v1 orbit sweeps sum small exact integers: Q = 0 exactly
    p.set_path(1)
    assert np.all(_gpu(p, np.ones(N ** d)) == 0.0)
    p.set_path(0)
    Qc = _gpu(p, np.full(N ** d, 0.3))
    _, G, _ = oracle.collide(np.full(N ** d, 0.3), d, N, Nbar, p.Ntilde, 8.0, points=np.arange(4))
    assert np.abs(Qc).max() <= 1e-13 * G.max()


@pytest.mark.parametrize("name", ["c1", "c3", "c4"])
def test_collide_graph_replay(name):
    """Repeated dvm_collide_batched calls with the same buffers replay one captured
    CUDA graph (include/dvm.h): the same bits as direct launches, f read at
    replay time, and plan settings / workspace growth invalidate the graph."""
    cfg = dvm_inputs.CONFIGS[name]
    f0 = dvm_inputs.make(name)
    p = _plan(cfg.d, cfg.N, cfg.Nbar)
    ref = _plan(cfg.d, cfg.N, cfg.Nbar)
    ref.set_graphs(False)
    f = torch.from_numpy(f0.copy()).cuda()
    q = torch.empty_like(f)
    want = _gpu(ref, f0)
    l0 = p.launches()
    for _ in range(4):  # direct, captured, replayed, replayed
        p.collide(f, q)
        torch.cuda.synchronize()
        assert np.array_equal(q.cpu().numpy(), want)
    assert p.launches() - l0 >= 4  # replays still count their kernels
    # new data in the same buffer: the replay reads it
    f1 = f0 * (1.0 + 0.05 * np.cos(np.arange(f0.size)).reshape(f0.shape))
    f.copy_(torch.from_numpy(f1))
    p.collide(f, q)
    torch.cuda.synchronize()
    assert np.array_equal(q.cpu().numpy(), _gpu(ref, f1))
    # a larger batch grows the workspace; the old key is captured afresh afterwards
    f2 = torch.from_numpy(np.concatenate([f1, f0], axis=0)).cuda()
    p.collide(f2)
    for _ in range(3):
        p.collide(f, q)
        torch.cuda.synchronize()
        assert np.array_equal(q.cpu().numpy(), _gpu(ref, f1))
    # a setting change invalidates the graph (path 1 = v1 sweeps: equal to rounding)
    p.set_path(1)
    ref.set_path(1)
    for _ in range(3):
        p.collide(f, q)
        torch.cuda.synchronize()
    assert np.array_equal(q.cpu().numpy(), _gpu(ref, f1))


def test_collide_inside_user_graph_capture():
    """A caller capturing the plan's stream into its own CUDA graph gets plain
    launches (the collide graph cache steps aside): replaying the caller's graph
    gives the direct result."""
    cfg = dvm_inputs.CONFIGS["c1"]
    f0 = dvm_inputs.make("c1")
    p = _plan(cfg.d, cfg.N, cfg.Nbar)
    f = torch.from_numpy(f0.copy()).cuda()
    q = torch.empty_like(f)
    want = _gpu(p, f0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        p.collide(f, q)  # warm on this stream (workspace, tables)
        p.collide(f, q)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        p.collide(f, q)
        p.collide(f, q)
    q.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(q.cpu().numpy(), want)


def test_determinism_bitwise():
    cfg = dvm_inputs.CONFIGS["c4"]
    f = dvm_inputs.make("c4")
    p = _plan(3, cfg.N, cfg.Nbar)
    assert np.array_equal(_gpu(p, f), _gpu(p, f))
    p2 = _plan(3, cfg.N, cfg.Nbar)
    assert np.array_equal(_gpu(p, f), _gpu(p2, f))


@pytest.mark.parametrize("name,world", [("c3", 4), ("c4", 3), ("c1", 8)])
def test_direction_shards_sum_to_full(name, world):
    """Sequentially on one GPU: the sum of the shard partials equals the full
    evaluation (the multi-GPU all-reduce adds exactly these partials)."""
    cfg = dvm_inputs.CONFIGS[name]
    f = dvm_inputs.make(name)
    full = _gpu(_plan(cfg.d, cfg.N, cfg.Nbar), f)
    acc = np.zeros_like(full)
    seen = np.zeros(_plan(cfg.d, cfg.N, cfg.Nbar).A, dtype=int)
    for r in range(world):
        p = _plan(cfg.d, cfg.N, cfg.Nbar, shard_rank=r, shard_world=world)
        seen += p.directions()[3]
        acc += _gpu(p, f)
    assert np.all(seen == 1)
    np.testing.assert_allclose(acc, full, rtol=0, atol=1e-13 * np.abs(full).max())


def test_host_entry_point_matches_device():
    cfg = dvm_inputs.CONFIGS["c4"]
    f = dvm_inputs.make("c4")
    p = _plan(3, cfg.N, cfg.Nbar)
    assert np.array_equal(p.collide_host(f), _gpu(p, f))


@pytest.mark.parametrize("d,N,Nbar,cells", [(2, 16, 4, 300), (3, 32, 2, 258)])
def test_host_entry_point_pipelined_batches(d, N, Nbar, cells):
    """dvm_collide_batched_host with >= 256 cells runs 4 pipelined chunks (copy
    streams + the plan's stream): equal to the device-resident batch (2D: bitwise,
    cells are independent; 3D: to rounding, the direction chunking may differ),
    also with a host cell stride > N^d."""
    rng = np.random.default_rng(d * 100 + cells)
    f = rng.uniform(0.0, 1.0, size=(cells, N ** d))
    p = _plan(d, N, Nbar)
    qd = _gpu(p, f)
    qh = p.collide_host(f)
    if d == 2:
        assert np.array_equal(qh, qd)
    else:
        np.testing.assert_allclose(qh, qd, rtol=0, atol=1e-13 * np.abs(qd).max())
    # strided host cells
    import ctypes
    from paper_1201_3986_b200 import dvm as _d
    stride = N ** d + 5
    fs = np.zeros((cells, stride))
    fs[:, :N ** d] = f
    qs = np.full((cells, stride), 7.0)
    st = _d.load().dvm_collide_batched_host(p._h, ctypes.c_void_p(fs.ctypes.data), ctypes.c_void_p(qs.ctypes.data),
                                           cells, stride)
    assert st == 0
    np.testing.assert_allclose(qs[:, :N ** d], qd, rtol=0, atol=1e-13 * np.abs(qd).max())
    assert np.all(qs[:, N ** d:] == 7.0)


def test_batched_edge_cases():
    from paper_1201_3986_b200 import DvmError
    p = _plan(2, 16, 4)
    f = np.random.default_rng(1).uniform(0, 1, size=(5, 256))
    Qb = _gpu(p, f)
    for c in range(5):
        # the FFT loss transforms cells in pairs: a cell's rounding depends on its
        # batch partner, so batched == single holds to rounding, not bitwise
        q1 = _gpu(p, f[c]).reshape(-1)
        np.testing.assert_allclose(Qb[c], q1, rtol=0, atol=1e-13 * np.abs(q1).max())
    assert np.array_equal(Qb, _gpu(p, f))  # same call, same bits
    ft = torch.from_numpy(f).cuda()
    with pytest.raises(DvmError) as ei:
        p.collide(ft, out=ft)
    assert ei.value.name == "DVM_E_ALIAS"
    # zero cells is a no-op
    import ctypes
    from paper_1201_3986_b200 import dvm as _d
    st = _d.load().dvm_collide_batched(p._h, ctypes.c_void_p(ft.data_ptr()),
                                       ctypes.c_void_p(ft.data_ptr() + 8 * ft.numel()), 0, 0)
    assert st == 0
    # strided cells (cell_stride > N^d)
    big = torch.zeros((5, 300), dtype=torch.float64, device="cuda")
    big[:, :256] = ft
    out = torch.full_like(big, 7.0)
    st = _d.load().dvm_collide_batched(p._h, ctypes.c_void_p(big.data_ptr()), ctypes.c_void_p(out.data_ptr()), 5, 300)
    assert st == 0
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    np.testing.assert_allclose(o[:, :256], Qb, rtol=0, atol=1e-13 * np.abs(Qb).max())
    assert np.all(o[:, 256:] == 7.0)


@pytest.mark.parametrize("d,N,Nbar,Nt,cells", [(3, 32, 4, 7, 1), (3, 64, 8, 14, 3), (3, 32, 3, 5, 40),
                                               (3, 64, 2, 5, 1), (3, 64, 1, 4, 2), (3, 32, 4, 7, 3)])
def test_gain3d_path_matches_orbit_path(d, N, Nbar, Nt, cells):
    """The 3D frame-plane gain kernel + FFT loss and the v1 orbit sweeps evaluate
    the same operator (different summation orders): agreement to rounding."""
    f = np.random.default_rng(N + cells).uniform(0.0, 1.0, size=(cells, N ** d))
    p = _plan(d, N, Nbar, Ntilde=Nt)
    q2 = _gpu(p, f)
    p.set_path(1)
    q1 = _gpu(p, f)
    np.testing.assert_allclose(q2, q1, rtol=0, atol=1e-13 * np.abs(q1).max())
    if N <= 64:
        pts = np.arange(0, N ** d, N ** d // 97)
        Qo, _, _ = oracle.collide(f[0], d, N, Nbar, Nt, 8.0, points=pts)
        _assert_parity(q2[0][pts], Qo[0], f"gain3d path N={N}")


def test_gain3d_ragged_batches():
    """Odd cell counts (the last cell pair is padded) and direction chunking for
    small batches: every cell equals its single-cell evaluation to rounding and
    matches the oracle on sampled nodes."""
    N, Nbar, Nt = 32, 2, 5
    f = np.random.default_rng(11).uniform(0.0, 1.0, size=(5, N ** 3))
    p = _plan(3, N, Nbar, Ntilde=Nt)
    for cells in (1, 3, 5):
        qb = _gpu(p, f[:cells])
        for c in range(cells):
            q1 = _gpu(p, f[c]).reshape(-1)
            np.testing.assert_allclose(qb[c], q1, rtol=0, atol=1e-13 * np.abs(q1).max())
    pts = np.arange(0, N ** 3, 331)
    Qo, _, _ = oracle.collide(f[4], 3, N, Nbar, Nt, 8.0, points=pts)
    _assert_parity(qb[4][pts], Qo[0], "gain3d ragged batch")


@pytest.mark.parametrize("Nbar,Nt,cells", [(2, 5, 1), (1, 4, 2), (2, 14, 3), (3, 7, 5), (8, 14, 2)])
def test_fgain3d_path_matches_frame_path(Nbar, Nt, cells):
    """3D N = 64 gain by per-direction FFT filtering (dvm_set_path(4)) against the
    frame-plane kernel (path 2) and the oracle on sampled nodes; ragged pair
    counts and direction chunking (few cells) included."""
    N = 64
    f = np.random.default_rng(Nbar * 10 + cells).uniform(0.0, 1.0, size=(cells, N ** 3))
    p = _plan(3, N, Nbar, Ntilde=Nt)
    p.set_path(2)
    q2 = _gpu(p, f)
    p.set_path(4)
    q4 = _gpu(p, f)
    np.testing.assert_allclose(q4, q2, rtol=0, atol=1e-12 * np.abs(q2).max())
    assert np.array_equal(q4, _gpu(p, f))  # repeated call: bitwise
    pts = np.arange(0, N ** 3, N ** 3 // 61)
    Qo, _, _ = oracle.collide(f[cells - 1], 3, N, Nbar, Nt, 8.0, points=pts)
    _assert_parity(q4[cells - 1][pts], Qo[0], f"fgain3d N̄={Nbar} Ñ={Nt}")


@pytest.mark.parametrize("world", [2, 4, 8])
def test_parity_c5_strong_scaling_rank_blocks(world):
    """c5 as one rank of bench.py's strong-scaling run launches it (BASELINE c5:
    512 cells sharded across 2/4/8 GPUs; parallel.cell_range gives the last rank
    512/world contiguous cells, one batched call, so another direction-chunk
    count than the 512-cell launch).  Six cells of the block (first, last and
    four seeded) on 128 nodes each (as in the 512-cell test) against the oracle."""
    from paper_1201_3986_b200.parallel import cell_range
    cfg = dvm_inputs.CONFIGS["c5"]
    first, count = cell_range(512, world - 1, world)
    f = dvm_inputs.make("c5")[first:first + count]
    p = _plan(3, cfg.N, cfg.Nbar)
    Qg = _gpu(p, f)
    rng = np.random.default_rng(world)
    cells = sorted({0, count - 1, *(int(c) for c in rng.choice(count, size=4, replace=False))})
    pts = np.stack([_c5_points(f[c], 300 + c) for c in cells])
    Qo, _, _ = oracle.collide(f[cells], 3, cfg.N, cfg.Nbar, p.Ntilde, cfg.L, points=pts, diagnostics=False)
    worst = max(_assert_parity(Qg[c][pts[i]], Qo[i], f"c5 world {world} block cell {first + c}")
                for i, c in enumerate(cells))
    print(f"c5 rank {world - 1}/{world} ({count} cells): worst {worst:.3e}")
    sums = Qg.sum(axis=1)
    assert np.all(np.abs(sums) <= 1e-12 * np.abs(Qg).sum(axis=1))


def test_fgain3d_chunked_rounds_match_frame_path():
    """A batch with more pairs than groups and several direction chunks per pair
    (20 cells = 10 pairs on 9 groups: the chunk rule picks more than one chunk
    and the groups take several rounds) equals the frame-plane path; c5 inputs."""
    f = dvm_inputs.make("c5", cells=20)
    p = _plan(3, 64, 8)
    p.set_path(2)
    q2 = _gpu(p, f)
    p.set_path(4)
    q4 = _gpu(p, f)
    np.testing.assert_allclose(q4, q2, rtol=0, atol=1e-12 * np.abs(q2).max())
    assert np.array_equal(q4, _gpu(p, f))


def test_fgain3d_large_ntilde_falls_back():
    """Ñ > 16 exceeds the 3D kernels' tap tables (2 M_e <= 32): the plan still
    builds and both auto mode and dvm_set_path(4) evaluate by the orbit sweeps
    (bitwise the v1 path, parity with the oracle)."""
    N, Nbar, Nt = 64, 2, 20
    f = np.random.default_rng(7).uniform(0.0, 1.0, size=(2, N ** 3))
    p = _plan(3, N, Nbar, Ntilde=Nt)
    q = _gpu(p, f)
    pts = np.arange(0, N ** 3, N ** 3 // 41)
    Qo, _, _ = oracle.collide(f[1], 3, N, Nbar, Nt, 8.0, points=pts)
    _assert_parity(q[1][pts], Qo[0], "auto, Ñ=20")
    p.set_path(4)
    q4 = _gpu(p, f)
    p.set_path(1)
    assert np.array_equal(q4, _gpu(p, f)) and np.array_equal(q, q4)


def test_fgain3d_direction_shards_sum_to_full():
    """Direction-sharded plans (each rank a subset of lines) on the FFT gain path
    sum to the full operator."""
    N, Nbar, Nt = 64, 3, 7
    f = np.random.default_rng(3).uniform(0.0, 1.0, size=(2, N ** 3))
    p = _plan(3, N, Nbar, Ntilde=Nt)
    p.set_path(4)
    full = _gpu(p, f)
    acc = np.zeros_like(full)
    for r in range(3):
        ps = _plan(3, N, Nbar, Ntilde=Nt, shard_rank=r, shard_world=3)
        ps.set_path(4)
        acc += _gpu(ps, f)
    np.testing.assert_allclose(acc, full, rtol=0, atol=1e-12 * np.abs(full).max())


@pytest.mark.parametrize("N,Nbar,Nt,cells", [(16, 4, 4, 1), (64, 8, 14, 3), (256, 16, 57, 1), (128, 5, 20, 2),
                                            (32, 7, 7, 5)])
def test_pair2d_path_matches_orbit_path(N, Nbar, Nt, cells):
    """The 2D direction-pair kernels + FFT loss and the v1 orbit sweeps evaluate
    the same operator (different summation orders): agreement to rounding, and
    oracle parity on sampled nodes."""
    f = np.random.default_rng(N + cells).uniform(0.0, 1.0, size=(cells, N ** 2))
    p = _plan(2, N, Nbar, Ntilde=Nt)
    p.set_path(2)  # the pair kernels also below the auto threshold
    q2 = _gpu(p, f)
    p.set_path(1)
    q1 = _gpu(p, f)
    np.testing.assert_allclose(q2, q1, rtol=0, atol=1e-13 * np.abs(q1).max())
    pts = np.arange(0, N ** 2, max(1, N ** 2 // 157))
    Qo, _, _ = oracle.collide(f[-1], 2, N, Nbar, Nt, 8.0, points=pts)
    _assert_parity(q2[-1][pts], Qo[0], f"pair2d N={N}")


@pytest.mark.parametrize("N,Nbar,Nt,cells", [(16, 4, 4, 1), (16, 2, 7, 3), (32, 5, 7, 2), (64, 8, 14, 3), (64, 3, 20, 1)])
def test_small2d_path_matches_orbit_path(N, Nbar, Nt, cells):
    """2D small grids (dvm_set_path 5, auto for N <= 64): gain and loss per pair
    unit from shared memory (loss as f [a (Box − W_B) + a (Box − W_A)]) against
    the v1 orbit sweeps and the oracle; ragged batches, M up to 20."""
    f = np.random.default_rng(3 * N + cells).uniform(0.0, 1.0, size=(cells, N ** 2))
    p = _plan(2, N, Nbar, Ntilde=Nt)
    p.set_path(5)
    q5 = _gpu(p, f)
    assert np.array_equal(q5, _gpu(p, f))
    p.set_path(1)
    q1 = _gpu(p, f)
    np.testing.assert_allclose(q5, q1, rtol=0, atol=1e-13 * np.abs(q1).max())
    Qo, _, _ = oracle.collide(f[-1], 2, N, Nbar, Nt, 8.0)
    _assert_parity(q5[-1], Qo, f"small2d N={N}")
    assert abs(q5[-1].sum()) <= 1e-13 * np.abs(q5[-1]).sum()  # mass, per pair exactly


# ---------------------------------------------------------------- time steppers (CUDA graphs)
@pytest.mark.parametrize("d,N,Nbar,Nt,path", [(2, 64, 8, 14, 0), (2, 64, 8, 14, 2), (3, 32, 2, 5, 0)])
def test_stepper_graph_replay_is_bitwise(d, N, Nbar, Nt, path):
    """Steps 2..n replay one captured CUDA graph: identical bits and moments to
    direct launches, for Euler and RK2 (v1, pair2d + FFT loss, gain3d)."""
    f0 = dvm_inputs.two_bumps(d, N, 8.0, 1.0, 0.01, 4).reshape(-1)
    p = _plan(d, N, Nbar, Ntilde=Nt)
    p.set_path(path)
    for method in ("euler", "rk2"):
        out = []
        for graphs in (True, False):
            p.set_graphs(graphs)
            f = torch.from_numpy(f0.copy()).cuda()
            m = getattr(p, method)(f, 0.01, 6)
            out.append((f.cpu().numpy(), m))
        assert np.array_equal(out[0][0], out[1][0]), method
        assert np.array_equal(out[0][1], out[1][1]), method
    p.set_graphs(True)


def test_rk2_matches_oracle_heun():
    """TVD-RK2 (Heun) on c1 for 3 steps against the same
    scheme evaluated with the CPU oracle."""
    cfg = dvm_inputs.CONFIGS["c1"]
    f0 = dvm_inputs.make("c1")[0]
    p = _plan(2, cfg.N, cfg.Nbar)
    dt = 0.05
    f = torch.from_numpy(f0.copy()).cuda()
    m = p.rk2(f, dt, 3)
    fo = f0.copy()
    for _ in range(3):
        q0 = oracle.collide(fo, 2, cfg.N, cfg.Nbar, p.Ntilde, cfg.L)[0].reshape(-1)
        f1 = fo + dt * q0
        q1 = oracle.collide(f1, 2, cfg.N, cfg.Nbar, p.Ntilde, cfg.L)[0].reshape(-1)
        fo = 0.5 * (fo + (f1 + dt * q1))
    fg = f.cpu().numpy()
    assert np.abs(fg - fo).max() <= 1e-13 * np.abs(fo).max()
    # mass exactly conserved by every stage
    assert np.all(np.abs(m[:, 0] - m[0, 0]) <= 1e-13 * m[0, 0])


# ---------------------------------------------------------------- space-dependent N̄
@pytest.mark.parametrize("d,N,levels,nb", [
    (3, 32, [1, 2, 4], [4, 1, 2, 4, 1, 2, 2]),        # buckets of 2, 3, 2 cells (odd: 3D pairs padded)
    (3, 64, [2, 8], [8, 2, 8, 8, 2]),                 # the c5 grid, k_fg2 on odd buckets
    (2, 64, [2, 5, 8], [[8, 2], [5, 8], [8, 8], [2, 5], [8, 8]]),  # 2D-shaped [cells, N, N] input
])
def test_adaptive_nbar_levels_abi(d, N, levels, nb):
    """dvm_collide_batched_levels (space-dependent N̄): every
    cell equals its single-level evaluation (to rounding) and the oracle at its
    own N̄ on sampled nodes; ragged (odd) buckets and a [cells, N, N] input."""
    from paper_1201_3986_b200 import DvmError
    from paper_1201_3986_b200.adaptive import AdaptiveNbar
    nb = np.asarray(nb).reshape(-1)
    ad = AdaptiveNbar(d, N, levels)
    cells = nb.size
    f = np.stack([dvm_inputs.two_bumps(d, N, 8.0, 0.5 + 0.3 * c, 0.02, c).reshape(-1) for c in range(cells)])
    shape = (cells,) + (N,) * d if d == 2 else (cells, N ** d)
    ft = torch.from_numpy(f.reshape(shape)).cuda()
    q = ad.collide(ft, nb).cpu().numpy().reshape(cells, -1)
    qd = ad.collide(ft, torch.from_numpy(nb).cuda()).cpu().numpy().reshape(cells, -1)  # device levels
    assert np.array_equal(q, qd)
    pts = np.arange(0, N ** d, max(1, N ** d // 61))
    for c in range(cells):
        q1 = ad.plans[int(nb[c])].collide(ft.reshape(cells, -1)[c].contiguous()).cpu().numpy()
        np.testing.assert_allclose(q[c], q1, rtol=0, atol=1e-13 * np.abs(q1).max())
        Qo, _, _ = oracle.collide(f[c], d, N, int(nb[c]), ad.Ntilde, 8.0, points=pts, diagnostics=False)
        _assert_parity(q[c][pts], Qo[0], f"levels cell {c} N̄={nb[c]}")
    bad = nb.copy()
    bad[1] = 3 if 3 not in levels else 99
    with pytest.raises((DvmError, ValueError)):
        ad.collide(ft, bad)
    with pytest.raises(DvmError) as ei:
        ad.collide(ft, torch.from_numpy(bad).cuda())
    assert ei.value.name == "DVM_E_SHAPE"


def test_adaptive_reference_policy():
    from paper_1201_3986_b200.adaptive import equilibrium_levels
    # the reference policy: a Maxwellian cell gets the lowest level
    m = dvm_inputs.make("c5", cells=2)
    lv, delta = equilibrium_levels(torch.from_numpy(m).cuda(), 3, 64, 8.0, [2, 8], [0.05])
    assert lv.shape == (2,) and np.all(delta < 0.05) and np.all(lv == 2)


def test_adaptive_levels_with_transport():
    """Space-dependent N̄ inside a transport + collision splitting (PAPER.md:
    907-911; tools/inhomogeneous.py at a small size): levels re-chosen every step,
    bucket sizes changing from step to step; mass conserved to rounding, every
    step's Q per cell equal to that cell's single-level evaluation, and the
    adaptive trajectory close to the uniform-N̄ one."""
    from paper_1201_3986_b200.adaptive import AdaptiveNbar, equilibrium_levels
    N, X, levels = 32, 16, [2, 7]
    h, dx = 16.0 / N, 1.0 / X
    v = (torch.arange(N, dtype=torch.float64) - N // 2) * h
    VX, VY = torch.meshgrid(v, v, indexing="ij")
    dt = 0.5 * dx / float(v.abs().max())
    def mx(rho, ux, T):
        return (rho / (2 * np.pi * T) * torch.exp(-((VX - ux) ** 2 + VY ** 2) / (2 * T))).reshape(-1)
    f0 = torch.stack([0.5 * (mx(1.0, 1.2, 0.5) + mx(1.0, -1.2, 0.5)) if 0.3 < (i + 0.5) * dx < 0.7
                      else mx(1.0 + 0.3 * np.sin(2 * np.pi * (i + 0.5) * dx), 0.0, 1.0) for i in range(X)]).cuda()
    vx = VX.reshape(-1).cuda()
    pos = (vx > 0).double()
    def transport(f):
        return f - dt / dx * vx * (pos * (f - torch.roll(f, 1, 0)) + (1 - pos) * (torch.roll(f, -1, 0) - f))
    ad = AdaptiveNbar(2, N, levels)
    single = {nb: _plan(2, N, nb, Ntilde=ad.Ntilde) for nb in levels}
    full = single[levels[-1]]
    fa, fu = f0.clone(), f0.clone()
    m0 = float(fa.sum())
    seen = set()
    for _ in range(6):
        fa, fu = transport(fa), transport(fu)
        nb, _ = equilibrium_levels(fa, 2, N, 8.0, levels, [0.02])
        seen.add(int((nb == levels[0]).sum()))
        qa = ad.collide(fa, nb)
        qs = torch.stack([single[int(nb[c])].collide(fa[c].contiguous()) for c in range(X)])
        torch.cuda.synchronize()
        np.testing.assert_allclose(qa.cpu().numpy(), qs.cpu().numpy(), rtol=0,
                                   atol=1e-13 * float(qs.abs().max()))
        fa += dt * qa
        fu += dt * full.collide(fu)
    assert abs(float(fa.sum()) - m0) <= 1e-12 * m0
    assert 0 < min(seen) < X  # both levels in use
    assert float((fa - fu).abs().sum() / fu.abs().sum()) < 1e-3


# ---------------------------------------------------------------- spectral reference path (dvm_set_path(3))
@pytest.mark.parametrize("d,N,Nbar,Nt,cells", [(2, 16, 4, 4, 1), (2, 64, 8, 14, 2), (3, 32, 2, 5, 1), (3, 32, 4, 7, 2)])
def test_spectral_path_matches_oracle(d, N, Nbar, Nt, cells):
    """The paper's per-direction spectral evaluation (S_e + i T_e from one inverse
    transform of f̂ (ŝ_e + i t̂_e)) against the oracle and the default path."""
    f = np.stack([dvm_inputs.two_bumps(d, N, 8.0, 1.0 + 0.2 * c, 0.01, c).reshape(-1) for c in range(cells)])
    p = _plan(d, N, Nbar, Ntilde=Nt)
    q0 = _gpu(p, f)
    p.set_path(3)
    q3 = _gpu(p, f)
    np.testing.assert_allclose(q3, q0, rtol=0, atol=1e-12 * np.abs(q0).max())
    pts = np.arange(0, N ** d, max(1, N ** d // 211))
    for c in range(cells):
        Qo, _, _ = oracle.collide(f[c], d, N, Nbar, Nt, 8.0, points=pts)
        _assert_parity(q3[c][pts], Qo[0], f"spectral d={d} N={N} cell {c}")


def test_triple_agreement_c1():
    """GPU (every path) == direct-sum oracle == the paper's pseudo-spectral route
    (dense β(K,L), oracle/cross.py) on c1."""
    from oracle import cross
    cfg = dvm_inputs.CONFIGS["c1"]
    f = dvm_inputs.make("c1")[0]
    p = _plan(2, cfg.N, cfg.Nbar)
    Qo = oracle.collide(f, 2, cfg.N, cfg.Nbar, p.Ntilde, cfg.L)[0].reshape(-1)
    Qb, _ = cross.dense_beta_Q(f, 2, cfg.N, cfg.Nbar, p.Ntilde, cfg.L)
    _assert_parity(Qb, Qo, "dense beta vs oracle")
    for path in (0, 1, 2, 3):
        p.set_path(path)
        _assert_parity(_gpu(p, f).reshape(-1), Qb, f"path {path} vs dense beta")


# ---------------------------------------------------------------- general weights a(k) b(l) (dvm_set_weights)
@pytest.mark.parametrize("d,N,Nbar,Nt,cells", [(2, 16, 4, 4, 1), (2, 64, 8, 14, 3), (3, 16, 2, 3, 2), (3, 32, 2, 5, 1)])
def test_weighted_spectral_matches_oracle(d, N, Nbar, Nt, cells):
    """Γ̃_{k,l} = a(k) b(l) with seeded even tables (eq:decoup):
    the spectral path against the weighted oracle; mass conserved."""
    a = dvm_inputs.even_weights(d, Nt, 10 + N)
    b = dvm_inputs.even_weights(d, Nt, 20 + N, 0.2, 1.0)
    f = np.stack([dvm_inputs.two_bumps(d, N, 8.0, 1.0 + 0.2 * c, 0.01, c).reshape(-1) for c in range(cells)])
    p = _plan(d, N, Nbar, Ntilde=Nt)
    p.set_weights(a, b)
    q = _gpu(p, f)
    pts = None if N ** d <= 4096 else np.arange(0, N ** d, N ** d // 197)
    for c in range(cells):
        Qo, Go, _ = oracle.collide(f[c], d, N, Nbar, Nt, 8.0, points=pts, a_box=a, b_box=b)
        qc = q[c] if pts is None else q[c][pts]
        _assert_parity(qc, Qo[0], f"weighted d={d} N={N} cell {c}")
        assert abs(q[c].sum()) <= 1e-12 * np.abs(q[c]).sum()
    # the weights enter: the built-in operator differs
    p.set_weights(None, None)
    q0 = _gpu(p, f)
    assert np.abs(q0 - q).max() > 1e-3 * np.abs(q).max()


@pytest.mark.parametrize("d,N,Nbar,Nt", [(2, 64, 8, 14), (3, 32, 4, 7)])
def test_weighted_builtin_tables_equal_default_path(d, N, Nbar, Nt):
    """The built-in a(k) = h^{d+1}|k|/gcd(k), b = 1 passed as tables reproduces
    the default path (to rounding): the weighted λ and filters index the box right."""
    p = _plan(d, N, Nbar, Ntilde=Nt)
    h = p.h
    a = np.zeros((2 * Nt + 1,) * d)
    for k in itertools.product(range(-Nt, Nt + 1), repeat=d):
        if any(k):
            g = 0
            for c in k:
                g = math.gcd(g, abs(c))
            a[tuple(c + Nt for c in k)] = h ** (d + 1) * math.sqrt(sum(c * c for c in k)) / g
    f = np.stack([dvm_inputs.two_bumps(d, N, 8.0, 1.3, 0.01, 5).reshape(-1)] * 2)
    q0 = _gpu(p, f)
    p.set_weights(a, np.ones_like(a))
    q1 = _gpu(p, f)
    np.testing.assert_allclose(q1, q0, rtol=0, atol=1e-12 * np.abs(q0).max())
    p.set_weights(a, None)  # None keeps b = 1
    np.testing.assert_allclose(_gpu(p, f), q0, rtol=0, atol=1e-12 * np.abs(q0).max())


def test_weighted_errors_and_reset():
    from paper_1201_3986_b200 import DvmError
    p = _plan(2, 16, 4, Ntilde=4)
    f = dvm_inputs.make("c1")[0]
    q_default = _gpu(p, f)
    odd = np.arange(81, dtype=np.float64).reshape(9, 9)
    with pytest.raises(DvmError):
        p.set_weights(odd, None)
    np.testing.assert_array_equal(_gpu(p, f), q_default)  # rejected tables leave the plan unchanged
    p.set_weights(dvm_inputs.even_weights(2, 4, 1), None)
    for path in (1, 2, 4):
        p.set_path(path)
        with pytest.raises(DvmError):
            _gpu(p, f)
    p.set_path(3)
    _gpu(p, f)
    p.set_weights(None, None)
    p.set_path(0)
    np.testing.assert_array_equal(_gpu(p, f), q_default)


# ---------------------------------------------------------------- BKW accuracy workload
def test_bkw_rk2_matches_oracle_heun():
    """The BKW workload's stepping (dvm_rk2 on the operator with the Carleman
    weights a(k) = h^2/(π gcd k), reading R24) on a c1-sized grid (N = 16, box
    T = 5.5, N̄ = Ñ = 3) equals the same TVD-RK2 (Heun) evaluated with the CPU
    oracle and the same weight table, for 3 steps."""
    from paper_1201_3986_b200 import bkw
    N, T, Nbar, dt, steps = 16, 5.5, 3, 0.01, 3
    p = bkw.make_plan(N, Nbar, T)
    a_box = bkw.carleman_weights(p.Ntilde, p.h)
    v2 = bkw.grid_v2(N, T)
    f0 = bkw.f_exact(0.0, v2).reshape(-1)
    f = torch.from_numpy(f0.copy()).cuda()
    p.rk2(f, dt, steps)
    fo = f0.copy()
    for _ in range(steps):
        q0 = oracle.collide(fo, 2, N, Nbar, p.Ntilde, T, a_box=a_box)[0].reshape(-1)
        f1 = fo + dt * q0
        q1 = oracle.collide(f1, 2, N, Nbar, p.Ntilde, T, a_box=a_box)[0].reshape(-1)
        fo = 0.5 * (fo + (f1 + dt * q1))
    assert np.abs(f.cpu().numpy() - fo).max() <= 1e-13 * np.abs(fo).max()


def test_bkw_carleman_weights_are_the_bkw_operator():
    """Reading R24: with a(k) = h^2/(π gcd k) the operator converges to the
    exact BKW time derivative (L1 residual of the best constant fit -> 0 with N,
    best constant -> ~1.08, the |x|,|y| <= Ñh truncation), while the printed
    h^3|k|/gcd k does not (a residual near 20 % at every N)."""
    from paper_1201_3986_b200 import bkw
    res = {}
    for weights in ("carleman", "printed"):
        for N in (16, 32, 64):
            T = bkw.PAPER_BOX[N]
            p = bkw.make_plan(N, _plan(2, N, 1, L=T).Ntilde, T, weights)
            v2 = bkw.grid_v2(N, T)
            q = p.collide(torch.from_numpy(bkw.f_exact(0.0, v2).reshape(-1)).cuda()).cpu().numpy()
            ft = bkw.dfdt_exact(0.0, v2).reshape(-1)
            c = float(np.dot(q, ft) / np.dot(q, q))
            res[weights, N] = (c, np.abs(c * q - ft).sum() / np.abs(ft).sum())
    assert res["carleman", 16][1] > res["carleman", 32][1] > res["carleman", 64][1]
    assert res["carleman", 64][1] < 0.02 and 1.0 < res["carleman", 64][0] < 1.15
    assert all(res["printed", N][1] > 0.15 for N in (16, 32, 64))


def test_bkw_e1_decreases_with_N():
    """Table 1's trend: with the physical operator (c = 1) the
    relative L1 error after one RK2 step of dt = 0.01 from the BKW datum
    decreases as the grid is refined (paper's boxes, all lines N̄ = Ñ)."""
    from paper_1201_3986_b200 import bkw
    errs = []
    for N in (16, 32, 64):
        Nt = _plan(2, N, 1, L=bkw.PAPER_BOX[N]).Ntilde
        errs.append(bkw.run(N, Nt)[0])
    assert errs[0] > errs[1] > errs[2] > 0, errs


# ---------------------------------------------------------------- 3D N = 32 direction-pair spectral gain (path 6)
@pytest.mark.parametrize("Nbar,Nt,cells,shard", [(4, 7, 1, None), (2, 5, 3, None), (4, 7, 1, (1, 3)), (1, 3, 2, None)])
def test_fg32_path_matches_oracle(Nbar, Nt, cells, shard):
    """dvm_set_path(6): T_a + i T_b = IFFT(f̂ (t̂_a + i t̂_b)) for direction pairs of
    one real cell (reading R23), taps for S_e, partials in chunk order: every
    node against the oracle (c4 geometry), odd direction counts (a lone last
    direction), several cells and a direction shard."""
    f = np.stack([dvm_inputs.two_bumps(3, 32, 8.0, 1.0 + 0.25 * c, 0.01, 40 + c).reshape(-1) for c in range(cells)])
    kw = {} if shard is None else {"shard_rank": shard[0], "shard_world": shard[1]}
    p = _plan(3, 32, Nbar, Ntilde=Nt, **kw)
    p.set_path(6)
    q6 = _gpu(p, f)
    assert np.array_equal(q6, _gpu(p, f))  # bitwise repeatable
    dirs = p.directions()[0][p.directions()[3].astype(bool)] if shard else None
    for c in range(cells):
        Qo, _, _ = oracle.collide(f[c], 3, 32, Nbar, Nt, 8.0, dirs=dirs, diagnostics=False)
        _assert_parity(q6[c], Qo[0], f"fg32 N̄={Nbar} Ñ={Nt} cell {c}")


# ---------------------------------------------------------------- 2D tile kernel (path 7, auto for N >= 128)
@pytest.mark.parametrize("N,Nbar,Nt,cells,shard", [(256, 16, 57, 1, None), (128, 10, 28, 2, None), (16, 4, 4, 3, None),
                                                   (64, 8, 14, 2, (1, 3)), (128, 5, 20, 1, (2, 4))])
def test_tile2d_path_matches_oracle(N, Nbar, Nt, cells, shard):
    """dvm_set_path(7): one CTA per 16 x 16 tile with a halo of Ñ in shared
    memory, every pair unit's windows per node, Q = −fΛ + G:
    against the oracle (sampled nodes, every node for small grids), the line-walk
    pair kernels (path 2), several cells and direction shards."""
    f = np.stack([dvm_inputs.two_bumps(2, N, 8.0, 0.8 + 0.3 * c, 0.01, 60 + c).reshape(-1) for c in range(cells)])
    kw = {} if shard is None else {"shard_rank": shard[0], "shard_world": shard[1]}
    p = _plan(2, N, Nbar, Ntilde=Nt, **kw)
    p.set_path(7)
    q7 = _gpu(p, f)
    assert np.array_equal(q7, _gpu(p, f))
    p.set_path(2)
    q2 = _gpu(p, f)
    np.testing.assert_allclose(q7, q2, rtol=0, atol=1e-13 * np.abs(q2).max())
    pts = None if N ** 2 <= 4096 else np.arange(0, N ** 2, N ** 2 // 211)
    dirs = p.directions()[0][p.directions()[3]] if shard else None
    for c in range(cells):
        Qo, _, _ = oracle.collide(f[c], 2, N, Nbar, Nt, 8.0, points=pts, dirs=dirs, diagnostics=False)
        qc = q7[c] if pts is None else q7[c][pts]
        _assert_parity(qc, Qo[0], f"tile2d N={N} cell {c}")


def test_tuning_switches():
    """dvm_set_tuning: unknown keys and bad values are rejected (plan unchanged);
    timing_dbg changes Q (it skips work) and 0 restores the bitwise result;
    max_groups / ring_slots / fg_chunks change only the schedule (same operator to rounding)."""
    from paper_1201_3986_b200 import DvmError
    f = dvm_inputs.make("c5", cells=4)
    p = _plan(3, 64, 8)
    q0 = _gpu(p, f)
    for key, val in (("no_such_key", 1), ("ring_slots", 9), ("g3_cl", 3), ("timing_dbg", 99), ("fg_chunks", -1)):
        with pytest.raises(DvmError) as ei:
            p.set_tuning(key, val)
        assert ei.value.name == "DVM_E_STATE"
    p.set_tuning("timing_dbg", 4)  # skip the taps: wrong by design
    assert not np.allclose(_gpu(p, f), q0)
    p.set_tuning("timing_dbg", 0)
    assert np.array_equal(_gpu(p, f), q0)
    p.set_tuning("max_groups", 1)
    p.set_tuning("ring_slots", 3)
    np.testing.assert_allclose(_gpu(p, f), q0, rtol=0, atol=1e-12 * np.abs(q0).max())
    p.set_tuning("max_groups", 0)
    p.set_tuning("fg_chunks", 5)  # 2 pairs x 5 direction chunks on the 9 groups
    np.testing.assert_allclose(_gpu(p, f), q0, rtol=0, atol=1e-12 * np.abs(q0).max())
