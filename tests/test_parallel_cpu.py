"""Multi-process (world_size 2, gloo, CPU) tests of the N>1 plumbing.

The direction-sharded reduction runs through paper_1201_3986_b200.parallel's
sharded_collide exactly as on the GPUs; only the per-rank compute step is the
oracle restricted to the rank's LPT share of the directions (the GPU kernel
cannot run here).  Cell sharding is checked for exact coverage.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import dvm_inputs
from oracle import oracle
from paper_1201_3986_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _points(name):
    cfg = dvm_inputs.CONFIGS[name]
    nodes = cfg.N ** cfg.d
    return None if nodes <= 4096 else np.arange(0, nodes, nodes // 997)


def _owners(name, world):
    """The shard sets: 2D whole pair units {e, e⊥} exactly as libdvm assigns
    them (parallel.owners_2d); 3D a stand-in LPT cost (libdvm's 3D cost needs the
    plan's perp rows; tests/test_gpu_parity.py checks that mirror on the GPU)."""
    cfg = dvm_inputs.CONFIGS[name]
    Nt = oracle.ntilde_rule(cfg.N, cfg.Nbar)
    dirs = oracle.directions(cfg.d, cfg.Nbar)
    M = Nt // np.abs(dirs).max(axis=1)
    if cfg.d == 2:
        return dirs, parallel.owners_2d(dirs, M, world)
    return dirs, parallel.lpt_assign(M + 1, world)


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = dvm_inputs.CONFIGS[name]
        f = dvm_inputs.make(name)
        Nt = oracle.ntilde_rule(cfg.N, cfg.Nbar)
        dirs, owner = _owners(name, world)
        mine = dirs[owner == rank]
        pts = _points(name)

        def partial(x):
            Qp, _, _ = oracle.collide(x, cfg.d, cfg.N, cfg.Nbar, Nt, cfg.L, points=pts, dirs=mine,
                                      nthreads=max(1, (os.cpu_count() or 2) // world), diagnostics=False)
            return torch.from_numpy(Qp)

        Q = parallel.sharded_collide(partial, f)
        # cell sharding: contiguous, disjoint, complete
        first, count = parallel.cell_range(13, rank, world)
        got = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(got, torch.tensor([first, count]))
        if rank == 0:
            q.put((Q.numpy(), [g.tolist() for g in got], len(mine)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c1", "c3", "c4"])
def test_direction_sharded_allreduce_gloo(name):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    Q, ranges, nmine = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = dvm_inputs.CONFIGS[name]
    Nt = oracle.ntilde_rule(cfg.N, cfg.Nbar)
    Qfull, _, _ = oracle.collide(dvm_inputs.make(name), cfg.d, cfg.N, cfg.Nbar, Nt, cfg.L, points=_points(name),
                                 diagnostics=False)
    np.testing.assert_allclose(Q, Qfull, rtol=0, atol=1e-13 * np.abs(Qfull).max())
    assert 0 < nmine < len(oracle.directions(cfg.d, cfg.Nbar))
    covered = sorted(c for f0, n in ranges for c in range(f0, f0 + n))
    assert covered == list(range(13))


@pytest.mark.parametrize("name,units", [("c1", 12), ("c2", 44), ("c3", 160)])
def test_2d_pair_units_never_split(name, units):
    """2D shards are whole pair units {e, e⊥} (no unit evaluated twice), every
    direction owned once, and the unit counts balanced (c3: <= ceil(160/G)+1)."""
    for world in (2, 4, 8):
        dirs, owner = _owners(name, world)
        u, costs = parallel.pair_units_2d(dirs, oracle.ntilde_rule(dvm_inputs.CONFIGS[name].N,
                                                                  dvm_inputs.CONFIGS[name].Nbar)
                                          // np.abs(dirs).max(axis=1))
        assert len(u) == units == len(dirs) // 2
        assert np.all(owner >= 0)
        for i, k in u:
            assert owner[i] == owner[k]
        per_rank = np.bincount([owner[i] for i, _ in u], minlength=world)
        assert per_rank.sum() == units
        assert per_rank.max() <= -(-units // world) + 1


def test_lpt_assign_properties():
    rng = np.random.default_rng(0)
    costs = rng.integers(1, 50, size=300)
    for world in (1, 2, 3, 8):
        owner = parallel.lpt_assign(costs, world)
        loads = np.bincount(owner, weights=costs, minlength=world)
        assert set(owner.tolist()) <= set(range(world))
        # LPT guarantee: makespan <= 4/3 OPT <= 4/3 (mean + max cost)
        assert loads.max() <= (4 / 3) * max(costs.sum() / world, costs.max()) + costs.max()
    assert np.array_equal(parallel.lpt_assign([5, 5, 5], 3), [0, 1, 2])


def test_cell_range():
    for n in (0, 1, 7, 512):
        for world in (1, 2, 3, 8):
            spans = [parallel.cell_range(n, r, world) for r in range(world)]
            assert sum(c for _, c in spans) == n
            pos = 0
            for f0, c in spans:
                assert f0 == pos
                pos += c
    with pytest.raises(ValueError):
        parallel.cell_range(4, 2, 2)


def _handle_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        hs = parallel.exchange_handles(bytes([rank + 1]) * 64)
        q.put((rank, hs))
    finally:
        dist.destroy_process_group()


def test_peer_window_handle_exchange_gloo():
    """The host side of the peer-memory reduction (parallel.PeerDirectionSharded):
    every rank receives every rank's 64-byte IPC handle, in rank order."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_handle_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [bytes([r + 1]) * 64 for r in range(world)]
    assert all(got[r] == want for r in range(world))
