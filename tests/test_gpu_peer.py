"""GPU: the direction-shard reduction over peer memory (include/dvm.h,
dvm_collide_push / dvm_peer_reduce; Q = Σ_r Q_r over the
ranks' direction shards).  One GPU per box here, so the ranks are either
virtual (several shard plans in one process, windows in one device's memory)
or two processes sharing the GPU through CUDA IPC; in both cases every push
completes before any reduce starts, so no kernel ever waits on another rank's
kernel on the same GPU.  Checks: every rank gets the same bits, equal to the
partials added in rank order, and the oracle's Q."""
import os
import socket

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


def _virtual_ranks(d, N, Nbar, f, world, epochs=2):
    from paper_1201_3986_b200 import Plan, dvm
    ncells = f.shape[0]
    plans = [Plan(d, N, Nbar, shard_rank=r, shard_world=world) for r in range(world)]
    wins = [p.peer_window_alloc(ncells, world) for p in plans]
    ft = torch.from_numpy(np.ascontiguousarray(f)).cuda()
    try:
        for epoch in range(1, epochs + 1):
            for r, p in enumerate(plans):
                p.collide_push(ft, wins, r, world, epoch)
            qs = [p.peer_reduce(wins[r], torch.empty_like(ft), world, epoch) for r, p in enumerate(plans)]
            torch.cuda.synchronize()
            qs = [q.cpu().numpy() for q in qs]
            # the partials added in rank order, evaluated separately
            parts = [p.collide(ft) for p in plans]
            ref = parts[0].clone()
            for q in parts[1:]:
                ref += q
            ref = ref.cpu().numpy()
            for q in qs:
                assert np.array_equal(q, qs[0]), "ranks disagree"
            assert np.array_equal(qs[0], ref), "not the rank-order sum of the partials"
        return qs[0]
    finally:
        for w in wins:
            dvm.peer_window_free(w)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_peer_reduce_c1_virtual_ranks(world):
    cfg = dvm_inputs.CONFIGS["c1"]
    f = dvm_inputs.make("c1")
    q = _virtual_ranks(2, cfg.N, cfg.Nbar, f, world)
    Qo, _, _ = oracle.collide(f, 2, cfg.N, cfg.Nbar, oracle.ntilde_rule(cfg.N, cfg.Nbar), cfg.L)
    assert np.abs(q - Qo).max() <= TOL * np.abs(Qo).max()


@pytest.mark.parametrize("name,world", [("c3", 4), ("c4", 2)])
def test_peer_reduce_baseline_grids_virtual_ranks(name, world):
    """c3 (the direction-sharded BASELINE config) and c4 at full size: the
    peer reduction equals the unsharded evaluation to rounding and the oracle
    on sampled nodes."""
    from paper_1201_3986_b200 import Plan
    cfg = dvm_inputs.CONFIGS[name]
    f = dvm_inputs.make(name)
    q = _virtual_ranks(cfg.d, cfg.N, cfg.Nbar, f, world, epochs=1)
    full = Plan(cfg.d, cfg.N, cfg.Nbar).collide(torch.from_numpy(f).cuda()).cpu().numpy()
    assert np.abs(q - full).max() <= 1e-13 * np.abs(full).max()
    pts = np.random.default_rng(3).choice(cfg.N ** cfg.d, size=200, replace=False)
    Qo, _, _ = oracle.collide(f, cfg.d, cfg.N, cfg.Nbar, oracle.ntilde_rule(cfg.N, cfg.Nbar), cfg.L,
                              points=np.sort(pts), diagnostics=False)
    assert np.abs(q[0][np.sort(pts)] - Qo[0]).max() <= TOL * np.abs(Qo[0]).max()


def test_peer_abi_errors():
    from paper_1201_3986_b200 import Plan, dvm
    p = Plan(2, 16, 4, shard_rank=1, shard_world=2)
    with pytest.raises(dvm.DvmError) as e:
        p.peer_window_alloc(1, 3)  # world differs from the plan's shard_world
    assert e.value.name == "DVM_E_STATE"
    w = p.peer_window_alloc(1, 2)
    ft = torch.zeros(256, dtype=torch.float64, device="cuda")
    with pytest.raises(dvm.DvmError) as e:
        p.collide_push(ft, [w, w], 0, 2, 1)  # rank differs from the plan's shard_rank
    assert e.value.name == "DVM_E_STATE"
    with pytest.raises(dvm.DvmError) as e:
        p.collide_push(ft, [w, w], 1, 2, 0)  # epoch 0
    assert e.value.name == "DVM_E_STATE"
    assert p.peer_window_bytes(1, 2) >= 2 * 256 * 8 + 2 * 4
    dvm.peer_window_free(w)


def _ipc_worker(rank, world, port, outdir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_1201_3986_b200 import Plan, dvm
    from paper_1201_3986_b200.parallel import exchange_handles
    cfg = dvm_inputs.CONFIGS["c2"]
    f = torch.from_numpy(dvm_inputs.make("c2")).cuda()
    p = Plan(2, cfg.N, cfg.Nbar, shard_rank=rank, shard_world=world)
    win = p.peer_window_alloc(1, world)
    handles = exchange_handles(dvm.ipc_handle(win))
    wins = [win if r == rank else dvm.ipc_open(h) for r, h in enumerate(handles)]
    dist.barrier()
    for epoch in (1, 2):
        p.collide_push(f, wins, rank, world, epoch)
        torch.cuda.synchronize()
        dist.barrier()  # every push is complete: the reduce below never waits on a kernel of this GPU
        q = p.peer_reduce(win, torch.empty_like(f), world, epoch)
        torch.cuda.synchronize()
        np.save(os.path.join(outdir, f"q{rank}_{epoch}.npy"), q.cpu().numpy())
        dist.barrier()
    for r, w in enumerate(wins):
        if r != rank:
            dvm.ipc_close(w)
    dist.barrier()
    dvm.peer_window_free(win)
    dist.destroy_process_group()


def test_peer_reduce_two_processes_ipc(tmp_path):
    """Two processes (gloo for the handle exchange and barriers) share the GPU:
    windows mapped through CUDA IPC, pushes into the other process's window,
    two epochs; both ranks get the same bits, equal to the unsharded Q to
    rounding (c2 grid)."""
    import torch.multiprocessing as mp
    from paper_1201_3986_b200 import Plan
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_ipc_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    cfg = dvm_inputs.CONFIGS["c2"]
    full = Plan(2, cfg.N, cfg.Nbar).collide(torch.from_numpy(dvm_inputs.make("c2")).cuda()).cpu().numpy()
    for epoch in (1, 2):
        q0 = np.load(tmp_path / f"q0_{epoch}.npy")
        q1 = np.load(tmp_path / f"q1_{epoch}.npy")
        assert np.array_equal(q0, q1)
        assert np.abs(q0 - full).max() <= 1e-13 * np.abs(full).max()
