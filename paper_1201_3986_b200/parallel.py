"""Multi-GPU plumbing (one process per GPU, torch.distributed).

Two shardings of the hot path (the decomposition eq:decD is
a sum over directions and the operator is local in x, so both are exact):

* direction sharding of ONE grid (c1-c4): rank r evaluates the LPT share of
  the directions (libdvm's dvm_plan_ex shard_rank/shard_world; in 2D whole
  pair units {e, e⊥}) into a partial Q_r, then one fp64 sum all-reduce over
  NVLink (NCCL) gives Q = sum_r Q_r;
* cell sharding of a batch (c5): contiguous blocks of cells per rank, no
  collective on the data path.

The compute step is injected (`partial_fn`) so that the same reduction code
path runs in the CPU `gloo` tests with the oracle standing in for the GPU
kernel (tests only) and on the GPU with libdvm.
"""
from __future__ import annotations

from typing import Callable, Sequence

import numpy as np


def cell_range(ncells: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of cells owned by `rank`: (first, count); remainders to low ranks."""
    if world < 1 or not 0 <= rank < world or ncells < 0:
        raise ValueError("bad cell sharding arguments")
    base, rem = divmod(ncells, world)
    first = rank * base + min(rank, rem)
    return first, base + (1 if rank < rem else 0)


def lpt_assign(costs: Sequence[int], world: int) -> np.ndarray:
    """Owner rank of every direction: longest-processing-time first, ties to the
    lowest rank, stable in direction order.  Mirrors libdvm's build_table."""
    costs = np.asarray(costs, dtype=np.int64)
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = np.zeros(world, dtype=np.int64)
    owner = np.zeros(len(costs), dtype=np.int64)
    for i in order:
        r = int(np.argmin(load))
        load[r] += costs[i]
        owner[i] = r
    return owner


def pair_units_2d(dirs: np.ndarray, M: Sequence[int]):
    """2D pair units {e, e⊥} of a direction table (e⊥ is again
    a direction of the table, with the same M_e): list of (i, mate) with
    i < mate in order of i, and the unit costs 64 + 2 M_e + 1 (the pair
    kernels' O(1) per-node work plus the O(M_e) segment prologue).  Mirrors
    libdvm's build_table for d = 2."""
    dirs = np.asarray(dirs)
    index = {tuple(int(c) for c in e): i for i, e in enumerate(dirs)}
    units, costs = [], []
    for i, (a, b) in enumerate(dirs):
        p = (-int(b), int(a))
        if p[0] < 0 or (p[0] == 0 and p[1] < 0):
            p = (-p[0], -p[1])
        k = index[p]
        if i < k:
            units.append((i, k))
            costs.append(64 + 2 * int(M[i]) + 1)
    return units, np.asarray(costs, dtype=np.int64)


def owners_2d(dirs: np.ndarray, M: Sequence[int], world: int) -> np.ndarray:
    """Owner rank of every 2D direction: LPT over whole pair units."""
    units, costs = pair_units_2d(dirs, M)
    uown = lpt_assign(costs, world)
    owner = np.full(len(dirs), -1, dtype=np.int64)
    for (i, k), r in zip(units, uown):
        owner[i] = owner[k] = r
    return owner


def sharded_collide(partial_fn: Callable, f, group=None):
    """Q = all_reduce_sum(partial_fn(f)) over the process group.

    partial_fn(f) returns this rank's partial Q (a torch tensor on the rank's
    device: CUDA + NCCL in production, CPU + gloo in tests)."""
    import torch.distributed as dist
    q = partial_fn(f)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(q, op=dist.ReduceOp.SUM, group=group)
    return q


class DirectionSharded:
    """Direction-sharded evaluation of one grid on this rank's GPU."""

    def __init__(self, d: int, N: int, Nbar: int, group=None, **plan_kw):
        import torch.distributed as dist
        from .dvm import Plan
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.group = group
        self.plan = Plan(d, N, Nbar, shard_rank=rank, shard_world=world, **plan_kw)

    def __call__(self, f, out=None):
        return sharded_collide(lambda x: self.plan.collide(x, out), f, self.group)


def exchange_handles(handle: bytes, group=None) -> list:
    """Every rank's 64-byte IPC handle, in rank order (all_gather_object; the
    handles are host bytes, so this runs on gloo and NCCL groups alike)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = [None] * world
    dist.all_gather_object(out, handle, group=group)
    return out


class PeerDirectionSharded:
    """Direction-sharded evaluation of a batch whose reduction runs over peer
    memory instead of NCCL (include/dvm.h, dvm_collide_push / dvm_peer_reduce):
    this rank's partial Q_r is pushed into slot r of every rank's peer window
    over NVLink, then every rank adds its window's slots in rank order.  The
    windows are exchanged once, at construction, as CUDA IPC handles."""

    def __init__(self, d: int, N: int, Nbar: int, ncells: int = 1, group=None, **plan_kw):
        import torch.distributed as dist
        from . import dvm
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.ncells = ncells
        self.plan = dvm.Plan(d, N, Nbar, shard_rank=self.rank, shard_world=self.world, **plan_kw)
        self.window = self.plan.peer_window_alloc(ncells, self.world)
        handles = exchange_handles(dvm.ipc_handle(self.window), group) if self.world > 1 else [None]
        self.windows = [self.window if r == self.rank else dvm.ipc_open(h) for r, h in enumerate(handles)]
        self.epoch = 0
        if self.world > 1:
            dist.barrier(group)  # every window is mapped before anyone pushes

    def __call__(self, f, out=None):
        import torch
        if f.numel() != self.ncells * self.plan.nodes:
            raise ValueError("f must hold the ncells given at construction")
        if out is None:
            out = torch.empty_like(f)
        self.epoch += 1
        self.plan.collide_push(f, self.windows, self.rank, self.world, self.epoch)
        return self.plan.peer_reduce(self.window, out, self.world, self.epoch)

    def close(self):
        from . import dvm
        for r, w in enumerate(self.windows):
            if r != self.rank and w:
                dvm.ipc_close(w)
        if self.window:
            dvm.peer_window_free(self.window)
        self.windows, self.window = [], 0
