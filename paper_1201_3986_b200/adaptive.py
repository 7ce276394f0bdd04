"""Space-dependent N̄ over a batch of spatial cells ("the
parameter N̄ can be made space dependent, according to the fact that some
regions in space deserve less accuracy than others, being close to
equilibrium").

One plan per N̄ level, all with the same Ñ (so the operators differ only in
the direction truncation of eq:decD).  Evaluation is one call of the C ABI's
dvm_collide_batched_levels: libdvm buckets the cells by level on the device,
evaluates each bucket as one batch with its plan and scatters Q back.  This
module only marshals arguments.

`equilibrium_levels` is a reference policy (not part of the operator): the
relative L1 distance of each cell to the lattice Maxwellian with its moments.
"""
from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np

from .dvm import Plan, _check, _dptr, _stream_ptr, load


class AdaptiveNbar:
    def __init__(self, d: int, N: int, levels: Sequence[int], Ntilde: int = 0, **plan_kw):
        levels = sorted(set(int(x) for x in levels))
        if not levels or levels[0] < 1:
            raise ValueError("levels must be positive N̄ values")
        probe = Plan(d, N, levels[-1], Ntilde=Ntilde, **plan_kw)
        self.Ntilde = probe.Ntilde  # the rule for the largest level, shared by every level
        self.levels = levels
        self.plans = {levels[-1]: probe}
        for nb in levels[:-1]:
            self.plans[nb] = Plan(d, N, nb, Ntilde=self.Ntilde, **plan_kw)
        self.d, self.N, self.nodes = d, N, probe.nodes
        self._handles = (ctypes.c_void_p * len(levels))(*[self.plans[nb]._h.value for nb in levels])

    def directions(self) -> dict:
        return {nb: p.A for nb, p in self.plans.items()}

    def collide(self, f, nbar_per_cell, out=None):
        """Q for f [cells, N^d] (CUDA float64) with cell c evaluated at N̄ =
        nbar_per_cell[c] (host sequence or CUDA int tensor of values from `levels`)."""
        import torch
        if not isinstance(f, torch.Tensor) or not f.is_cuda or f.dtype != torch.float64 or not f.is_contiguous():
            raise TypeError("f must be a contiguous CUDA float64 tensor")
        ncells = f.numel() // self.nodes
        if f.numel() != ncells * self.nodes:
            raise ValueError(f"f.numel() must be a multiple of N^d = {self.nodes}")
        lut = {nb: i for i, nb in enumerate(self.levels)}
        if isinstance(nbar_per_cell, torch.Tensor):
            nb = nbar_per_cell.to(device=f.device, dtype=torch.int64).reshape(-1)
            table = torch.full((max(self.levels) + 1,), -1, dtype=torch.int32, device=f.device)
            for v, i in lut.items():
                table[v] = i
            level = table[nb.clamp(0, max(self.levels))].masked_fill((nb < 0) | (nb > max(self.levels)), -1)
        else:
            nbh = np.asarray(nbar_per_cell, dtype=np.int64).reshape(-1)
            bad = set(np.unique(nbh).tolist()) - set(self.levels)
            if bad:
                raise ValueError(f"N̄ values {sorted(bad)} are not levels of this plan set")
            level = torch.from_numpy(np.array([lut[int(v)] for v in nbh], dtype=np.int32)).to(f.device)
        if level.numel() != ncells:
            raise ValueError("one N̄ per cell")
        level = level.to(torch.int32).contiguous()
        if out is None:
            out = torch.empty_like(f)
        lib = load()
        for p in self.plans.values():
            _check(lib.dvm_set_stream(p._h, _stream_ptr()), "dvm_set_stream")
        _check(lib.dvm_collide_batched_levels(ctypes.cast(self._handles, ctypes.c_void_p), len(self.levels),
                                              _dptr(f), _dptr(out), ncells, 0, _dptr(level)),
               "dvm_collide_batched_levels")
        return out


def equilibrium_levels(f, d: int, N: int, L: float, levels: Sequence[int], thresholds: Sequence[float]):
    """Reference policy: N̄ per cell from the relative L1 distance δ of the cell
    to the lattice Maxwellian with its mass, momentum and energy: the first
    level whose threshold exceeds δ (thresholds ascending, one per level but the
    last).  Host/torch computation, outside the operator."""
    import torch
    levels = list(levels)
    if len(thresholds) != len(levels) - 1:
        raise ValueError("one threshold per level but the last")
    h = 2.0 * L / N
    v1 = (torch.arange(N, dtype=torch.float64, device=f.device) - N // 2) * h
    grids = torch.meshgrid(*([v1] * d), indexing="ij")
    V = torch.stack([g.reshape(-1) for g in grids], dim=1)  # [N^d, d]
    fc = f.reshape(-1, N ** d)
    w = h ** d
    rho = fc.sum(1) * w
    u = (fc @ V) * w / rho[:, None]
    E = (fc * (V ** 2).sum(1)).sum(1) * w / rho
    T = (E - (u ** 2).sum(1)) / d
    dv2 = ((V[None, :, :] - u[:, None, :]) ** 2).sum(2)
    M = rho[:, None] / (2 * np.pi * T[:, None]) ** (d / 2) * torch.exp(-dv2 / (2 * T[:, None]))
    delta = (fc - M).abs().sum(1) / fc.abs().sum(1)
    out = np.full(fc.shape[0], levels[-1], dtype=np.int64)
    dl = delta.cpu().numpy()
    for i in range(len(levels) - 2, -1, -1):
        out[dl < thresholds[i]] = levels[i]
    return out, dl
