"""ctypes front-end of the C oracle (oracle/dvm_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg.  Never imported by the
product package ``paper_1201_3986_b200``.  Shares no code with it.

Every function follows the direct double sum written in dvm_oracle.c's header
(eq:DR, with the direction truncation of eq:decD,
PAPER.md:798-827, and the weights of PAPER.md:582-587).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dvm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C99 + OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O2", "-std=gnu99", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-shared", "-fPIC", _SRC, "-o", tmp, "-lm"]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            L.dvm_oracle_ntilde_rule.argtypes = [ctypes.c_int, ctypes.c_int]
            L.dvm_oracle_ntilde_rule.restype = ctypes.c_int
            L.dvm_oracle_directions.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
            L.dvm_oracle_directions.restype = ctypes.c_int64
            L.dvm_oracle_pairs.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                           ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
            L.dvm_oracle_pairs.restype = ctypes.c_int64
            L.dvm_oracle_collide.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_double, ctypes.c_void_p, ctypes.c_int64,
                                             ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_int]
            L.dvm_oracle_collide.restype = ctypes.c_int
            L.dvm_oracle_collide_w.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_double, ctypes.c_void_p, ctypes.c_int64,
                                               ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                               ctypes.c_int]
            L.dvm_oracle_collide_w.restype = ctypes.c_int
            _lib = L
    return _lib


def ntilde_rule(N: int, Nbar: int) -> int:
    """Reading R2: Ñ = max(floor(N/(3+√2)), N̄)."""
    return int(lib().dvm_oracle_ntilde_rule(N, Nbar))


def directions(d: int, Nbar: int) -> np.ndarray:
    """Canonical primitive lines of order <= N̄, lexicographic."""
    n = lib().dvm_oracle_directions(d, Nbar, None)
    out = np.zeros((max(n, 1), d), dtype=np.int32)
    lib().dvm_oracle_directions(d, Nbar, out.ctypes.data)
    return out[:n]


def pairs(d: int, Ntilde: int, Nbar: int, h: float, dirs: np.ndarray | None = None):
    """The oracle's pair list (k, l, a(k)) in its summation order."""
    nd, dp = _dirs_arg(dirs, d)
    n = lib().dvm_oracle_pairs(d, Ntilde, Nbar, h, nd, dp, 0, None, None, None)
    k = np.zeros((max(n, 1), d), dtype=np.int32)
    l = np.zeros((max(n, 1), d), dtype=np.int32)
    a = np.zeros(max(n, 1), dtype=np.float64)
    lib().dvm_oracle_pairs(d, Ntilde, Nbar, h, nd, dp, n, k.ctypes.data, l.ctypes.data, a.ctypes.data)
    return k[:n], l[:n], a[:n]


def _dirs_arg(dirs, d):
    if dirs is None:
        return -1, None
    arr = np.ascontiguousarray(np.asarray(dirs, dtype=np.int32).reshape(-1, d))
    _dirs_arg._keep = arr  # keep alive for the duration of the call
    return arr.shape[0], arr.ctypes.data


def collide(f: np.ndarray, d: int, N: int, Nbar: int, Ntilde: int, L: float = 8.0,
            points: np.ndarray | None = None, dirs: np.ndarray | None = None,
            nthreads: int = 0, a_box: np.ndarray | None = None, b_box: np.ndarray | None = None,
            diagnostics: bool = True):
    """Direct-sum Q, G, Lo for f of shape [cells, N^d] (or [N]*d / [cells]+[N]*d).

    points: optional node indices (row-major) -> outputs [cells, npts]; a 1-D
    array is used for every cell, a [cells, npts] array gives each cell its own;
    dirs: optional subset of canonical lines (direction-sharding tests);
    a_box, b_box: optional general decoupled weights a(k), b(l) (eq:decoup,
    PAPER.md:575-579) tabulated over [-Ñ,Ñ]^d (shape [2Ñ+1]*d, index k + Ñ);
    Γ̃_{k,l} = a(k) b(l) replaces h^{d+1}|k|/gcd(k) (a_box None: that default;
    b_box None: b = 1).
    diagnostics: False skips G and Lo (returned as None); Q is unchanged.
    Returns (Q, G, Lo) as float64 arrays of shape [cells, npts or N^d].
    """
    nodes = N ** d
    fa = np.ascontiguousarray(np.asarray(f, dtype=np.float64).reshape(-1, nodes))
    ncells = fa.shape[0]
    per_cell = 0
    if points is None:
        npts, pp, pk = -1, None, None
        nout = nodes
    else:
        pk = np.asarray(points, dtype=np.int64)
        if pk.ndim == 2:
            if pk.shape[0] != ncells:
                raise ValueError("per-cell points must have shape [cells, npts]")
            per_cell = 1
            npts = pk.shape[1]
        else:
            npts = pk.size
        pk = np.ascontiguousarray(pk.reshape(-1))
        pp = pk.ctypes.data
        nout = npts
    Q = np.zeros((ncells, nout), dtype=np.float64)
    G = np.zeros_like(Q) if diagnostics else None
    Lo = np.zeros_like(Q) if diagnostics else None
    if dirs is None:
        nd, dp, keep = -1, None, None
    else:
        keep = np.ascontiguousarray(np.asarray(dirs, dtype=np.int32).reshape(-1, d))
        nd, dp = keep.shape[0], keep.ctypes.data
    box = (2 * Ntilde + 1) ** d
    wa = None if a_box is None else np.ascontiguousarray(np.asarray(a_box, dtype=np.float64).reshape(-1))
    wb = None if b_box is None else np.ascontiguousarray(np.asarray(b_box, dtype=np.float64).reshape(-1))
    for w in (wa, wb):
        if w is not None and w.size != box:
            raise ValueError(f"weight tables must have (2Ñ+1)^d = {box} entries")
    rc = lib().dvm_oracle_collide_w(d, N, Nbar, Ntilde, float(L), fa.ctypes.data, ncells, npts, pp, per_cell,
                                    nd, dp, None if wa is None else wa.ctypes.data,
                                    None if wb is None else wb.ctypes.data, Q.ctypes.data,
                                    None if G is None else G.ctypes.data,
                                    None if Lo is None else Lo.ctypes.data, int(nthreads))
    if rc != 0:
        raise ValueError(f"dvm_oracle_collide failed with {rc}")
    del keep, pk, wa, wb
    return Q, G, Lo
