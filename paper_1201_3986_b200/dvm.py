"""Thin Python binding of libdvm (include/dvm.h): argument marshalling only.

Every step of the operator runs in the CUDA library; this module only passes
device pointers (torch tensors' data_ptr), sizes and the current CUDA stream
through the C ABI and turns status codes into exceptions.  There is no CPU
fallback: if libdvm.so is missing or no GPU is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# DVM_LIB: an alternative build of the same library (A/B timing in tools/)
LIB_PATH = os.environ.get("DVM_LIB") or os.path.join(_HERE, "libdvm.so")

DVM_MAXWELL_2D = 0
DVM_HARD_SPHERES_3D = 1

STATUS = {0: "DVM_OK", 1: "DVM_E_NULL", 2: "DVM_E_DIM", 3: "DVM_E_KERNEL", 4: "DVM_E_ORDER",
          5: "DVM_E_UNSUPPORTED", 6: "DVM_E_SHAPE", 7: "DVM_E_ALIAS", 8: "DVM_E_NOMEM", 9: "DVM_E_CUDA",
          10: "DVM_E_STATE"}


class DvmError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{where}: {self.name}" + (f" ({detail})" if detail else ""))


class PlanParams(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int), ("N", ctypes.c_int), ("Nbar", ctypes.c_int), ("Ntilde", ctypes.c_int),
                ("L", ctypes.c_double), ("kernel", ctypes.c_int), ("device", ctypes.c_int),
                ("stream", ctypes.c_void_p), ("shard_rank", ctypes.c_int), ("shard_world", ctypes.c_int)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int), ("N", ctypes.c_int), ("Nbar", ctypes.c_int), ("Ntilde", ctypes.c_int),
                ("kernel", ctypes.c_int), ("A", ctypes.c_int), ("A_local", ctypes.c_int),
                ("rows_total", ctypes.c_int), ("nodes", ctypes.c_int64), ("L", ctypes.c_double),
                ("h", ctypes.c_double), ("workspace_bytes", ctypes.c_size_t), ("launches", ctypes.c_uint64)]


_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libdvm.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libdvm.so not found at {path}; run `python -m paper_1201_3986_b200.build` "
                          "or __graft_entry__.build()")
    L = ctypes.CDLL(path)
    P, I64, V, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_double
    sig = {
        "dvm_plan": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(P)], ctypes.c_int),
        "dvm_plan_ex": ([ctypes.POINTER(PlanParams), ctypes.POINTER(P)], ctypes.c_int),
        "dvm_plan_info": ([P, ctypes.POINTER(PlanInfo)], ctypes.c_int),
        "dvm_plan_directions": ([P, V, V, V, V], ctypes.c_int),
        "dvm_plan_geometry": ([P, ctypes.c_int, V, V, V, V, V, V, ctypes.c_int], ctypes.c_int),
        "dvm_set_stream": ([P, V], ctypes.c_int),
        "dvm_collide": ([P, V, V], ctypes.c_int),
        "dvm_collide_batched": ([P, V, V, I64, I64], ctypes.c_int),
        "dvm_collide_batched_host": ([P, V, V, I64, I64], ctypes.c_int),
        "dvm_moments": ([P, V, V], ctypes.c_int),
        "dvm_euler": ([P, V, D, ctypes.c_int, V], ctypes.c_int),
        "dvm_rk2": ([P, V, D, ctypes.c_int, V], ctypes.c_int),
        "dvm_copy_cells": ([P, V, V, V, V, I64], ctypes.c_int),
        "dvm_set_graphs": ([P, ctypes.c_int], ctypes.c_int),
        "dvm_sync": ([P], ctypes.c_int),
        "dvm_plan_destroy": ([P], ctypes.c_int),
        "dvm_status_str": ([ctypes.c_int], ctypes.c_char_p),
        "dvm_last_error": ([], ctypes.c_char_p),
        "dvm_abi_version": ([], ctypes.c_int),
        "dvm_profile_enable": ([P, ctypes.c_int], ctypes.c_int),
        "dvm_profile_read": ([P, V, V, ctypes.c_int], ctypes.c_int),
        "dvm_profile_name": ([ctypes.c_int], ctypes.c_char_p),
        "dvm_set_path": ([P, ctypes.c_int], ctypes.c_int),
        "dvm_set_weights": ([P, V, V], ctypes.c_int),
        "dvm_set_tuning": ([P, ctypes.c_char_p, ctypes.c_int], ctypes.c_int),
        "dvm_collide_batched_levels": ([V, ctypes.c_int, V, V, I64, I64, V], ctypes.c_int),
        "dvm_peer_window_bytes": ([P, I64, ctypes.c_int], ctypes.c_size_t),
        "dvm_peer_window_alloc": ([P, I64, ctypes.c_int, ctypes.POINTER(V)], ctypes.c_int),
        "dvm_peer_window_free": ([V], ctypes.c_int),
        "dvm_ipc_handle": ([V, ctypes.c_char_p], ctypes.c_int),
        "dvm_ipc_open": ([ctypes.c_char_p, ctypes.POINTER(V)], ctypes.c_int),
        "dvm_ipc_close": ([V], ctypes.c_int),
        "dvm_collide_push": ([P, V, I64, V, ctypes.c_int, ctypes.c_int, ctypes.c_uint], ctypes.c_int),
        "dvm_peer_reduce": ([P, V, V, I64, ctypes.c_int, ctypes.c_uint], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def _check(status: int, where: str):
    if status != 0:
        detail = load().dvm_last_error().decode(errors="replace")
        raise DvmError(status, where, detail)


def _stream_ptr():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


class Plan:
    """A dvm_plan_t: direction table + geometry on the device, workspace."""

    def __init__(self, d: int, N: int, Nbar: int, kernel: Optional[int] = None, Ntilde: int = 0,
                 L: float = 8.0, device: int = -1, shard_rank: int = 0, shard_world: int = 1,
                 stream=None):
        lib = load()
        if kernel is None:
            kernel = DVM_MAXWELL_2D if d == 2 else DVM_HARD_SPHERES_3D
        prm = PlanParams(d, N, Nbar, Ntilde, L, kernel, device,
                         ctypes.c_void_p(stream) if stream is not None else None, shard_rank, shard_world)
        h = ctypes.c_void_p()
        _check(lib.dvm_plan_ex(ctypes.byref(prm), ctypes.byref(h)), "dvm_plan_ex")
        self._h = h
        self.d, self.N, self.Nbar = d, N, Nbar
        inf = self.info()
        self.Ntilde, self.A, self.L, self.h = inf["Ntilde"], inf["A"], inf["L"], inf["h"]
        self.nodes = inf["nodes"]

    # ------------------------------------------------------------ inspection
    def info(self) -> dict:
        inf = PlanInfo()
        _check(load().dvm_plan_info(self._h, ctypes.byref(inf)), "dvm_plan_info")
        return {k: getattr(inf, k) for k, _ in PlanInfo._fields_}

    def directions(self):
        A, d = self.A, self.d
        dirs = np.zeros((A, d), dtype=np.int32)
        M = np.zeros(A, dtype=np.int32)
        a = np.zeros(A, dtype=np.float64)
        loc = np.zeros(A, dtype=np.int32)
        _check(load().dvm_plan_directions(self._h, dirs.ctypes.data, M.ctypes.data, a.ctypes.data,
                                          loc.ctypes.data), "dvm_plan_directions")
        return dirs, M, a, loc.astype(bool)

    def geometry(self, idx: int):
        d = self.d
        u = np.zeros(d, dtype=np.int32)
        w = np.zeros(d, dtype=np.int32)
        n = ctypes.c_int(0)
        cap = 4096
        b = np.zeros(cap, dtype=np.int32)
        lo = np.zeros(cap, dtype=np.int32)
        hi = np.zeros(cap, dtype=np.int32)
        _check(load().dvm_plan_geometry(self._h, idx, u.ctypes.data, w.ctypes.data, ctypes.byref(n),
                                        b.ctypes.data, lo.ctypes.data, hi.ctypes.data, cap), "dvm_plan_geometry")
        k = n.value
        return u, w, np.stack([b[:k], lo[:k], hi[:k]], axis=1)

    def launches(self) -> int:
        return int(self.info()["launches"])

    # ------------------------------------------------------------ evaluation
    def _prep(self, f, out, ncells=None):
        import torch
        if not isinstance(f, torch.Tensor) or not f.is_cuda or f.dtype != torch.float64:
            raise TypeError("f must be a CUDA float64 tensor")
        if not f.is_contiguous():
            raise ValueError("f must be contiguous")
        if f.numel() % self.nodes:
            raise ValueError(f"f.numel() must be a multiple of N^d = {self.nodes}")
        n = f.numel() // self.nodes if ncells is None else ncells
        if out is None:
            out = torch.empty_like(f)
        elif not out.is_cuda or out.dtype != torch.float64 or not out.is_contiguous() or out.numel() != f.numel():
            raise ValueError("out must be a contiguous CUDA float64 tensor shaped like f")
        lib = load()
        _check(lib.dvm_set_stream(self._h, _stream_ptr()), "dvm_set_stream")
        return lib, out, n

    def collide(self, f, out=None):
        """Q = D^{Ñ,N̄}(f,f) on the device for f of N^d (or cells * N^d) doubles."""
        lib, out, n = self._prep(f, out)
        _check(lib.dvm_collide_batched(self._h, _dptr(f), _dptr(out), n, 0), "dvm_collide_batched")
        return out

    collide_batched = collide

    # ------------------------------------------------ peer-memory shard reduction
    def peer_window_alloc(self, ncells: int, world: int) -> int:
        """This rank's peer window (include/dvm.h): device pointer as an int."""
        out = ctypes.c_void_p()
        _check(load().dvm_peer_window_alloc(self._h, ncells, world, ctypes.byref(out)), "dvm_peer_window_alloc")
        return int(out.value)

    def peer_window_bytes(self, ncells: int, world: int) -> int:
        return int(load().dvm_peer_window_bytes(self._h, ncells, world))

    def collide_push(self, f, windows, rank: int, world: int, epoch: int):
        """Q_rank of this shard into slot `rank` of every window (windows: device
        pointers as mapped in this process, windows[rank] the local one)."""
        lib, _, n = self._prep(f, f)
        arr = (ctypes.c_void_p * len(windows))(*[ctypes.c_void_p(int(w)) for w in windows])
        _check(lib.dvm_collide_push(self._h, _dptr(f), n, ctypes.cast(arr, ctypes.c_void_p), rank, world, epoch),
               "dvm_collide_push")

    def peer_reduce(self, window: int, out, world: int, epoch: int):
        """out = sum of the window's slots in rank order, once every push of `epoch` arrived."""
        lib, out, n = self._prep(out, out)
        _check(lib.dvm_peer_reduce(self._h, ctypes.c_void_p(int(window)), _dptr(out), n, world, epoch),
               "dvm_peer_reduce")
        return out

    def collide_host(self, f_host: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
        """End-to-end through the C ABI with HOST buffers (copies inside the call)."""
        f_host = np.ascontiguousarray(f_host, dtype=np.float64)
        if f_host.size % self.nodes:
            raise ValueError("f size must be a multiple of N^d")
        if out is None:
            out = np.empty_like(f_host)
        lib = load()
        _check(lib.dvm_set_stream(self._h, _stream_ptr()), "dvm_set_stream")
        _check(lib.dvm_collide_batched_host(self._h, ctypes.c_void_p(f_host.ctypes.data),
                                            ctypes.c_void_p(out.ctypes.data), f_host.size // self.nodes, 0),
               "dvm_collide_batched_host")
        return out

    def collide_host_ptr(self, f_ptr: int, q_ptr: int, ncells: int):
        """Same with raw host pointers (e.g. pinned torch tensors)."""
        lib = load()
        _check(lib.dvm_set_stream(self._h, _stream_ptr()), "dvm_set_stream")
        _check(lib.dvm_collide_batched_host(self._h, ctypes.c_void_p(f_ptr), ctypes.c_void_p(q_ptr), ncells, 0),
               "dvm_collide_batched_host")

    def _prep_inplace(self, f):
        import torch
        if not isinstance(f, torch.Tensor) or not f.is_cuda or f.dtype != torch.float64 or not f.is_contiguous():
            raise TypeError("f must be a contiguous CUDA float64 tensor")
        if f.numel() != self.nodes:
            raise ValueError(f"f must hold one cell of N^d = {self.nodes} values")
        lib = load()
        _check(lib.dvm_set_stream(self._h, _stream_ptr()), "dvm_set_stream")
        return lib

    def moments(self, f) -> np.ndarray:
        lib = self._prep_inplace(f)
        out = np.zeros(self.d + 2, dtype=np.float64)
        _check(lib.dvm_moments(self._h, _dptr(f), out.ctypes.data), "dvm_moments")
        return out

    def euler(self, f, dt: float, nsteps: int, moments: bool = True):
        """In-place explicit Euler f <- f + dt Q(f) (one cell); returns moments [nsteps+1, d+2]."""
        lib = self._prep_inplace(f)
        mom = np.zeros((nsteps + 1, self.d + 2), dtype=np.float64) if moments else None
        _check(lib.dvm_euler(self._h, _dptr(f), float(dt), int(nsteps),
                             mom.ctypes.data if mom is not None else None), "dvm_euler")
        return mom

    def rk2(self, f, dt: float, nsteps: int, moments: bool = True):
        """In-place TVD-RK2 (Heun) steps (one cell); returns moments [nsteps+1, d+2]."""
        lib = self._prep_inplace(f)
        mom = np.zeros((nsteps + 1, self.d + 2), dtype=np.float64) if moments else None
        _check(lib.dvm_rk2(self._h, _dptr(f), float(dt), int(nsteps),
                           mom.ctypes.data if mom is not None else None), "dvm_rk2")
        return mom

    def copy_cells(self, src, src_idx, dst, dst_idx, ncells: int):
        """dst[dst_idx[c]] = src[src_idx[c]] (CUDA float64 cells, CUDA int64 indices or None)."""
        lib = load()
        _check(lib.dvm_set_stream(self._h, _stream_ptr()), "dvm_set_stream")
        _check(lib.dvm_copy_cells(self._h, _dptr(src), _dptr(src_idx) if src_idx is not None else None,
                                  _dptr(dst), _dptr(dst_idx) if dst_idx is not None else None, int(ncells)),
               "dvm_copy_cells")

    def set_graphs(self, enable: bool):
        """Enable/disable the CUDA-graph replay of the time steppers."""
        _check(load().dvm_set_graphs(self._h, 1 if enable else 0), "dvm_set_graphs")

    def set_path(self, path: int):
        """0 = auto, 1 = v1 orbit sweeps, 2 = FFT-loss kernels (gain3d / pair2d),
        3 = spectral reference, 4 = 3D N = 64 FFT gain, 5 = 2D small-grid pairs,
        6 = 3D N = 32 spectral direction pairs, 7 = 2D tiles."""
        _check(load().dvm_set_path(self._h, int(path)), "dvm_set_path")

    def set_tuning(self, key: str, value: int):
        """dvm_set_tuning: "max_groups", "ring_slots", "fg_chunks", "g3_cl", "verbose",
        "timing_dbg" (timing only: Q wrong)."""
        _check(load().dvm_set_tuning(self._h, key.encode(), int(value)), "dvm_set_tuning")

    def set_weights(self, a_box=None, b_box=None):
        """General decoupled weights a(k), b(l) (eq:decoup) as host arrays of shape
        [2Ñ+1]*d indexed by k + Ñ (None: built-in values; both None: built-in operator)."""
        import numpy as np
        side = 2 * self.Ntilde + 1
        arrs = []
        for w in (a_box, b_box):
            if w is None:
                arrs.append(None)
                continue
            w = np.ascontiguousarray(np.asarray(w, dtype=np.float64))
            if w.size != side ** self.d:
                raise ValueError(f"weight tables need (2Ñ+1)^d = {side ** self.d} entries")
            arrs.append(w)
        _check(load().dvm_set_weights(self._h, *(None if w is None else w.ctypes.data for w in arrs)),
               "dvm_set_weights")

    def profile(self, enable: bool = True):
        """Start (clear) / stop per-kernel CUDA-event timing inside libdvm."""
        lib = load()
        _check(lib.dvm_set_stream(self._h, _stream_ptr()), "dvm_set_stream")
        _check(lib.dvm_profile_enable(self._h, 1 if enable else 0), "dvm_profile_enable")

    def profile_read(self) -> dict:
        """{kernel class: (total ms, launches)} of the recorded launches."""
        lib = load()
        n = 0
        names = []
        while lib.dvm_profile_name(n) is not None:
            names.append(lib.dvm_profile_name(n).decode())
            n += 1
        ms = np.zeros(n, dtype=np.float64)
        cnt = np.zeros(n, dtype=np.uint64)
        _check(lib.dvm_profile_read(self._h, ms.ctypes.data, cnt.ctypes.data, n), "dvm_profile_read")
        return {names[k]: (float(ms[k]), int(cnt[k])) for k in range(n)}

    def sync(self):
        _check(load().dvm_sync(self._h), "dvm_sync")

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            load().dvm_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def peer_window_free(window: int):
    _check(load().dvm_peer_window_free(ctypes.c_void_p(int(window))), "dvm_peer_window_free")


def ipc_handle(dptr: int) -> bytes:
    """64-byte CUDA IPC handle of a device allocation (e.g. a peer window)."""
    buf = ctypes.create_string_buffer(64)
    _check(load().dvm_ipc_handle(ctypes.c_void_p(int(dptr)), buf), "dvm_ipc_handle")
    return buf.raw


def ipc_open(handle: bytes) -> int:
    """Map another process's allocation; returns the device pointer here."""
    if len(handle) != 64:
        raise ValueError("CUDA IPC handles are 64 bytes")
    out = ctypes.c_void_p()
    _check(load().dvm_ipc_open(ctypes.c_char_p(bytes(handle)), ctypes.byref(out)), "dvm_ipc_open")
    return int(out.value)


def ipc_close(dptr: int):
    _check(load().dvm_ipc_close(ctypes.c_void_p(int(dptr))), "dvm_ipc_close")
