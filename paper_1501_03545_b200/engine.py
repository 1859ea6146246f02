"""Per-device handle on the C ABI: one hrg_context (device workspace + last
result) per CUDA device, plus helpers to move results to host numpy arrays
(pinned when torch's CUDA runtime is available) or device torch tensors."""

from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from .geometry import ModelParams, model_constants


@dataclass(frozen=True)
class Shard:
    """Angular sector [2pi*index/count, 2pi*(index+1)/count) of query vertices."""

    index: int = 0
    count: int = 1


def default_device() -> int:
    for var in ("HRGEN_B200_DEVICE", "LOCAL_RANK"):
        if os.environ.get(var):
            return int(os.environ[var])
    return 0


def make_model(model: ModelParams) -> _lib.Model:
    c = model_constants(model.R, model.alpha)
    return _lib.Model(n=int(model.n), alpha=float(model.alpha), R=float(model.R), **c)


def _pinned_empty(shape, dtype):
    """Host array in page-locked memory when torch's CUDA allocator is
    available (cached pinned blocks, so repeated calls do not re-pin)."""
    try:
        import torch
        if torch.cuda.is_available():
            tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.int64): torch.int64,
                   np.dtype(np.int32): torch.int32}[np.dtype(dtype)]
            return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()
    except Exception:  # pragma: no cover - fall back to pageable host memory
        pass
    return np.empty(shape, dtype=dtype)


class Engine:
    def __init__(self, device: int | None = None, stream: int | None = None):
        L = _lib.load()
        self.device = default_device() if device is None else int(device)
        ctx = ctypes.c_void_p()
        _lib.check(L.hrg_context_create(self.device, ctypes.c_void_p(stream or 0),
                                        ctypes.byref(ctx)))
        self._ctx = ctx
        self._L = L
        self.last_stats: _lib.Stats | None = None
        # one context = one set of device buffers and one last result: a
        # generation and the copy of its result must not interleave with
        # another thread's (hold `lock` across both; the methods take it too)
        self.lock = threading.RLock()
        self.trig = _lib.TRIG_LIBM

    def __del__(self):
        try:
            if getattr(self, "_ctx", None):
                self._L.hrg_context_destroy(self._ctx)
                self._ctx = None
        except Exception:
            pass

    def set_stream(self, stream: int | None):
        with self.lock:
            _lib.check(self._L.hrg_context_set_stream(self._ctx, ctypes.c_void_p(stream or 0)))

    def launches(self) -> int:
        """Kernel launches this engine's context has queued (library kernels
        such as CUB's not counted)."""
        out = ctypes.c_int64()
        _lib.check(self._L.hrg_context_launches(self._ctx, ctypes.byref(out)))
        return out.value

    def set_trig(self, mode: int):
        """sin/cos of later calls: _lib.TRIG_LIBM (hrgen's glibc arithmetic,
        the default) or _lib.TRIG_CR (correctly rounded)."""
        with self.lock:
            _lib.check(self._L.hrg_context_set_trig(self._ctx, int(mode)))
            self.trig = int(mode)

    # -- work ---------------------------------------------------------------
    def generate(self, model: ModelParams, seed: int, order: int = _lib.ORDER_SAMPLE,
                 shard: Shard | None = None) -> _lib.Stats:
        st = _lib.Stats()
        sh = _lib.Shard(shard.index, shard.count) if shard else None
        with self.lock:
            _lib.check(self._L.hrg_generate(self._ctx, ctypes.byref(make_model(model)),
                                            ctypes.c_uint64(int(seed)), order,
                                            ctypes.byref(sh) if sh else None, ctypes.byref(st)))
            self.last_stats = st
        return st

    def edges_from_coords(self, model: ModelParams, phi, r_poincare,
                          shard: Shard | None = None) -> _lib.Stats:
        st = _lib.Stats()
        sh = _lib.Shard(shard.index, shard.count) if shard else None
        phi, r_poincare, kind = self._coords(phi, r_poincare)
        if kind == _lib.MEM_DEVICE:
            p_phi, p_rp = phi.data_ptr(), r_poincare.data_ptr()
        else:
            p_phi, p_rp = phi.ctypes.data, r_poincare.ctypes.data
        with self.lock:
            _lib.check(self._L.hrg_edges_from_coords(self._ctx, ctypes.byref(make_model(model)),
                                                     ctypes.c_void_p(p_phi), ctypes.c_void_p(p_rp),
                                                     kind, ctypes.byref(sh) if sh else None,
                                                     ctypes.byref(st)))
            self.last_stats = st
        return st

    def _coords(self, phi, r_poincare):
        """Validated coordinate pair: equal length, 1-d, float64, contiguous;
        CUDA tensors on this engine's device stay on the device (converted
        there if needed), everything else becomes host numpy arrays."""
        if getattr(phi, "is_cuda", False) or getattr(r_poincare, "is_cuda", False):
            import torch
            dev = torch.device("cuda", self.device)
            phi = torch.as_tensor(phi, device=dev).to(torch.float64).contiguous()
            r_poincare = torch.as_tensor(r_poincare, device=dev).to(torch.float64).contiguous()
            shape_phi, shape_rp = tuple(phi.shape), tuple(r_poincare.shape)
            kind = _lib.MEM_DEVICE
        else:
            phi = np.ascontiguousarray(phi, dtype=np.float64)
            r_poincare = np.ascontiguousarray(r_poincare, dtype=np.float64)
            shape_phi, shape_rp = phi.shape, r_poincare.shape
            kind = _lib.MEM_HOST
        if len(shape_phi) != 1 or shape_phi != shape_rp:
            from .errors import ParameterDomainError
            raise ParameterDomainError(
                f"phi and r_poincare must be 1-d arrays of equal length (got {shape_phi} and "
                f"{shape_rp})")
        return phi, r_poincare, kind

    def edges_brute_force(self, phi, r_poincare, radius: float) -> int:
        """hrgen generate_brute_force on the device; returns the near-tie count."""
        phi, r_poincare, kind = self._coords(phi, r_poincare)
        if kind == _lib.MEM_DEVICE:
            phi, r_poincare = phi.cpu().numpy(), r_poincare.cpu().numpy()
        ties = ctypes.c_int64()
        with self.lock:
            _lib.check(self._L.hrg_edges_brute_force(self._ctx, phi.size, phi.ctypes.data,
                                                     r_poincare.ctypes.data, _lib.MEM_HOST,
                                                     float(radius), ctypes.byref(ties)))
        return ties.value

    def sample_points(self, model: ModelParams, seed: int, order: int = _lib.ORDER_SAMPLE):
        n = int(model.n)
        phi, rn, rp = (np.empty(n, np.float64) for _ in range(3))
        with self.lock:
            _lib.check(self._L.hrg_sample_points(self._ctx, ctypes.byref(make_model(model)),
                                                 ctypes.c_uint64(int(seed)), order, _lib.MEM_HOST,
                                                 phi.ctypes.data, rn.ctypes.data, rp.ctypes.data))
        return phi, rn, rp

    # -- results ------------------------------------------------------------
    def sizes(self):
        n = ctypes.c_int64()
        nnz = ctypes.c_int64()
        with self.lock:
            _lib.check(self._L.hrg_result_sizes(self._ctx, ctypes.byref(n), ctypes.byref(nnz)))
        return n.value, nnz.value

    def copy_csr(self, index_dtype=np.int64, pinned=True):
        with self.lock:
            return self._copy_csr(index_dtype, pinned)

    def _copy_csr(self, index_dtype, pinned):
        n, nnz = self.sizes()
        alloc = _pinned_empty if pinned else (lambda s, d: np.empty(s, d))
        indptr = alloc(n + 1, np.int64)
        indices = alloc(nnz, index_dtype)
        _lib.check(self._L.hrg_copy_result(self._ctx, _lib.MEM_HOST, None, None, None,
                                           indptr.ctypes.data, indices.ctypes.data,
                                           np.dtype(index_dtype).itemsize))
        return indptr, indices

    def copy_coords(self, pinned=False):
        with self.lock:
            return self._copy_coords(pinned)

    def _copy_coords(self, pinned):
        n, _ = self.sizes()
        alloc = _pinned_empty if pinned else (lambda s, d: np.empty(s, d))
        phi, rn, rp = (alloc(n, np.float64) for _ in range(3))
        _lib.check(self._L.hrg_copy_result(self._ctx, _lib.MEM_HOST, phi.ctypes.data,
                                           rn.ctypes.data, rp.ctypes.data, None, None, 8))
        return phi, rn, rp

    def copy_result_into(self, phi=None, r_native=None, r_poincare=None, indptr=None,
                         indices=None):
        """Copy into caller-provided host numpy arrays (any may be None)."""
        def ptr(a):
            return None if a is None else a.ctypes.data
        ib = indices.dtype.itemsize if indices is not None else 8
        with self.lock:
            _lib.check(self._L.hrg_copy_result(self._ctx, _lib.MEM_HOST, ptr(phi), ptr(r_native),
                                               ptr(r_poincare), ptr(indptr), ptr(indices), ib))

    def device_csr(self):
        """(indptr int64, indices int32) as torch CUDA tensors (device copies)."""
        import torch
        with self.lock:
            n, nnz = self.sizes()
            dev = torch.device("cuda", self.device)
            indptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
            indices = torch.empty(max(nnz, 0), dtype=torch.int32, device=dev)
            _lib.check(self._L.hrg_copy_result(self._ctx, _lib.MEM_DEVICE, None, None, None,
                                               indptr.data_ptr(), indices.data_ptr(), 4))
        return indptr, indices

    def debug_sincos(self, x, mode=_lib.TRIG_LIBM):
        """Device sin/cos of host angles: mode 0 glibc's (the product's
        default), 1 correctly rounded (fast path), 2 correctly rounded (full)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        s = np.empty_like(x)
        c = np.empty_like(x)
        with self.lock:
            _lib.check(self._L.hrg_debug_sincos(self._ctx, x.size, x.ctypes.data, int(mode),
                                                s.ctypes.data, c.ctypes.data))
        return s, c

    def debug_sincos_compare(self, n, seed=0):
        """(mismatches, rejected) of the fast sin/cos against the full one."""
        mm = ctypes.c_int64()
        rj = ctypes.c_int64()
        _lib.check(self._L.hrg_debug_sincos_compare(self._ctx, int(n), ctypes.c_uint64(seed),
                                                    ctypes.byref(mm), ctypes.byref(rj)))
        return mm.value, rj.value

    def synchronize(self):
        _lib.check(self._L.hrg_synchronize(self._ctx))


_engines: dict[int, Engine] = {}
_engines_lock = threading.Lock()


def get_engine(device: int | None = None) -> Engine:
    dev = default_device() if device is None else int(device)
    with _engines_lock:
        eng = _engines.get(dev)
        if eng is None:
            eng = Engine(dev)
            _engines[dev] = eng
        return eng
