"""Thin Python binding of the C ABI in include/geninv.h (ctypes; argument marshalling only).

Every step of the path runs in libgeninv.so's sm_100a kernels.  There is no
CPU or eager fallback: if the library cannot be loaded, or no CUDA device is
present, every call raises.

Functions mirror the C names (geninv_d, geninv_batched_d, geninv_gram_d, ...)
and take torch tensors (CUDA float64, row-major) for device buffers.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GENINV_LIB", os.path.join(_HERE, "libgeninv.so"))  # instrumented builds only

GENINV_OK, GENINV_EINVAL, GENINV_ENONFINITE, GENINV_ENOTSPD, GENINV_ECUDA, GENINV_ENOMEM, GENINV_EALIGN, \
    GENINV_ESTATE, GENINV_ENCCL, GENINV_ERANGE = range(10)


class GeninvError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"geninv status {status}: {msg}")
        self.status = status


class _Opts(ctypes.Structure):
    _fields_ = [("tol_rel", ctypes.c_double), ("tol_abs", ctypes.c_double)]


class _Info(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("rank", ctypes.c_int64), ("transposed", ctypes.c_int32),
                ("status", ctypes.c_int32), ("min_acc", ctypes.c_double), ("max_drop", ctypes.c_double),
                ("min_pivot", ctypes.c_double), ("order", ctypes.c_int32), ("not_psd_hint", ctypes.c_int32)]


@dataclass
class Info:
    tol: float
    rank: int
    transposed: bool
    status: int
    min_acc: float
    max_drop: float
    min_pivot: float
    order: int = 0       # a7 product order of geninv_d: 0 = X G', 1 = K (K' G') (low rank, f4)
    not_psd_hint: int = 0  # a tentative pivot below -s * tol (user-supplied A not PSD; reported, not an error)

    @property
    def mu_acc(self):
        return self.min_acc / self.tol if self.tol > 0 else float("inf")

    @property
    def mu_drop(self):
        return self.max_drop / self.tol if self.tol > 0 else (0.0 if self.max_drop == 0 else float("inf"))


_lib = None

_SIGS = {
    "geninv_create": [ctypes.c_void_p, ctypes.c_int],
    "geninv_set_stream": [ctypes.c_void_p, ctypes.c_void_p],
    "geninv_destroy": [ctypes.c_void_p],
    "geninv_d": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                 ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
    "geninv_host_d": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                      ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
    "geninv_batched_d": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                         ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                         ctypes.c_void_p, ctypes.c_void_p],
    "geninv_gram_d": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                      ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64],
    "geninv_from_gram_d": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_void_p],
    "geninv_apply_d": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                       ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64],
    "geninv_set_emulation": [ctypes.c_void_p, ctypes.c_int32],
    "geninv_frchol_d": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                        ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
    "geninv_spd_inverse_d": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                             ctypes.c_int64],
    "geninv_copy_x": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p],
    "geninv_d_async": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                       ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p],
    "geninv_sharded_d": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                         ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                         ctypes.c_void_p, ctypes.c_void_p],
    "geninv_solve_d": [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                       ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
}

EXPORTED = sorted(list(_SIGS) + ["geninv_strerror", "geninv_launch_count"])


def load(path: str = LIB_PATH):
    """Load libgeninv.so (raises if it is missing -- there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libgeninv.so not built ({path}); run `python -m paper_0804_4809_b200.build`")
    lib = ctypes.CDLL(path)
    for name, args in _SIGS.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.geninv_strerror.argtypes = [ctypes.c_int]
    lib.geninv_strerror.restype = ctypes.c_char_p
    lib.geninv_launch_count.argtypes = [ctypes.c_void_p]
    lib.geninv_launch_count.restype = ctypes.c_int64
    _lib = lib
    return lib


def _check(st: int):
    if st != GENINV_OK:
        raise GeninvError(st, load().geninv_strerror(st).decode())


def _opts(tol_rel=1e-9, tol_abs=-1.0):
    return _Opts(tol_rel, tol_abs)


def _dev(t: torch.Tensor, name: str):
    if not (t.is_cuda and t.dtype == torch.float64 and t.dim() in (2, 3) and t.stride(-1) == 1):
        raise ValueError(f"{name}: need a CUDA float64 row-major tensor (unit column stride)")
    return t.data_ptr()


class Handle:
    """Owns a geninv_handle (workspace + stream) on one CUDA device."""

    def __init__(self, device: int | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("geninv needs a CUDA device (no CPU fallback)")
        lib = load()
        self.device = torch.cuda.current_device() if device is None else device
        h = ctypes.c_void_p()
        _check(lib.geninv_create(ctypes.byref(h), self.device))
        self._h = h
        self._lib = lib
        self.use_stream(torch.cuda.current_stream(self.device))

    def set_emulation(self, mode: int):
        """a7 arithmetic: 0 = FP64 tensor cores (DMMA, default), 1 = emulated on the INT8 tensor cores."""
        _check(self._lib.geninv_set_emulation(self._h, int(mode)))

    def use_stream(self, stream: torch.cuda.Stream):
        _check(self._lib.geninv_set_stream(self._h, ctypes.c_void_p(stream.cuda_stream)))

    def close(self):
        if getattr(self, "_h", None):
            self._lib.geninv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launch_count(self) -> int:
        return int(self._lib.geninv_launch_count(self._h))

    # ---------------------------------------------------------------- whole path
    def geninv_d(self, G: torch.Tensor, Gp: torch.Tensor | None = None, tol_rel=1e-9, tol_abs=-1.0):
        """G+ of G (m x n) -> (Gp (n x m), Info)."""
        m, n = G.shape
        if Gp is None:
            Gp = torch.empty(n, m, dtype=torch.float64, device=G.device)
        info = _Info()
        rank = ctypes.c_int64()
        o = _opts(tol_rel, tol_abs)
        _check(self._lib.geninv_d(self._h, _dev(G, "G"), m, n, G.stride(0), _dev(Gp, "Gp"), Gp.stride(0),
                                  ctypes.byref(rank), ctypes.byref(o), ctypes.byref(info)))
        return Gp, _info(info)

    def geninv_d_async(self, G: torch.Tensor, Gp: torch.Tensor | None = None, rank: torch.Tensor | None = None,
                       tol_rel=1e-9, tol_abs=-1.0):
        """G+ without host synchronisation -> (Gp, rank int64[1] on the device)."""
        m, n = G.shape
        if Gp is None:
            Gp = torch.empty(n, m, dtype=torch.float64, device=G.device)
        if rank is None:
            rank = torch.empty(1, dtype=torch.int64, device=G.device)
        o = _opts(tol_rel, tol_abs)
        _check(self._lib.geninv_d_async(self._h, _dev(G, "G"), m, n, G.stride(0), _dev(Gp, "Gp"), Gp.stride(0),
                                        ctypes.c_void_p(rank.data_ptr()), ctypes.byref(o)))
        return Gp, rank

    def geninv_host_d(self, G: torch.Tensor, Gp: torch.Tensor, tol_rel=1e-9, tol_abs=-1.0):
        """Host-buffer variant (G, Gp CPU float64 tensors, ideally pinned)."""
        if G.is_cuda or Gp.is_cuda or G.dtype != torch.float64 or Gp.dtype != torch.float64:
            raise ValueError("geninv_host_d takes CPU float64 tensors")
        m, n = G.shape
        info = _Info()
        rank = ctypes.c_int64()
        o = _opts(tol_rel, tol_abs)
        _check(self._lib.geninv_host_d(self._h, G.data_ptr(), m, n, G.stride(0), Gp.data_ptr(), Gp.stride(0),
                                       ctypes.byref(rank), ctypes.byref(o), ctypes.byref(info)))
        return Gp, _info(info)

    def geninv_batched_d(self, G: torch.Tensor, Gp: torch.Tensor | None = None, rank: torch.Tensor | None = None,
                         tol_rel=1e-9, tol_abs=-1.0):
        """G: (batch, m, n) -> (Gp (batch, n, m), rank int32[batch]); does not synchronise."""
        b, m, n = G.shape
        if Gp is None:
            Gp = torch.empty(b, n, m, dtype=torch.float64, device=G.device)
        if rank is None:
            rank = torch.empty(b, dtype=torch.int32, device=G.device)
        o = _opts(tol_rel, tol_abs)
        _check(self._lib.geninv_batched_d(self._h, _dev(G, "G"), m, n, G.stride(1), G.stride(0), b, _dev(Gp, "Gp"),
                                          Gp.stride(1), Gp.stride(0), rank.data_ptr(), ctypes.byref(o)))
        return Gp, rank

    def geninv_solve_d(self, G: torch.Tensor, F: torch.Tensor, W: torch.Tensor | None = None, tol_rel=1e-9,
                       tol_abs=-1.0):
        """Minimum-norm least-squares W = G+ F (G: m x n, F: m x k) -> (W (n x k), Info)."""
        m, n = G.shape
        k = F.shape[1]
        if W is None:
            W = torch.empty(n, k, dtype=torch.float64, device=G.device)
        info = _Info()
        rank = ctypes.c_int64()
        o = _opts(tol_rel, tol_abs)
        _check(self._lib.geninv_solve_d(self._h, _dev(G, "G"), m, n, G.stride(0), _dev(F, "F"), k, F.stride(0),
                                        _dev(W, "W"), W.stride(0), ctypes.byref(rank), ctypes.byref(o),
                                        ctypes.byref(info)))
        return W, _info(info)

    def geninv_sharded_d(self, nccl_comm: int, G_local: torch.Tensor, trans: int, Gp_local: torch.Tensor,
                         tol_rel=1e-9, tol_abs=-1.0):
        """One sharded step (local Gram, ncclAllReduce of A, replicated factorisation, local block of G+)."""
        m, n = G_local.shape
        info = _Info()
        rank = ctypes.c_int64()
        o = _opts(tol_rel, tol_abs)
        _check(self._lib.geninv_sharded_d(self._h, ctypes.c_void_p(nccl_comm), _dev(G_local, "G"), m, n,
                                          G_local.stride(0), int(trans), _dev(Gp_local, "Gp"), Gp_local.stride(0),
                                          ctypes.byref(rank), ctypes.byref(o), ctypes.byref(info)))
        return Gp_local, _info(info)

    # ---------------------------------------------------------------- split form
    def geninv_gram_d(self, G: torch.Tensor, trans: int, A: torch.Tensor):
        m, n = G.shape
        _check(self._lib.geninv_gram_d(self._h, _dev(G, "G"), m, n, G.stride(0), int(trans), _dev(A, "A"),
                                       A.stride(0)))
        return A

    def geninv_from_gram_d(self, A: torch.Tensor, tol_rel=1e-9, tol_abs=-1.0):
        s = A.shape[0]
        info = _Info()
        rank = ctypes.c_int64()
        o = _opts(tol_rel, tol_abs)
        _check(self._lib.geninv_from_gram_d(self._h, _dev(A, "A"), s, A.stride(0), ctypes.byref(rank),
                                            ctypes.byref(o), ctypes.byref(info)))
        return _info(info)

    def geninv_apply_d(self, G: torch.Tensor, trans: int, Gp: torch.Tensor):
        m, n = G.shape
        _check(self._lib.geninv_apply_d(self._h, _dev(G, "G"), m, n, G.stride(0), int(trans), _dev(Gp, "Gp"),
                                        Gp.stride(0)))
        return Gp

    # ---------------------------------------------------------------- single steps
    def geninv_frchol_d(self, A: torch.Tensor, tol_rel=1e-9, tol_abs=-1.0):
        """a2+a3 on A (s x s lower) -> (L (s x r), piv int32[r], Info)."""
        s = A.shape[0]
        ld = (s + 1) // 2 * 2
        Lbuf = torch.empty(s, ld, dtype=torch.float64, device=A.device)
        piv = torch.empty(s, dtype=torch.int32, device=A.device)
        info = _Info()
        rank = ctypes.c_int64()
        o = _opts(tol_rel, tol_abs)
        _check(self._lib.geninv_frchol_d(self._h, _dev(A, "A"), s, A.stride(0), _dev(Lbuf, "L"), ld,
                                         piv.data_ptr(), ctypes.byref(rank), ctypes.byref(o), ctypes.byref(info)))
        r = rank.value
        return Lbuf[:, :r], piv[:r], _info(info)

    def geninv_spd_inverse_d(self, B: torch.Tensor, M: torch.Tensor | None = None):
        r = B.shape[0]
        if M is None:
            M = torch.empty(r, (r + 1) // 2 * 2, dtype=torch.float64, device=B.device)
        _check(self._lib.geninv_spd_inverse_d(self._h, _dev(B, "B"), r, B.stride(0), _dev(M, "M"), M.stride(0)))
        return M[:, :r]

    def geninv_copy_x(self) -> torch.Tensor:
        """A copy of the handle's X = L M M L' (s x s)."""
        s = ctypes.c_int64()
        _check(self._lib.geninv_copy_x(self._h, None, 0, ctypes.byref(s)))
        n = s.value
        out = torch.empty(n, max(2, (n + 1) // 2 * 2), dtype=torch.float64, device=f"cuda:{self.device}")
        _check(self._lib.geninv_copy_x(self._h, ctypes.c_void_p(out.data_ptr()), out.stride(0), None))
        return out[:, :n]


def _info(i: _Info) -> Info:
    return Info(i.tol, int(i.rank), bool(i.transposed), int(i.status), i.min_acc, i.max_drop, i.min_pivot,
                int(i.order), int(i.not_psd_hint))
