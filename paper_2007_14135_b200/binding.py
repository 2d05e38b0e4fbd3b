"""Thin ctypes binding of libdoa.so (include/doa.h).  Argument marshalling only: every step of the
hot path runs in the CUDA kernels behind the C ABI.  PyTorch supplies device memory and streams.

There is no fallback: if libdoa.so is missing or cannot be loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DOA_LIB") or os.path.join(_HERE, "libdoa.so")   # DOA_LIB: tuning builds only

ALG = {"phd": 0, "music": 1, "ev": 2, "mn": 3}
ENGINE = {"toeplitz_fp64": 0, "direct_fp32": 1, "direct_tf32x3": 2}           # doa_plan_set_engine (include/doa.h)
INFO_NOCONV, INFO_DEGENERATE, INFO_CAND_OVERFLOW, INFO_UNDERDETERMINED = 1, 2, 4, 8
STATUS = {0: "DOA_OK", 1: "DOA_ERR_INVALID_ARG", 2: "DOA_ERR_UNSUPPORTED", 3: "DOA_ERR_OUT_OF_MEMORY",
          4: "DOA_ERR_CUDA"}

EXPORTS = ("doa_generate", "doa_plan_create", "doa_plan_create_array", "doa_plan_destroy", "doa_plan_capacity",
           "doa_plan_info", "doa_covariance", "doa_eig",
           "doa_spectrum", "doa_peaks", "doa_run", "doa_run_multi", "doa_scan_multi", "doa_run_host", "doa_plan_set_engine",
           "doa_last_launch_count",
           "doa_status_string", "doa_last_error", "doa_version")


class DoaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class PlanInfo(C.Structure):
    """doa_plan_info_t (include/doa.h)."""
    _fields_ = [("M", C.c_int32), ("D", C.c_int32), ("alg", C.c_int32), ("geom", C.c_int32),
                ("device", C.c_int32), ("capacity", C.c_int32), ("L", C.c_int64), ("max_batch", C.c_int64),
                ("engine", C.c_int32), ("reserved", C.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libdoa.so not built at {LIB_PATH}; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    vp, dp, fp, i32p, i64, i32, d = C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_double
    L.doa_plan_create.argtypes = [C.POINTER(C.c_void_p), i32, d, i32, d, d, i64, i32, i64]
    L.doa_plan_create_array.argtypes = [C.POINTER(C.c_void_p), i32, C.POINTER(C.c_double), i32, d, d, i64, d, d,
                                        i64, i32, i32, i64]
    L.doa_plan_destroy.argtypes = [vp]
    L.doa_plan_capacity.argtypes = [vp]
    L.doa_plan_capacity.restype = i32
    L.doa_plan_info.argtypes = [vp, C.POINTER(PlanInfo)]
    L.doa_covariance.argtypes = [vp, fp, i64, i64, dp, vp]
    L.doa_eig.argtypes = [vp, dp, i64, dp, dp, i32p, vp]
    L.doa_spectrum.argtypes = [vp, dp, dp, i64, fp, i32p, vp]
    L.doa_peaks.argtypes = [vp, i64, i32p, fp, i32p, i32p, vp]
    L.doa_run.argtypes = [vp, fp, i64, i64, i32p, fp, i32p, fp, i32p, vp]
    L.doa_run_host.argtypes = [C.POINTER(C.c_void_p), i32, fp, i64, i64, i32p, fp, i32p, i32p, vp]
    L.doa_run_multi.argtypes = [C.POINTER(C.c_void_p), i32, fp, i64, i64, i32p, fp, i32p, i32p, vp]
    L.doa_scan_multi.argtypes = [C.POINTER(C.c_void_p), i32, i64, vp]
    L.doa_plan_set_engine.argtypes = [vp, i32]
    L.doa_generate.argtypes = [i32, d, i32, dp, i32, d, C.c_uint64, i64, i64, i64, fp, vp]
    L.doa_last_launch_count.restype = i32
    L.doa_status_string.argtypes = [C.c_int]
    L.doa_status_string.restype = C.c_char_p
    L.doa_last_error.restype = C.c_char_p
    L.doa_version.restype = i32
    for name in EXPORTS:
        if name not in ("doa_plan_capacity", "doa_last_launch_count", "doa_status_string", "doa_last_error",
                        "doa_version"):
            getattr(L, name).restype = C.c_int
    return L


lib = _load()


def _check(st: int):
    if st != 0:
        raise DoaError(st, lib.doa_last_error().decode())


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        if not t.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return t.data_ptr()
    return t


def _stream(stream):
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return stream


def _f32(X):
    """complex64 tensor -> its interleaved float view pointer owner."""
    if X.dtype == torch.complex64:
        return torch.view_as_real(X)
    return X


def _f64(X):
    if X.dtype == torch.complex128:
        return torch.view_as_real(X)
    return X


# ----------------------------------------------------------------------------- argument validation
# The C ABI takes raw pointers and sizes; a tensor of the wrong shape, dtype or device would make a
# kernel read out of bounds (or fault and poison the CUDA context).  Every wrapper therefore checks
# its tensors against the plan (doa_plan_info) before calling into libdoa, raising ValueError.
_INFO_CACHE: dict = {}


def _hval(plan):
    return plan.value if isinstance(plan, C.c_void_p) else int(plan)


def plan_info(plan) -> PlanInfo:
    """doa_plan_info of a plan handle (cached: a plan's parameters never change)."""
    key = _hval(plan)
    info = _INFO_CACHE.get(key)
    if info is None:
        info = PlanInfo()
        _check(lib.doa_plan_info(key, C.byref(info)))
        _INFO_CACHE[key] = info
    return info


def _need(t, name, dtype, shape, device):
    """t must be a contiguous `dtype` tensor of `shape` (None = any extent) on CUDA device ordinal
    `device` (or on the host when device is None)."""
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name}: expected a torch.Tensor, got {type(t).__name__}")
    if t.dtype != dtype:
        raise ValueError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if t.dim() != len(shape) or any(e is not None and int(a) != e for a, e in zip(t.shape, shape)):
        want = tuple("*" if e is None else e for e in shape)
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {want}")
    if device is None:
        if t.device.type != "cpu":
            raise ValueError(f"{name}: must be a host (CPU) tensor, got {t.device}")
    elif t.device.type != "cuda" or t.device.index != device:
        raise ValueError(f"{name}: must be on cuda:{device} (the plan's device), got {t.device}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")


def _need_P(P, B, pi):
    """P: float32 (B, L) — or (B, naz, nel) for a general-array plan — on the plan's device."""
    _need(P, "P", torch.float32, (B,) + (None,) * (P.dim() - 1) if isinstance(P, torch.Tensor) else (B, None),
          pi.device)
    if P.dim() not in (2, 3) or P.numel() != B * pi.L:
        raise ValueError(f"P: shape {tuple(P.shape)}, expected ({B}, {pi.L}) elements per frame")


# ----------------------------------------------------------------------------- same-named calls
def doa_plan_create(M, d_over_lambda, D, theta0_deg, dtheta_deg, L, alg, max_batch):
    h = C.c_void_p()
    a = ALG[alg] if isinstance(alg, str) else int(alg)
    _check(lib.doa_plan_create(C.byref(h), M, d_over_lambda, D, theta0_deg, dtheta_deg, L, a, max_batch))
    return h


def doa_plan_create_array(M, positions, D, az0_deg, daz_deg, naz, el0_deg, del_deg, nel, az_wrap, alg, max_batch):
    """positions: (M, 3) element coordinates in wavelengths (host array-like)."""
    import numpy as np
    pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(M, 3)
    h = C.c_void_p()
    a = ALG[alg] if isinstance(alg, str) else int(alg)
    _check(lib.doa_plan_create_array(C.byref(h), M, pos.ctypes.data_as(C.POINTER(C.c_double)), D, az0_deg, daz_deg,
                                     naz, el0_deg, del_deg, nel, int(bool(az_wrap)), a, max_batch))
    return h


def doa_generate(M, d_over_lambda, D, theta_deg, snr_db, seed, frame0, X, stream=None):
    """On-device Eq. 1 snapshots (NEXT-3).  theta_deg: float64 CUDA tensor (D,) or (B, D);
    X: complex64 CUDA tensor (B, N, M), overwritten."""
    dev = torch.cuda.current_device()
    _need(X, "X", torch.complex64, (None, None, M), dev)
    B, N = X.shape[0], X.shape[1]
    _need(theta_deg, "theta_deg", torch.float64, (B, None) if theta_deg.dim() == 2 else (None,), dev)
    if D >= 1 and theta_deg.shape[-1] != D:               # D itself is validated by the C side
        raise ValueError(f"theta_deg: {theta_deg.shape[-1]} angles per frame, expected D = {D}")
    per_frame = 1 if theta_deg.dim() == 2 else 0
    _check(lib.doa_generate(M, d_over_lambda, D, _ptr(theta_deg), per_frame, snr_db, int(seed), frame0, B, N,
                            _ptr(_f32(X)), _stream(stream)))


def doa_plan_destroy(plan):
    _INFO_CACHE.pop(_hval(plan), None)
    _check(lib.doa_plan_destroy(plan))


def doa_covariance(plan, X, R, stream=None):
    """X: complex64 (B, N, M) CUDA tensor -> R: complex128 (B, M, M) CUDA tensor."""
    pi = plan_info(plan)
    _need(X, "X", torch.complex64, (None, None, pi.M), pi.device)
    B, N = X.shape[0], X.shape[1]
    _need(R, "R", torch.complex128, (B, pi.M, pi.M), pi.device)
    _check(lib.doa_covariance(plan, _ptr(_f32(X)), B, N, _ptr(_f64(R)), _stream(stream)))


def doa_eig(plan, R, lam, V, info, stream=None):
    pi = plan_info(plan)
    _need(R, "R", torch.complex128, (None, pi.M, pi.M), pi.device)
    B = R.shape[0]
    _need(lam, "lam", torch.float64, (B, pi.M), pi.device)
    _need(V, "V", torch.complex128, (B, pi.M, pi.M), pi.device)
    _need(info, "info", torch.int32, (B,), pi.device)
    _check(lib.doa_eig(plan, _ptr(_f64(R)), B, _ptr(lam), _ptr(_f64(V)), _ptr(info), _stream(stream)))


def doa_spectrum(plan, lam, V, info, P=None, stream=None):
    pi = plan_info(plan)
    _need(lam, "lam", torch.float64, (None, pi.M), pi.device)
    B = lam.shape[0]
    _need(V, "V", torch.complex128, (B, pi.M, pi.M), pi.device)
    _need(info, "info", torch.int32, (B,), pi.device)
    if P is not None:
        _need_P(P, B, pi)
    _check(lib.doa_spectrum(plan, _ptr(lam), _ptr(_f64(V)), B, _ptr(P), _ptr(info), _stream(stream)))


def doa_peaks(plan, B, idx, val, npk, info, stream=None):
    pi = plan_info(plan)
    _need(idx, "idx", torch.int32, (B, pi.D), pi.device)
    _need(val, "val", torch.float32, (B, pi.D), pi.device)
    _need(npk, "npk", torch.int32, (B,), pi.device)
    _need(info, "info", torch.int32, (B,), pi.device)
    _check(lib.doa_peaks(plan, B, _ptr(idx), _ptr(val), _ptr(npk), _ptr(info), _stream(stream)))


def doa_run(plan, X, idx, val, npk, info, P=None, stream=None):
    pi = plan_info(plan)
    _need(X, "X", torch.complex64, (None, None, pi.M), pi.device)
    B, N = X.shape[0], X.shape[1]
    _need(idx, "idx", torch.int32, (B, pi.D), pi.device)
    _need(val, "val", torch.float32, (B, pi.D), pi.device)
    _need(npk, "npk", torch.int32, (B,), pi.device)
    _need(info, "info", torch.int32, (B,), pi.device)
    if P is not None:
        _need_P(P, B, pi)
    _check(lib.doa_run(plan, _ptr(_f32(X)), B, N, _ptr(idx), _ptr(val), _ptr(npk), _ptr(P), _ptr(info),
                       _stream(stream)))


def doa_run_multi(plans, X, idx, val, npk, info, stream=None):
    """Several plans (sharing M, D) on one device batch: X complex64 (B, N, M); outputs on the
    device, idx/val (nplans, B, D), npk/info (nplans, B)."""
    if not isinstance(plans, (list, tuple)):
        plans = [plans]
    pi = plan_info(plans[0])
    n = len(plans)
    _need(X, "X", torch.complex64, (None, None, pi.M), pi.device)
    B, N = X.shape[0], X.shape[1]
    _need(idx, "idx", torch.int32, (n, B, pi.D), pi.device)
    _need(val, "val", torch.float32, (n, B, pi.D), pi.device)
    _need(npk, "npk", torch.int32, (n, B), pi.device)
    _need(info, "info", torch.int32, (n, B), pi.device)
    arr = (C.c_void_p * n)(*[_hval(p) for p in plans])
    _check(lib.doa_run_multi(arr, n, _ptr(_f32(X)), B, N, _ptr(idx), _ptr(val), _ptr(npk), _ptr(info),
                             _stream(stream)))


def doa_plan_set_engine(plan, engine):
    """Scan engine of a ULA plan: "toeplitz_fp64" | "direct_fp32" (or the DOA_ENGINE_* value)."""
    e = ENGINE[engine] if isinstance(engine, str) else int(engine)
    _check(lib.doa_plan_set_engine(plan, e))


def doa_scan_multi(plans, B, stream=None):
    """S4-S6 again for 1..4 grid-sharing ULA plans from the coefficients they hold (include/doa.h);
    the candidate lists are rebuilt for a following doa_peaks."""
    if not isinstance(plans, (list, tuple)):
        plans = [plans]
    n = len(plans)
    arr = (C.c_void_p * n)(*[_hval(p) for p in plans])
    _check(lib.doa_scan_multi(arr, n, int(B), _stream(stream)))


def run_multi(plans, X, stream=None):
    """Convenience: all `plans` (Plan objects sharing M, D, device) on X -> (idx, val, npk, info)
    device tensors of shape (nplans, B, D) / (nplans, B)."""
    dev = plans[0].device
    B, n, D = X.shape[0], len(plans), plans[0].D
    idx = torch.empty((n, B, D), dtype=torch.int32, device=dev)
    val = torch.empty((n, B, D), dtype=torch.float32, device=dev)
    npk = torch.empty((n, B), dtype=torch.int32, device=dev)
    info = torch.empty((n, B), dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        doa_run_multi([p.h for p in plans], X, idx, val, npk, info, stream)
    return idx, val, npk, info


def doa_run_host(plans, X_host, idx, val, npk, info, stream=None):
    """plans: one plan handle or a list sharing M, D.  Host (CPU) tensors in and out:
    idx/val (nplans, B, D), npk/info (nplans, B).  Pinned X_host gives overlapped async copies."""
    if not isinstance(plans, (list, tuple)):
        plans = [plans]
    pi = plan_info(plans[0])
    n = len(plans)
    _need(X_host, "X_host", torch.complex64, (None, None, pi.M), None)
    B, N = X_host.shape[0], X_host.shape[1]
    _need(idx, "idx", torch.int32, (n, B, pi.D), None)
    _need(val, "val", torch.float32, (n, B, pi.D), None)
    _need(npk, "npk", torch.int32, (n, B), None)
    _need(info, "info", torch.int32, (n, B), None)
    arr = (C.c_void_p * n)(*[_hval(p) for p in plans])
    _check(lib.doa_run_host(arr, n, _ptr(_f32(X_host)), B, N, _ptr(idx), _ptr(val), _ptr(npk),
                            _ptr(info), _stream(stream)))


def doa_last_launch_count() -> int:
    return int(lib.doa_last_launch_count())


# ----------------------------------------------------------------------------- convenience
def _device(device) -> torch.device:
    d = torch.device(device)
    if d.type != "cuda":
        raise ValueError(f"plans live on a CUDA device, got {d}")
    return torch.device("cuda", torch.cuda.current_device() if d.index is None else d.index)


class Plan:
    """Owns one doa_plan_t.  Methods allocate outputs with torch on the plan's device."""

    def __init__(self, M, D, alg, dtheta, L=None, theta0=-90.0, d_over_lambda=0.5, max_batch=1,
                 device="cuda", engine="toeplitz_fp64"):
        if L is None:             # last grid point <= 90 deg (the C side's end check)
            L = int(math.floor((90.0 - theta0) / dtheta + 1e-9)) + 1
        self.M, self.D, self.alg, self.L, self.theta0, self.dtheta = M, D, alg, L, theta0, dtheta
        self.device = _device(device)
        self.max_batch = max_batch
        self.h = None
        with torch.cuda.device(self.device):
            self.h = doa_plan_create(M, d_over_lambda, D, theta0, dtheta, L, alg, max_batch)
        self.cap = int(lib.doa_plan_capacity(self.h))
        self.engine = "toeplitz_fp64"
        if engine != "toeplitz_fp64":
            self.set_engine(engine)

    def set_engine(self, engine):
        """"toeplitz_fp64" (the product), "direct_fp32" or "direct_tf32x3" (SURVEY §8(f) NEXT-2 A/B engines:
        the direct form on the FP32 pipe or on tcgen05 tensor cores)."""
        with torch.cuda.device(self.device):
            doa_plan_set_engine(self.h, engine)
        self.engine = engine

    @classmethod
    def array(cls, positions, D, alg, az0=0.0, daz=1.0, naz=360, el0=90.0, del_=1.0, nel=1, az_wrap=True,
              max_batch=1, device="cuda"):
        """General-geometry plan on an azimuth x elevation grid (doa_plan_create_array)."""
        self = cls.__new__(cls)
        M = len(positions)
        self.M, self.D, self.alg, self.L = M, D, alg, naz * nel
        self.naz, self.nel = naz, nel
        self.device = _device(device)
        self.max_batch = max_batch
        self.h = None
        with torch.cuda.device(self.device):
            self.h = doa_plan_create_array(M, positions, D, az0, daz, naz, el0, del_, nel, az_wrap, alg, max_batch)
        self.cap = int(lib.doa_plan_capacity(self.h))
        return self

    def close(self):
        if self.h is not None:
            with torch.cuda.device(self.device):
                doa_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _outs(self, B):
        dev = self.device
        return (torch.empty((B, self.D), dtype=torch.int32, device=dev),
                torch.empty((B, self.D), dtype=torch.float32, device=dev),
                torch.empty((B,), dtype=torch.int32, device=dev),
                torch.zeros((B,), dtype=torch.int32, device=dev))

    def covariance(self, X, stream=None):
        R = torch.empty((X.shape[0], self.M, self.M), dtype=torch.complex128, device=self.device)
        with torch.cuda.device(self.device):
            doa_covariance(self.h, X, R, stream)
        return R

    def eig(self, R, stream=None):
        B = R.shape[0]
        lam = torch.empty((B, self.M), dtype=torch.float64, device=self.device)
        V = torch.empty((B, self.M, self.M), dtype=torch.complex128, device=self.device)
        info = torch.empty((B,), dtype=torch.int32, device=self.device)
        with torch.cuda.device(self.device):
            doa_eig(self.h, R, lam, V, info, stream)
        return lam, V, info

    def spectrum(self, lam, V, info=None, want_P=False, stream=None):
        B = lam.shape[0]
        if info is None:
            info = torch.zeros((B,), dtype=torch.int32, device=self.device)
        P = torch.empty((B, self.L), dtype=torch.float32, device=self.device) if want_P else None
        with torch.cuda.device(self.device):
            doa_spectrum(self.h, lam, V, info, P, stream)
        return P, info

    def peaks(self, B, info=None, stream=None):
        idx, val, npk, info0 = self._outs(B)
        info = info0 if info is None else info
        with torch.cuda.device(self.device):
            doa_peaks(self.h, B, idx, val, npk, info, stream)
        return idx, val, npk, info

    def run(self, X, want_P=False, stream=None):
        B = X.shape[0]
        idx, val, npk, info = self._outs(B)
        P = torch.empty((B, self.L), dtype=torch.float32, device=self.device) if want_P else None
        with torch.cuda.device(self.device):
            doa_run(self.h, X, idx, val, npk, info, P, stream)
        return idx, val, npk, info, P

    def run_host(self, X_host, others=(), stream=None):
        """End-to-end from host memory for this plan and `others` (Plans sharing M, D)."""
        plans = [self] + list(others)
        B, n = X_host.shape[0], len(plans)
        idx = torch.empty((n, B, self.D), dtype=torch.int32)
        val = torch.empty((n, B, self.D), dtype=torch.float32)
        npk = torch.empty((n, B), dtype=torch.int32)
        info = torch.empty((n, B), dtype=torch.int32)
        with torch.cuda.device(self.device):
            doa_run_host([p.h for p in plans], X_host, idx, val, npk, info, stream)
        if not others:
            return idx[0], val[0], npk[0], info[0]
        return idx, val, npk, info
