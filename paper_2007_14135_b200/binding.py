"""Thin ctypes binding of libdoa.so (include/doa.h).  Argument marshalling only: every step of the
hot path runs in the CUDA kernels behind the C ABI.  PyTorch supplies device memory and streams.

There is no fallback: if libdoa.so is missing or cannot be loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DOA_LIB") or os.path.join(_HERE, "libdoa.so")   # DOA_LIB: tuning builds only

ALG = {"phd": 0, "music": 1, "ev": 2, "mn": 3}
INFO_NOCONV, INFO_DEGENERATE, INFO_CAND_OVERFLOW, INFO_UNDERDETERMINED = 1, 2, 4, 8
STATUS = {0: "DOA_OK", 1: "DOA_ERR_INVALID_ARG", 2: "DOA_ERR_UNSUPPORTED", 3: "DOA_ERR_OUT_OF_MEMORY",
          4: "DOA_ERR_CUDA"}

EXPORTS = ("doa_generate", "doa_plan_create", "doa_plan_create_array", "doa_plan_destroy", "doa_plan_capacity", "doa_covariance", "doa_eig",
           "doa_spectrum", "doa_peaks", "doa_run", "doa_run_host", "doa_last_launch_count",
           "doa_status_string", "doa_last_error", "doa_version")


class DoaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


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
    L.doa_covariance.argtypes = [vp, fp, i64, i64, dp, vp]
    L.doa_eig.argtypes = [vp, dp, i64, dp, dp, i32p, vp]
    L.doa_spectrum.argtypes = [vp, dp, dp, i64, fp, i32p, vp]
    L.doa_peaks.argtypes = [vp, i64, i32p, fp, i32p, i32p, vp]
    L.doa_run.argtypes = [vp, fp, i64, i64, i32p, fp, i32p, fp, i32p, vp]
    L.doa_run_host.argtypes = [C.POINTER(C.c_void_p), i32, fp, i64, i64, i32p, fp, i32p, i32p, vp]
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
    B, N = X.shape[0], X.shape[1]
    per_frame = 1 if theta_deg.dim() == 2 else 0
    _check(lib.doa_generate(M, d_over_lambda, D, _ptr(theta_deg), per_frame, snr_db, int(seed), frame0, B, N,
                            _ptr(_f32(X)), _stream(stream)))


def doa_plan_destroy(plan):
    _check(lib.doa_plan_destroy(plan))


def doa_covariance(plan, X, R, stream=None):
    """X: complex64 (B, N, M) CUDA tensor -> R: complex128 (B, M, M) CUDA tensor."""
    B, N = X.shape[0], X.shape[1]
    _check(lib.doa_covariance(plan, _ptr(_f32(X)), B, N, _ptr(_f64(R)), _stream(stream)))


def doa_eig(plan, R, lam, V, info, stream=None):
    _check(lib.doa_eig(plan, _ptr(_f64(R)), R.shape[0], _ptr(lam), _ptr(_f64(V)), _ptr(info), _stream(stream)))


def doa_spectrum(plan, lam, V, info, P=None, stream=None):
    _check(lib.doa_spectrum(plan, _ptr(lam), _ptr(_f64(V)), lam.shape[0], _ptr(P), _ptr(info), _stream(stream)))


def doa_peaks(plan, B, idx, val, npk, info, stream=None):
    _check(lib.doa_peaks(plan, B, _ptr(idx), _ptr(val), _ptr(npk), _ptr(info), _stream(stream)))


def doa_run(plan, X, idx, val, npk, info, P=None, stream=None):
    B, N = X.shape[0], X.shape[1]
    _check(lib.doa_run(plan, _ptr(_f32(X)), B, N, _ptr(idx), _ptr(val), _ptr(npk), _ptr(P), _ptr(info),
                       _stream(stream)))


def doa_run_host(plans, X_host, idx, val, npk, info, stream=None):
    """plans: one plan handle or a list sharing M, D.  Host (CPU) tensors in and out:
    idx/val (nplans, B, D), npk/info (nplans, B).  Pinned X_host gives overlapped async copies."""
    if not isinstance(plans, (list, tuple)):
        plans = [plans]
    arr = (C.c_void_p * len(plans))(*[p.value if isinstance(p, C.c_void_p) else p for p in plans])
    B, N = X_host.shape[0], X_host.shape[1]
    _check(lib.doa_run_host(arr, len(plans), _ptr(_f32(X_host)), B, N, _ptr(idx), _ptr(val), _ptr(npk),
                            _ptr(info), _stream(stream)))


def doa_last_launch_count() -> int:
    return int(lib.doa_last_launch_count())


# ----------------------------------------------------------------------------- convenience
class Plan:
    """Owns one doa_plan_t.  Methods allocate outputs with torch on the plan's device."""

    def __init__(self, M, D, alg, dtheta, L=None, theta0=-90.0, d_over_lambda=0.5, max_batch=1,
                 device="cuda"):
        if L is None:
            L = int(round((90.0 - theta0) / dtheta)) + 1
        self.M, self.D, self.alg, self.L, self.theta0, self.dtheta = M, D, alg, L, theta0, dtheta
        self.device = torch.device(device)
        self.max_batch = max_batch
        self.h = doa_plan_create(M, d_over_lambda, D, theta0, dtheta, L, alg, max_batch)
        self.cap = int(lib.doa_plan_capacity(self.h))

    @classmethod
    def array(cls, positions, D, alg, az0=0.0, daz=1.0, naz=360, el0=90.0, del_=1.0, nel=1, az_wrap=True,
              max_batch=1, device="cuda"):
        """General-geometry plan on an azimuth x elevation grid (doa_plan_create_array)."""
        self = cls.__new__(cls)
        M = len(positions)
        self.M, self.D, self.alg, self.L = M, D, alg, naz * nel
        self.naz, self.nel = naz, nel
        self.device = torch.device(device)
        self.max_batch = max_batch
        self.h = None
        self.h = doa_plan_create_array(M, positions, D, az0, daz, naz, el0, del_, nel, az_wrap, alg, max_batch)
        self.cap = int(lib.doa_plan_capacity(self.h))
        return self

    def close(self):
        if self.h is not None:
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
        doa_covariance(self.h, X, R, stream)
        return R

    def eig(self, R, stream=None):
        B = R.shape[0]
        lam = torch.empty((B, self.M), dtype=torch.float64, device=self.device)
        V = torch.empty((B, self.M, self.M), dtype=torch.complex128, device=self.device)
        info = torch.empty((B,), dtype=torch.int32, device=self.device)
        doa_eig(self.h, R, lam, V, info, stream)
        return lam, V, info

    def spectrum(self, lam, V, info=None, want_P=False, stream=None):
        B = lam.shape[0]
        if info is None:
            info = torch.zeros((B,), dtype=torch.int32, device=self.device)
        P = torch.empty((B, self.L), dtype=torch.float32, device=self.device) if want_P else None
        doa_spectrum(self.h, lam, V, info, P, stream)
        return P, info

    def peaks(self, B, info=None, stream=None):
        idx, val, npk, info0 = self._outs(B)
        info = info0 if info is None else info
        doa_peaks(self.h, B, idx, val, npk, info, stream)
        return idx, val, npk, info

    def run(self, X, want_P=False, stream=None):
        B = X.shape[0]
        idx, val, npk, info = self._outs(B)
        P = torch.empty((B, self.L), dtype=torch.float32, device=self.device) if want_P else None
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
        doa_run_host([p.h for p in plans], X_host, idx, val, npk, info, stream)
        if not others:
            return idx[0], val[0], npk[0], info[0]
        return idx, val, npk, info
