"""ORACLE — test infrastructure only (see oracle/oracle.cpp header).

ctypes wrapper around liboracle.so, the plain fp64 CPU reference of the DOA hot path.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference legs may import
this package.  It never imports the product package and the product never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

ALG = {"phd": 0, "music": 1, "ev": 2, "mn": 3}
INFO_NOCONV, INFO_DEGENERATE, INFO_UNDERDETERMINED = 1, 2, 8


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (plain -O2, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               "-pthread", "-o", _LIB + ".tmp", _SRC]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            dp, fp, ip, i32p = (C.POINTER(C.c_double), C.POINTER(C.c_float), C.POINTER(C.c_int),
                                C.POINTER(C.c_int32))
            L.oracle_covariance.argtypes = [fp, C.c_int64, C.c_int, dp]
            L.oracle_covariance.restype = None
            L.oracle_eig.argtypes = [dp, C.c_int, dp, dp, ip]
            L.oracle_eig.restype = C.c_int
            L.oracle_projector.argtypes = [C.c_int, C.c_int, C.c_int, dp, dp, dp, ip]
            L.oracle_projector.restype = None
            L.oracle_spectrum.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, dp, dp, C.c_double,
                                          C.c_double, C.c_int64, dp, C.c_int, ip]
            L.oracle_spectrum.restype = None
            L.oracle_peaks.argtypes = [dp, C.c_int64, C.c_int, i32p, dp, i32p]
            L.oracle_peaks.restype = C.c_int64
            L.oracle_run_batch.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                           C.c_int64, fp, C.c_int64, C.c_int64, i32p, fp, i32p, i32p, i32p,
                                           fp, C.c_int]
            L.oracle_run_batch.restype = None
            L.oracle_spectrum_array.argtypes = [C.c_int, C.c_int, C.c_int, dp, dp, dp, C.c_double, C.c_double,
                                                C.c_int64, C.c_double, C.c_double, C.c_int64, dp, C.c_int, ip]
            L.oracle_spectrum_array.restype = None
            L.oracle_peaks2d.argtypes = [dp, C.c_int64, C.c_int64, C.c_int, C.c_int, i32p, dp, i32p]
            L.oracle_peaks2d.restype = C.c_int64
            L.oracle_run_array_batch.argtypes = [C.c_int, C.c_int, C.c_int, dp, C.c_double, C.c_double, C.c_int64,
                                                 C.c_double, C.c_double, C.c_int64, C.c_int, fp, C.c_int64,
                                                 C.c_int64, i32p, fp, i32p, i32p, fp, C.c_int]
            L.oracle_run_array_batch.restype = None
            _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def covariance(X: np.ndarray) -> np.ndarray:
    """X[N][M] complex64 -> R[M][M] complex128 (Eq. 3)."""
    X = np.ascontiguousarray(X, dtype=np.complex64)
    N, M = X.shape
    R = np.empty((M, M), dtype=np.complex128)
    lib().oracle_covariance(_p(X.view(np.float32), C.c_float), N, M, _p(R.view(np.float64), C.c_double))
    return R


def eig(R: np.ndarray):
    """R[M][M] -> (lambda[M] ascending, V[M][M] (column j = eigvec j), sweeps, info)."""
    R = _c128(R)
    M = R.shape[0]
    lam = np.empty(M)
    V = np.empty((M, M), dtype=np.complex128)
    info = C.c_int(0)
    sw = lib().oracle_eig(_p(R.view(np.float64), C.c_double), M, _p(lam, C.c_double),
                          _p(V.view(np.float64), C.c_double), C.byref(info))
    return lam, V, sw, info.value


def projector(alg: str, D: int, lam: np.ndarray, V: np.ndarray):
    """Table 3 Step-4 matrix C -> (C[M][M], info)."""
    V = _c128(V)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    M = V.shape[0]
    Cm = np.empty((M, M), dtype=np.complex128)
    info = C.c_int(0)
    lib().oracle_projector(ALG[alg], M, D, _p(lam, C.c_double), _p(V.view(np.float64), C.c_double),
                           _p(Cm.view(np.float64), C.c_double), C.byref(info))
    return Cm, info.value


def spectrum(alg: str, D: int, d_over_lambda: float, lam, V, theta0: float, dtheta: float, L: int,
             threads: int = 1):
    """Floored quadratic form f_c[L] (P = 1/f_c) -> (f, info)."""
    V = _c128(V)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    M = V.shape[0]
    f = np.empty(L)
    info = C.c_int(0)
    lib().oracle_spectrum(ALG[alg], M, D, d_over_lambda, _p(lam, C.c_double), _p(V.view(np.float64), C.c_double),
                          theta0, dtheta, L, _p(f, C.c_double), threads, C.byref(info))
    return f, info.value


def peaks(f: np.ndarray, D: int):
    """findPeaks + PeakSelection -> (idx[D] (-1 pad), fval[D], npk, n_candidates)."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    idx = np.empty(D, dtype=np.int32)
    fv = np.empty(D)
    npk = C.c_int32(0)
    n = lib().oracle_peaks(_p(f, C.c_double), len(f), D, _p(idx, C.c_int32), _p(fv, C.c_double), C.byref(npk))
    return idx, fv, npk.value, n


def run_batch(alg: str, X: np.ndarray, D: int, d_over_lambda: float, theta0: float, dtheta: float, L: int,
              threads: int = 1, want_P: bool = False):
    """Whole path for X[B][N][M] -> dict(idx[B][D], val[B][D] f32, npk[B], info[B], sweeps[B], P[B][L]|None)."""
    X = np.ascontiguousarray(X, dtype=np.complex64)
    B, N, M = X.shape
    idx = np.empty((B, D), dtype=np.int32)
    val = np.empty((B, D), dtype=np.float32)
    npk = np.empty(B, dtype=np.int32)
    info = np.empty(B, dtype=np.int32)
    sweeps = np.empty(B, dtype=np.int32)
    P = np.empty((B, L), dtype=np.float32) if want_P else None
    lib().oracle_run_batch(ALG[alg], M, D, d_over_lambda, theta0, dtheta, L, _p(X.view(np.float32), C.c_float),
                           B, N, _p(idx, C.c_int32), _p(val, C.c_float), _p(npk, C.c_int32), _p(info, C.c_int32),
                           _p(sweeps, C.c_int32), _p(P, C.c_float) if want_P else None, threads)
    return dict(idx=idx, val=val, npk=npk, info=info, sweeps=sweeps, P=P)


# ---------------------------------------------------------------------------- NEXT-1: general arrays
def spectrum_array(alg: str, D: int, pos, lam, V, az0, daz, naz, el0, del_, nel, threads: int = 1):
    """Eq. 2 steering for element positions pos[M][3] (wavelengths) over the azimuth-major
    az x el grid -> (f[naz*nel], info)."""
    V = _c128(V)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
    M = V.shape[0]
    f = np.empty(naz * nel)
    info = C.c_int(0)
    lib().oracle_spectrum_array(ALG[alg], M, D, _p(pos, C.c_double), _p(lam, C.c_double),
                                _p(V.view(np.float64), C.c_double), az0, daz, naz, el0, del_, nel,
                                _p(f, C.c_double), threads, C.byref(info))
    return f, info.value


def peaks2d(f, naz: int, nel: int, wrap: bool, D: int):
    """2-D findPeaks (8-neighbourhood, raster tie rule, optional azimuth wrap) + PeakSelection
    -> (idx[D] raster indices (-1 pad), fval[D], npk, n_candidates)."""
    f = np.ascontiguousarray(f, dtype=np.float64).reshape(-1)
    idx = np.empty(D, dtype=np.int32)
    fv = np.empty(D)
    npk = C.c_int32(0)
    n = lib().oracle_peaks2d(_p(f, C.c_double), naz, nel, int(bool(wrap)), D, _p(idx, C.c_int32),
                             _p(fv, C.c_double), C.byref(npk))
    return idx, fv, npk.value, n


def run_array_batch(alg: str, X, D: int, pos, az0, daz, naz, el0, del_, nel, wrap: bool, threads: int = 1,
                    want_P: bool = False):
    X = np.ascontiguousarray(X, dtype=np.complex64)
    B, N, M = X.shape
    pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
    L = naz * nel
    idx = np.empty((B, D), dtype=np.int32)
    val = np.empty((B, D), dtype=np.float32)
    npk = np.empty(B, dtype=np.int32)
    info = np.empty(B, dtype=np.int32)
    P = np.empty((B, L), dtype=np.float32) if want_P else None
    lib().oracle_run_array_batch(ALG[alg], M, D, _p(pos, C.c_double), az0, daz, naz, el0, del_, nel,
                                 int(bool(wrap)), _p(X.view(np.float32), C.c_float), B, N, _p(idx, C.c_int32),
                                 _p(val, C.c_float), _p(npk, C.c_int32), _p(info, C.c_int32),
                                 _p(P, C.c_float) if want_P else None, threads)
    return dict(idx=idx, val=val, npk=npk, info=info, P=P)
