"""SURVEY §8(f) NEXT-2 evidence: the fp32 direct-form scan (tools/fp32_direct/fp32_direct.cu) versus
the product's fp64 Toeplitz DMMA scan, on (a) speed at c4 (65536 frames x 18001 angles, MUSIC) and
(b) parity against the fp64 oracle on c2's frame at 0.01 and 0.001 deg for all four estimators
(max |dB| error after normalisation, Q17, and top-D index agreement).  Comparison code only.

    python tools/fp32_direct_eval.py > profiles/fp32_direct_r01.json
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SRC = os.path.join(ROOT, "tools", "fp32_direct", "fp32_direct.cu")
LIB = os.path.join(ROOT, "tools", "fp32_direct", "libfp32_direct.so")


def build():
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                        "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-o", LIB, SRC],
                       check=True)
    L = C.CDLL(LIB)
    L.fp32_direct_scan.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                   C.c_int64, C.c_int, C.c_void_p, C.c_void_p]
    return L


def noise_vectors(alg, lam, V, D):
    """w_k^(1/2) e_k for the direct form (Table 3 Step-3; EV 1/lambda, MN normalised w)."""
    import numpy as np
    M = V.shape[-1]
    K = M - D
    if alg == "phd":
        return V[..., :, :1].transpose(0, 2, 1)
    if alg == "music":
        return V[..., :, :K].transpose(0, 2, 1)
    if alg == "ev":
        return (V[..., :, :K] / np.sqrt(lam[..., None, :K])).transpose(0, 2, 1)
    En = V[..., :, :K]
    p = En @ np.conj(En[..., :1, :]).transpose(0, 2, 1)          # P_n e1
    p0 = np.sum(np.abs(En[..., 0, :]) ** 2, axis=-1)
    return (p / p0[:, None, None]).transpose(0, 2, 1)


def main():
    import numpy as np
    import torch

    import oracle
    import paper_2007_14135_b200 as doa
    from synth import get_config, generate
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from tiecert import max_db_error
    lib = build()
    out = {"what": "fp32 direct-form scan (north-star's FP32-pipe option) vs fp64 Toeplitz DMMA scan"}
    dev = torch.device("cuda")
    # ---- (a) speed on c4 (MUSIC)
    cfg = get_config("c4")
    X = torch.from_numpy(generate(cfg)).to(dev)
    plan = doa.Plan(cfg.M, cfg.D, "music", cfg.dtheta, max_batch=cfg.B)
    R = plan.covariance(X)
    lam, V, info = plan.eig(R)
    U = noise_vectors("music", lam.cpu().numpy(), V.cpu().numpy(), cfg.D).astype(np.complex64)
    Ud = torch.from_numpy(np.ascontiguousarray(U)).to(dev)
    F = torch.empty((cfg.B, cfg.L), dtype=torch.float32, device=dev)
    s = torch.cuda.current_stream().cuda_stream

    def t(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best

    ms_direct = t(lambda: lib.fp32_direct_scan(Ud.data_ptr(), cfg.B, U.shape[1], cfg.M, -90.0, cfg.dtheta, 0.5,
                                               cfg.L, 1, F.data_ptr(), s))
    ms_ours = t(lambda: plan.spectrum(lam, V))
    out["c4_music_ms"] = {"fp32_direct (writes f, no peak search)": ms_direct,
                          "fp64 Toeplitz DMMA doa_spectrum (coef + scan + peaks)": ms_ours,
                          "speedup_of_product": ms_direct / ms_ours}
    del F
    # ---- (b) parity on c2's frame
    par = {}
    for dth in (0.01, 0.001):
        c = get_config("c2").with_(dtheta=dth)
        Xh = generate(c)[0]
        ol, oV, _, _ = oracle.eig(oracle.covariance(Xh))
        for alg in ("phd", "music", "ev", "mn"):
            f, _ = oracle.spectrum(alg, c.D, 0.5, ol, oV, -90.0, dth, c.L, threads=8)
            oidx = oracle.peaks(f, c.D)[0]
            Uo = noise_vectors(alg, ol[None], oV[None], c.D).astype(np.complex64)   # best case: fp64 subspace
            Fd = torch.empty((1, c.L), dtype=torch.float32, device=dev)
            lib.fp32_direct_scan(torch.from_numpy(np.ascontiguousarray(Uo)).to(dev).data_ptr(), 1, Uo.shape[1],
                                 c.M, -90.0, dth, 0.5, c.L, 1, Fd.data_ptr(), s)
            torch.cuda.synchronize()
            fd = np.maximum(Fd.cpu().numpy()[0].astype(np.float64), 1e-300)
            gidx = oracle.peaks(fd, c.D)[0]
            par[f"{alg}@{dth}"] = {"max_db_err": max_db_error(1.0 / fd, 1.0 / f),
                                   "peaks_equal": bool(np.array_equal(gidx, oidx))}
            # the product path on the same frame
            p = doa.Plan(c.M, c.D, alg, dth, max_batch=1)
            idx, val, npk, inf, P = p.run(torch.from_numpy(Xh[None]).to(dev), want_P=True)
            par[f"{alg}@{dth}"]["product_max_db_err"] = max_db_error(P.cpu().numpy()[0], 1.0 / f)
            par[f"{alg}@{dth}"]["product_peaks_equal"] = bool(np.array_equal(idx.cpu().numpy()[0], oidx))
    out["parity_c2"] = par
    print(json.dumps(out))


if __name__ == "__main__":
    main()
