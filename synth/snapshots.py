"""Seeded snapshot generator for the paper's signal model.

X(t) = A(theta) S(t) + W(t)                      (Eq. 1, §3.1)
  - S: D uncorrelated narrowband sources, i.i.d. circular CN(0, 1)
  - W: zero-mean complex white Gaussian noise CN(0, sigma^2), sigma^2 = 10^(-SNR/10)
       (per element, per unit-power source)
  - A(theta): ULA special case of the steering vector of Eq. 2 in the north-star
       convention a_m(theta) = exp(-j*2*pi*(d/lambda)*m*sin(theta)), m = 0..M-1.

One independent PCG64 stream per frame, keyed by SeedSequence([seed, frame]), so any
contiguous shard of frames (one per GPU rank) regenerates bit-identical data.  Draw order
per frame: (random-DOA configs only) the D angles by rejection sampling; then Re S, Im S
(D x N standard normals each); then Re W, Im W (M x N each).  X is formed in float64 and
rounded once to complex64, stored snapshot-major as X[b][n][m] (the layout the C-ABI takes).

This module is input generation only: it contains none of the estimator's arithmetic.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .configs import Config


def steering_ula(theta_deg, M: int, d_over_lambda: float) -> np.ndarray:
    """Array manifold A(theta) of the signal model, shape (M, len(theta)), complex128."""
    th = np.atleast_1d(np.asarray(theta_deg, dtype=np.float64))
    m = np.arange(M, dtype=np.float64)[:, None]
    phase = -2.0 * np.pi * d_over_lambda * m * np.sin(np.deg2rad(th))[None, :]
    return np.exp(1j * phase)


def _rng(seed: int, frame: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), int(frame)])))


def _draw_angles(rng: np.random.Generator, cfg: Config) -> np.ndarray:
    while True:
        th = np.sort(rng.uniform(cfg.rand_lo, cfg.rand_hi, size=cfg.D))
        if cfg.D == 1 or np.min(np.diff(th)) >= cfg.rand_min_sep:
            return th


def frame_angles(cfg: Config, frame: int) -> np.ndarray:
    """The true DOAs (degrees, ascending) used for frame `frame`."""
    if cfg.sources is not None:
        return np.asarray(cfg.sources, dtype=np.float64)
    return _draw_angles(_rng(cfg.seed, frame), cfg)


def _one_frame(cfg: Config, frame: int, out: np.ndarray) -> None:
    rng = _rng(cfg.seed, frame)
    if cfg.sources is not None:
        th = np.asarray(cfg.sources, dtype=np.float64)
    else:
        th = _draw_angles(rng, cfg)
    D, N, M = len(th), cfg.N, cfg.M
    s = (rng.standard_normal((D, N)) + 1j * rng.standard_normal((D, N))) * np.sqrt(0.5)
    sigma = np.sqrt(10.0 ** (-cfg.snr_db / 10.0))
    w = (rng.standard_normal((M, N)) + 1j * rng.standard_normal((M, N))) * (sigma * np.sqrt(0.5))
    x = steering_ula(th, M, cfg.d_over_lambda) @ s + w          # (M, N) complex128
    out[:, :] = x.T.astype(np.complex64)                         # [n][m]


def generate(cfg: Config, frames=None, threads: int | None = None, noiseless: bool = False) -> np.ndarray:
    """Return X[b][n][m] complex64 for the given global frame indices (default: all cfg.B).

    `noiseless=True` drops W ("noiseless flag"), used by closed-form pins.
    """
    if frames is None:
        frames = range(cfg.B)
    frames = list(frames)
    out = np.empty((len(frames), cfg.N, cfg.M), dtype=np.complex64)
    if noiseless:
        c = cfg.with_(snr_db=float("inf"))
        for i, f in enumerate(frames):
            _one_frame(c, f, out[i])
        return out
    nproc = threads or min(64, os.cpu_count() or 1)
    if len(frames) < 512 or nproc <= 1:
        for i, f in enumerate(frames):
            _one_frame(cfg, f, out[i])
        return out
    # numpy's per-frame work is small and GIL-bound: fan out over forked processes that
    # write straight into a shared buffer (each frame's bytes depend only on (seed, frame)).
    import multiprocessing as mp
    from multiprocessing import shared_memory
    shm = shared_memory.SharedMemory(create=True, size=out.nbytes)
    try:
        chunks = [c for c in np.array_split(np.arange(len(frames)), nproc * 4) if len(c)]
        ctx = mp.get_context("fork")
        procs = []
        per = (len(chunks) + nproc - 1) // nproc
        for p in range(nproc):
            mine = chunks[p * per:(p + 1) * per]
            if not mine:
                continue
            pr = ctx.Process(target=_worker, args=(shm.name, out.shape, cfg, frames, mine))
            pr.start()
            procs.append(pr)
        for pr in procs:
            pr.join()
            if pr.exitcode != 0:
                raise RuntimeError(f"snapshot generator worker failed (exit {pr.exitcode})")
        out[...] = np.ndarray(out.shape, dtype=np.complex64, buffer=shm.buf)
    finally:
        shm.close()
        shm.unlink()
    return out


def _worker(name, shape, cfg, frames, chunks):
    from multiprocessing import shared_memory
    shm = shared_memory.SharedMemory(name=name)
    try:
        buf = np.ndarray(shape, dtype=np.complex64, buffer=shm.buf)
        for idx in chunks:
            for i in idx:
                _one_frame(cfg, frames[i], buf[i])
    finally:
        del buf
        shm.close()
