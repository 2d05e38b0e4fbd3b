"""Counter-based Eq. 1 snapshot generator (Philox4x32-10 + fp64 Box-Muller) in numpy — the same
generator as libdoa's doa_generate (csrc/generate.cu), used to check the device generator element
by element.  Input generation only (shared by tests of both sides); none of the estimator's
arithmetic is here.

Sample k of snapshot n of frame f (k < D: source k, else the noise of element k - D) comes from
Philox call (counter = (k//2, n, f mod 2^32, f >> 32), key = (seed mod 2^32, seed >> 32)), words
(2(k%2), 2(k%2)+1) -> u = (w + 0.5) 2^-32 -> z = sqrt(-2 ln u1) e^{j 2 pi u2} / sqrt(2).
X = A(theta) S + sigma W, a_m = exp(-j pi m u), u = 2 (d/lambda) sin theta, sigma^2 = 10^(-SNR/10)
(Eq. 1; Q6, Q13, Q14); fp64, rounded once to complex64, layout [B][N][M].
"""
from __future__ import annotations

import numpy as np

_M0, _M1, _W0, _W1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85
_MASK = 0xFFFFFFFF


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 on uint64 arrays holding 32-bit values; returns 4 arrays."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) & _MASK for c in (c0, c1, c2, c3))
    k0 = np.uint64(k0 & _MASK)
    k1 = np.uint64(k1 & _MASK)
    for _ in range(10):
        p0 = np.uint64(_M0) * c0
        p1 = np.uint64(_M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & np.uint64(_MASK)
        hi1, lo1 = p1 >> np.uint64(32), p1 & np.uint64(_MASK)
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0), lo1, (hi0 ^ c3 ^ k1), lo0
        k0 = (k0 + np.uint64(_W0)) & np.uint64(_MASK)
        k1 = (k1 + np.uint64(_W1)) & np.uint64(_MASK)
    return c0, c1, c2, c3


def _cnormal(a, b):
    u1 = (a.astype(np.float64) + 0.5) * 2.0 ** -32
    u2 = (b.astype(np.float64) + 0.5) * 2.0 ** -32
    r = np.sqrt(-2.0 * np.log(u1)) * 0.70710678118654752440
    ang = np.pi * (2.0 * u2)
    return r * np.cos(ang) + 1j * r * np.sin(ang)


def samples(D: int, M: int, seed: int, frames, N: int) -> np.ndarray:
    """CN(0,1) draws [B][N][D+M] (sources first, then per-element noise)."""
    frames = np.asarray(list(frames), dtype=np.uint64)
    B = frames.size
    K = D + M
    k = np.arange(K, dtype=np.uint64)
    n = np.arange(N, dtype=np.uint64)
    f = frames[:, None, None]
    c0 = np.broadcast_to((k // np.uint64(2))[None, None, :], (B, N, K))
    c1 = np.broadcast_to(n[None, :, None], (B, N, K))
    c2 = np.broadcast_to(f & np.uint64(_MASK), (B, N, K))
    c3 = np.broadcast_to(f >> np.uint64(32), (B, N, K))
    w0, w1, w2, w3 = philox4x32_10(c0, c1, c2, c3, seed & _MASK, seed >> 32)
    odd = (k % np.uint64(2)).astype(bool)[None, None, :]
    a = np.where(odd, w2, w0)
    b = np.where(odd, w3, w1)
    return _cnormal(a, b)


def generate(M: int, d_over_lambda: float, D: int, theta_deg, snr_db: float, seed: int, frames, N: int) -> np.ndarray:
    """X complex64 [B][N][M]; theta_deg: (D,) for every frame or (B, D)."""
    frames = list(frames)
    z = samples(D, M, seed, frames, N)
    S, W = z[..., :D], z[..., D:]
    th = np.asarray(theta_deg, dtype=np.float64)
    th = np.broadcast_to(th if th.ndim == 2 else th[None, :], (len(frames), D))
    u = 2.0 * d_over_lambda * np.sin(np.deg2rad(th))                     # [B][D]
    m = np.arange(M, dtype=np.float64)
    A = np.exp(-1j * np.pi * m[None, :, None] * u[:, None, :])          # [B][M][D]
    sigma = np.sqrt(10.0 ** (-snr_db / 10.0))
    X = np.einsum("bmd,bnd->bnm", A, S) + sigma * W
    return X.astype(np.complex64)
