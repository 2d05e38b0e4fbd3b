"""General-geometry (Eq. 2) snapshot generator and configurations — SURVEY §8(f) NEXT-1, the paper's
own workload: an 8-element uniform circular array (r = 10 m, 15 MHz carrier, 2 uncorrelated
sources, 15 dB SNR; §5) scanned over an azimuth x elevation grid
(360 x {1, 30, 60, 90}; Tables 8/10).

Steering (Eq. 2), positions in units of the wavelength:
    a_k(theta, phi) = exp{ j 2 pi (x_k sin(theta) sin(phi) + y_k cos(theta) sin(phi) + z_k cos(phi)) }
theta = azimuth, phi = "elevation" measured from +z (Eq. 2 carries z cos(phi); phi = 90 deg is the
array plane — the paper's naming, SPEC's reading).  Input generation only: no estimator
arithmetic lives here.
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Optional, Tuple

import numpy as np

C_LIGHT = 299_792_458.0


def uca_positions(M: int, radius_m: float, carrier_hz: float) -> np.ndarray:
    """(M, 3) element positions of a uniform circular array in the z = 0 plane, in wavelengths
    (element k at angle 2 pi k / M)."""
    lam = C_LIGHT / carrier_hz
    g = 2 * np.pi * np.arange(M) / M
    return np.stack([radius_m * np.cos(g), radius_m * np.sin(g), np.zeros(M)], axis=1) / lam


def steering_array(pos: np.ndarray, az_deg, el_deg) -> np.ndarray:
    """Eq. 2 for every (az, el) pair given (broadcast 1-D arrays of equal length): (M, n) complex128."""
    az = np.deg2rad(np.atleast_1d(np.asarray(az_deg, dtype=np.float64)))
    el = np.deg2rad(np.atleast_1d(np.asarray(el_deg, dtype=np.float64)))
    ux, uy, uz = np.sin(az) * np.sin(el), np.cos(az) * np.sin(el), np.cos(el)
    ph = 2 * np.pi * (np.outer(pos[:, 0], ux) + np.outer(pos[:, 1], uy) + np.outer(pos[:, 2], uz))
    return np.exp(1j * ph)


@dataclass(frozen=True)
class ArrayConfig:
    name: str
    positions: Tuple[Tuple[float, float, float], ...]   # wavelengths
    D: int
    N: int
    B: int
    snr_db: float
    seed: int
    sources: Tuple[Tuple[float, float], ...]            # (az, el) degrees
    az0: float = 0.0
    daz: float = 1.0
    naz: int = 360
    el0: float = 90.0
    del_: float = 1.0
    nel: int = 1
    az_wrap: bool = True

    @property
    def M(self) -> int:
        return len(self.positions)

    @property
    def pos(self) -> np.ndarray:
        return np.asarray(self.positions, dtype=np.float64)

    @property
    def L(self) -> int:
        return self.naz * self.nel

    def with_(self, **kw) -> "ArrayConfig":
        return replace(self, **kw)


def _uca8():
    return tuple(tuple(float(v) for v in row) for row in uca_positions(8, 10.0, 15e6))


# The paper's scenario (Figure 4 is missing from the text, so the two source directions are our
# choice, in the array plane): 8-element UCA, r = 10 m, 15 MHz, 2 sources, 15 dB.
ARRAY_CONFIGS = {
    # Table 5 grid: azimuth [0:1:359] x elevation [90]
    "e1": ArrayConfig("e1", positions=_uca8(), D=2, N=256, B=1, snr_db=15.0, seed=11,
                      sources=((37.0, 90.0), (152.0, 90.0)), naz=360, el0=90.0, nel=1),
    # Table 8/10 grid 360 x 90: azimuth [0:1:359] x elevation [1:1:90]
    "e1_360x90": ArrayConfig("e1_360x90", positions=_uca8(), D=2, N=256, B=1, snr_db=15.0, seed=11,
                             sources=((37.0, 90.0), (152.0, 90.0)), naz=360, el0=1.0, nel=90),
}


def _rng(seed: int, frame: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), 1 << 20, int(frame)])))


def generate_array(cfg: ArrayConfig, frames=None, noiseless: bool = False) -> np.ndarray:
    """X[b][n][m] complex64 for Eq. 1 with the Eq. 2 manifold; unit-power CN(0,1) sources,
    CN(0, sigma^2) noise, sigma^2 = 10^(-SNR/10); one PCG64 stream per frame."""
    frames = range(cfg.B) if frames is None else list(frames)
    src = np.asarray(cfg.sources, dtype=np.float64)
    A = steering_array(cfg.pos, src[:, 0], src[:, 1])          # (M, D)
    out = np.empty((len(frames), cfg.N, cfg.M), dtype=np.complex64)
    sigma = 0.0 if noiseless else np.sqrt(10.0 ** (-cfg.snr_db / 10.0))
    for i, f in enumerate(frames):
        rng = _rng(cfg.seed, f)
        D, N, M = len(src), cfg.N, cfg.M
        s = (rng.standard_normal((D, N)) + 1j * rng.standard_normal((D, N))) * np.sqrt(0.5)
        w = (rng.standard_normal((M, N)) + 1j * rng.standard_normal((M, N))) * (sigma * np.sqrt(0.5))
        out[i] = (A @ s + w).T.astype(np.complex64)
    return out
