"""Benchmark / parity configurations.

Each entry instantiates one line of BASELINE.json `configs` (or the north-star
target) with the concrete choices recorded in SURVEY.md §8(d) and DESIGN.md §3
("input recipe").  All use a ULA with d/lambda = 0.5 and the scan grid
theta_i = theta0 + i*dtheta, i in [0, L), theta0 = -90 deg.
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Optional, Tuple

ALGS = ("phd", "music", "ev", "mn")


def grid_size(theta0: float, theta1: float, dtheta: float) -> int:
    """L = round((theta1 - theta0)/dtheta) + 1."""
    return int(round((theta1 - theta0) / dtheta)) + 1


@dataclass(frozen=True)
class Config:
    name: str
    M: int                      # sensors
    D: int                      # sources (assumed known)
    N: int                      # snapshots per frame
    B: int                      # frames per batch
    snr_db: float               # per element, per source
    seed: int
    dtheta: float               # grid step, degrees
    theta0: float = -90.0
    theta1: float = 90.0
    d_over_lambda: float = 0.5
    sources: Optional[Tuple[float, ...]] = None   # fixed DOAs (deg); None => random per frame
    rand_lo: float = -60.0      # random DOAs: U[lo, hi] with min separation
    rand_hi: float = 60.0
    rand_min_sep: float = 10.0
    algs: Tuple[str, ...] = ALGS

    @property
    def L(self) -> int:
        return grid_size(self.theta0, self.theta1, self.dtheta)

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


CONFIGS = {
    # BASELINE configs[0]: MUSIC, M=8, D=2 at -20/+35, N=100, SNR 10, 1 deg grid, single frame
    "c1": Config("c1", M=8, D=2, N=100, B=1, snr_db=10.0, seed=0, dtheta=1.0,
                 sources=(-20.0, 35.0)),
    # configs[1]: M=16, D=3, N=1024, 0.01 deg grid, single frame (SNR / angles: SURVEY §8(d) C2)
    "c2": Config("c2", M=16, D=3, N=1024, B=1, snr_db=10.0, seed=2, dtheta=0.01,
                 sources=(-20.0, 10.0, 45.0)),
    # configs[2]: C2's frame at dtheta in {0.1, 0.01, 0.001, 0.0001}
    "c3_0.1": Config("c3_0.1", M=16, D=3, N=1024, B=1, snr_db=10.0, seed=2, dtheta=0.1,
                     sources=(-20.0, 10.0, 45.0)),
    "c3_0.001": Config("c3_0.001", M=16, D=3, N=1024, B=1, snr_db=10.0, seed=2, dtheta=0.001,
                       sources=(-20.0, 10.0, 45.0)),
    "c3_0.0001": Config("c3_0.0001", M=16, D=3, N=1024, B=1, snr_db=10.0, seed=2, dtheta=0.0001,
                        sources=(-20.0, 10.0, 45.0)),
    # configs[3]: batched streaming 65536 x M=16 x N=256, D=4, 0.01 deg (the bench workload)
    "c4": Config("c4", M=16, D=4, N=256, B=65536, snr_db=10.0, seed=4, dtheta=0.01),
    # north-star target: C4's data on a 0.001 deg grid
    "ns": Config("ns", M=16, D=4, N=256, B=65536, snr_db=10.0, seed=4, dtheta=0.001),
    # configs[4]: M=64, D=8 closely spaced (1.5 deg), N=4096, 0.001 deg, 8192 frames
    "c5": Config("c5", M=64, D=8, N=4096, B=8192, snr_db=10.0, seed=5, dtheta=0.001,
                 sources=tuple(10.0 + 1.5 * k for k in range(8))),
}


def get_config(name: str, **overrides) -> Config:
    cfg = CONFIGS[name]
    return cfg.with_(**overrides) if overrides else cfg
