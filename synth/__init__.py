"""Seeded synthetic snapshot generator shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the estimation method (no covariance, no
eigensolver, no spectrum, no peak rule).  It only draws array snapshots from the
paper's signal model (Eq. 1, §3.1 "Signal Data Model") and
describes the benchmark configurations (BASELINE.json `configs`).
"""
from .configs import CONFIGS, Config, grid_size, get_config
from .snapshots import generate, frame_angles, steering_ula

__all__ = ["CONFIGS", "Config", "grid_size", "get_config", "generate", "frame_angles", "steering_ula"]
