"""B200-native noise-subspace DOA estimation hot path (Eray & Temizel, arXiv 2007.14135).

The product is libdoa.so (CUDA, sm_100a) behind the C ABI in include/doa.h; this package is its
ctypes binding (binding.py) plus the frame-sharding driver for several GPUs (dist.py).
"""
from .binding import (ALG, ENGINE, INFO_CAND_OVERFLOW, INFO_DEGENERATE, INFO_NOCONV, INFO_UNDERDETERMINED, DoaError,
                      Plan, doa_covariance, doa_eig, doa_generate, doa_last_launch_count, doa_peaks, doa_plan_create,
                      doa_plan_set_engine,
                      doa_plan_destroy, doa_run, doa_run_host, doa_run_multi, doa_scan_multi, doa_spectrum, lib,
                      run_multi)

__all__ = ["ALG", "ENGINE", "doa_plan_set_engine", "INFO_CAND_OVERFLOW", "INFO_DEGENERATE", "INFO_NOCONV", "INFO_UNDERDETERMINED", "DoaError",
           "Plan", "doa_covariance", "doa_eig", "doa_generate", "doa_last_launch_count", "doa_peaks", "doa_plan_create",
           "doa_plan_destroy", "doa_run", "doa_run_host", "doa_run_multi", "doa_scan_multi", "doa_spectrum", "lib",
           "run_multi"]
