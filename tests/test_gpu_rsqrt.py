"""The eigensolvers' reciprocal square root and reciprocal (csrc/eig16.cu rsqrt_pos / rcp_pos,
csrc/eign.cu rsqrt_p / rcp_p): a MUFU seed plus one third-order correction.  The rotation
parameters of every Jacobi round go through them, so an inaccurate result would make the applied
rotations slightly non-unitary and the error would accumulate over the ~116 rounds of a 16 x 16
solve.  tools/rsqrt_check.cu evaluates the same formulas on the device over 4M log-uniform
arguments in [2^-300, 2^300] against correctly rounded 1/sqrt(x) and 1/x: the seeds must be within
2^-19 (the correction leaves (5/16) e^3 < 2^-57) and the results within one ulp."""
import json
import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_rsqrt_rcp_one_ulp(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = str(tmp_path / "rsqrt_check")
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe,
                    os.path.join(ROOT, "tools", "rsqrt_check.cu")], check=True, capture_output=True)
    out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    r = json.loads(out.strip().splitlines()[-1])
    assert r["samples"] >= 1 << 22
    assert r["rsqrt_seed_max_rel"] < 2.0 ** -19 and r["rcp_seed_max_rel"] < 2.0 ** -19
    ulp = 2.0 ** -52                                       # relative spacing at the bottom of a binade
    assert r["rsqrt_max_rel"] <= ulp and r["rcp_max_rel"] <= ulp
