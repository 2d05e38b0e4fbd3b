"""Pins for oracle.peaks — Table 2 Step-6 findPeaks + PeakSelection under the
readings SURVEY Q9-Q11.  Hand-derived golden cases (tests/golden/peak_rule_cases.txt) and an
independent library cross-check (scipy.signal.find_peaks on -f, for tie-free random data).
"""
import os

import numpy as np
import pytest
from scipy.signal import find_peaks


def _cases():
    path = os.path.join(os.path.dirname(__file__), "golden", "peak_rule_cases.txt")
    out = []
    with open(path) as fh:
        for line in fh:
            if not line.strip() or line.startswith("#"):
                continue
            D, f, idx, npk = [s.strip() for s in line.split("|")]
            out.append((int(D), [float(x) for x in f.split()], [int(x) for x in idx.split()], int(npk)))
    return out


@pytest.mark.parametrize("D,f,idx,npk", _cases())
def test_golden_cases(orc, D, f, idx, npk):
    got_idx, got_f, got_n, _ = orc.peaks(np.array(f), D)
    assert got_idx.tolist() == idx
    assert got_n == npk
    for k in range(npk):
        assert got_f[k] == f[idx[k]]


@pytest.mark.parametrize("seed", range(30))
def test_scipy_cross_check(orc, seed):
    rng = np.random.default_rng(seed)
    L = int(rng.integers(3, 400))
    f = rng.random(L) + 0.01                      # continuous: no ties almost surely
    D = int(rng.integers(1, 10))
    pk, _ = find_peaks(-f)                         # strict interior local maxima of -f
    order = sorted(pk.tolist(), key=lambda i: (f[i], i))
    exp = order[:D] + [-1] * max(0, D - len(order))
    idx, fv, npk, n = orc.peaks(f, D)
    assert n == len(pk)
    assert idx.tolist() == exp
    assert npk == min(D, len(pk))
