"""GPU parity at the north-star and C5 workloads in bench.py's launch configuration (full batch,
full grid), on sampled frames the oracle computes one by one.

* NS (the north-star target): c4's 65536 frames (M = 16, N = 256, D = 4, SNR 10)
  on the 0.001-degree grid, L = 180001.  Covariance + eig once for the whole batch, then spectrum
  + peaks per estimator, exactly as bench.py's step (`--workload ns`).  Frames b = 0 mod 1024 and
  the last one are checked for all four estimators: peak indices identical to the oracle's unless
  the oracle certifies a tie (Q18); the run's certified-tie count is recorded (tests/tiecert.py ->
  gpurun_out/parity_ties.json).  The scan's launch regime here differs from c4's (1452 angle
  columns, one frame chunk per column: each CTA streams all 8192 frame groups).
* C5 (BASELINE configs[4]): M = 64, D = 8 sources 1.5 deg apart (the smallest eigengap of any
  config), N = 4096, L = 180001, 8192 frames (16 GiB of snapshots) — generated on the device by
  doa_generate (NEXT-3, pinned element by element to its numpy twin in test_gpu_generate.py);
  frames b = 0 mod 512 and the last are copied back and given to the oracle as the same bytes.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as orc  # noqa: E402
from synth import get_config, generate  # noqa: E402
from tiecert import certify, delta_bound  # noqa: E402

ALGS = ["phd", "music", "ev", "mn"]


@pytest.fixture(scope="module")
def doa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2007_14135_b200 as d
    return d


def _bench_step(doa, cfg, Xd, B):
    """bench.py's step through the C ABI: S1-S2 once, S3-S7 per estimator; returns idx per alg."""
    base = doa.Plan(cfg.M, cfg.D, "music", cfg.dtheta, L=cfg.L, theta0=cfg.theta0, max_batch=B)
    R = base.covariance(Xd)
    lam, V, info0 = base.eig(R)
    del R
    out = {}
    for alg in ALGS:
        plan = doa.Plan(cfg.M, cfg.D, alg, cfg.dtheta, L=cfg.L, theta0=cfg.theta0, max_batch=B)
        info = info0.clone()
        plan.spectrum(lam, V, info)
        idx, val, npk, info = plan.peaks(B, info)
        out[alg] = (idx.cpu().numpy(), val.cpu().numpy(), npk.cpu().numpy(), info.cpu().numpy())
        plan.close()
    base.close()
    return out


def _check_sampled(cfg, Xs, sample, out, threads=16):
    """Peaks exact or certified (Q18); where identical, the peak values agree with the oracle's
    1/f within fp32 rounding plus the Q18 bound at that angle (two correct fp64 eigensolvers)."""
    for k, b in enumerate(sample):
        R = orc.covariance(Xs[k])
        ol, oV, _, oinfo = orc.eig(R)
        for alg in ALGS:
            f, _ = orc.spectrum(alg, cfg.D, cfg.d_over_lambda, ol, oV, cfg.theta0, cfg.dtheta, cfg.L,
                                threads=threads)
            oidx, ofv, onpk, _ = orc.peaks(f, cfg.D)
            idx, val, npk, info = (a[b] for a in out[alg])
            Cm, _ = orc.projector(alg, cfg.D, ol, oV)
            delta = delta_bound(alg, cfg.M, cfg.D, R, ol, Cm, f)
            ok, ties, why = certify(idx, oidx, f, delta, cfg.D)
            assert ok, f"{cfg.name} frame {b} {alg}: {why}"
            if np.array_equal(idx, oidx):
                n = int(onpk)
                assert npk == onpk
                rel = np.abs(val[:n].astype(np.float64) * ofv[:n] - 1.0)
                assert np.all(rel <= 1e-6 + delta[oidx[:n]]), (cfg.name, b, alg, rel, delta[oidx[:n]])


def test_ns_full_size_sampled(doa):
    cfg = get_config("ns")
    assert cfg.L == 180001 and cfg.B == 65536
    X = generate(cfg)
    out = _bench_step(doa, cfg, torch.from_numpy(X).cuda(), cfg.B)
    sample = list(range(0, cfg.B, 1024)) + [cfg.B - 1]
    _check_sampled(cfg, X[sample], sample, out)


def test_c5_full_size_sampled(doa):
    cfg = get_config("c5")
    assert cfg.M == 64 and cfg.L == 180001 and cfg.B == 8192 and cfg.N == 4096
    th = torch.tensor(cfg.sources, dtype=torch.float64, device="cuda")
    Xd = torch.empty((cfg.B, cfg.N, cfg.M), dtype=torch.complex64, device="cuda")
    doa.doa_generate(cfg.M, cfg.d_over_lambda, cfg.D, th, cfg.snr_db, cfg.seed, 0, Xd)
    sample = list(range(0, cfg.B, 512)) + [cfg.B - 1]
    Xs = Xd[sample].cpu().numpy()
    out = _bench_step(doa, cfg, Xd, cfg.B)
    del Xd
    _check_sampled(cfg, Xs, sample, out)
