"""NEXT-3: libdoa's on-device Eq. 1 generator (doa_generate) against the same counter-based
generator in numpy (synth/philox.py), element by element, and the hot path on device-generated
frames against the oracle on the same bytes."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as orc  # noqa: E402
from synth import philox  # noqa: E402
from tiecert import certify, delta_bound, max_db_error  # noqa: E402


@pytest.fixture(scope="module")
def doa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2007_14135_b200 as d
    return d


@pytest.mark.parametrize("M,D,N,snr,per_frame", [(16, 4, 256, 10.0, True), (8, 2, 100, 10.0, False),
                                                 (64, 8, 300, 0.0, False), (5, 3, 33, 30.0, True)])
def test_generate_matches_numpy_philox(doa, M, D, N, snr, per_frame):
    B, seed, frame0 = 7, 0x1234_5678_9ABC, 1_000_003
    rng = np.random.default_rng(M)
    th = rng.uniform(-60, 60, size=(B, D)) if per_frame else np.linspace(-40, 40, D)
    X = torch.empty((B, N, M), dtype=torch.complex64, device="cuda")
    doa.doa_generate(M, 0.5, D, torch.from_numpy(np.ascontiguousarray(th)).cuda(), snr, seed, frame0, X)
    g = X.cpu().numpy()
    ref = philox.generate(M, 0.5, D, th, snr, seed, range(frame0, frame0 + B), N)
    scale = np.max(np.abs(ref))
    # fp64 on both sides (libm vs CUDA log/sincospi differ in the last bits), one rounding to fp32
    assert np.max(np.abs(g - ref)) <= 4e-7 * scale
    assert np.mean(g == ref) > 0.9


def test_generate_is_batch_and_offset_invariant(doa):
    M, D, N = 16, 4, 64
    th = torch.tensor([-20.0, 0.0, 15.0, 40.0], dtype=torch.float64, device="cuda")
    a = torch.empty((10, N, M), dtype=torch.complex64, device="cuda")
    b = torch.empty((3, N, M), dtype=torch.complex64, device="cuda")
    doa.doa_generate(M, 0.5, D, th, 10.0, 42, 100, a)
    doa.doa_generate(M, 0.5, D, th, 10.0, 42, 105, b)
    assert torch.equal(a[5:8], b)


@pytest.mark.parametrize("alg", ["phd", "music", "ev", "mn"])
def test_hot_path_on_device_generated_frames(doa, alg):
    """c4-shaped frames generated on the device, estimated on the device, checked against the
    oracle on the same complex64 bytes (peaks exact or certified, Q18; P within 1e-3 dB, Q17)."""
    M, D, N, B, dth = 16, 4, 256, 24, 0.05
    L = int(round(180 / dth)) + 1
    rng = np.random.default_rng(4)
    th = np.sort(rng.uniform(-60, 60, size=(B, D)), axis=1)
    X = torch.empty((B, N, M), dtype=torch.complex64, device="cuda")
    doa.doa_generate(M, 0.5, D, torch.from_numpy(th).cuda(), 10.0, 2026, 0, X)
    plan = doa.Plan(M, D, alg, dth, L=L, max_batch=B)
    idx, val, npk, info, P = plan.run(X, want_P=True)
    idx, P, Xh = idx.cpu().numpy(), P.cpu().numpy(), X.cpu().numpy()
    for b in range(B):
        R = orc.covariance(Xh[b])
        lam, V, _, _ = orc.eig(R)
        f, _ = orc.spectrum(alg, D, 0.5, lam, V, -90.0, dth, L, threads=8)
        Cm, _ = orc.projector(alg, D, lam, V)
        oidx = orc.peaks(f, D)[0]
        ok, ties, why = certify(idx[b], oidx, f, delta_bound(alg, M, D, R, lam, Cm, f), D)
        assert ok, f"frame {b} {alg}: {why}"
        assert max_db_error(P[b], 1.0 / f) <= 1e-3
    plan.close()


def test_generate_rejects_bad_arguments(doa):
    X = torch.empty((2, 8, 4), dtype=torch.complex64, device="cuda")
    th = torch.zeros(2, dtype=torch.float64, device="cuda")
    with pytest.raises(doa.DoaError):
        doa.doa_generate(4, 0.5, 0, th, 10.0, 1, 0, X)              # D = 0
    with pytest.raises(doa.DoaError):
        doa.doa_generate(4, -0.5, 2, th, 10.0, 1, 0, X)             # d/lambda <= 0
