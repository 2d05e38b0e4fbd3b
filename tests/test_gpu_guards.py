"""GPU parity of the guard branches and of the binding's argument checks.

* Q12 (floor + fp32 saturation): an exact null injected through doa_spectrum must give
  P = FLT_MAX and a peak value FLT_MAX, like the oracle (pinned in test_oracle_spectrum.py).
* G1 (degenerate EV / MN): injected eigenpairs that hit the clamp / the unnormalised MN vector
  must give the oracle's spectrum element by element and the same DEGENERATE flags.
* Absolute P (not only normalised dB) for M up to 64 with K = M - D > 32 noise vectors — the MN
  normalisation p0 sums all K vectors.
* The Python binding rejects tensors whose shape, dtype or device does not match the plan
  (ValueError) before anything reaches the C ABI.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as orc  # noqa: E402
from synth import get_config, generate  # noqa: E402
from tiecert import certify, delta_bound  # noqa: E402

ALGS = ["phd", "music", "ev", "mn"]
FMAX = np.finfo(np.float32).max


@pytest.fixture(scope="module")
def doa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2007_14135_b200 as d
    return d


def _inject(doa, alg, D, lam, V, theta0=-90.0, dtheta=1.0, L=181):
    M = V.shape[0]
    plan = doa.Plan(M, D, alg, dtheta, L=L, theta0=theta0, max_batch=1)
    lt = torch.from_numpy(np.ascontiguousarray(lam, dtype=np.float64)[None].copy()).cuda()
    Vt = torch.from_numpy(np.ascontiguousarray(V, dtype=np.complex128)[None].copy()).cuda()
    P, info = plan.spectrum(lt, Vt, want_P=True)
    idx, val, npk, info = plan.peaks(1, info)
    out = [t.cpu().numpy()[0] for t in (P, idx, val, npk, info)]
    plan.close()
    return out


def _v3(cols):
    return np.ascontiguousarray(np.array(cols, dtype=np.complex128).T)


@pytest.mark.parametrize("alg", ["phd", "music"])
def test_exact_null_saturates_like_oracle(doa, alg):
    c = np.sqrt(0.5)
    V = _v3([[c, -c], [c, c]])                      # e_min = (c, -c): exact null at theta = 0
    lam = np.array([0.0, 2.0])
    P, idx, val, npk, info = _inject(doa, alg, 1, lam, V)
    f, _ = orc.spectrum(alg, 1, 0.5, lam, V, -90.0, 1.0, 181)
    assert f[90] == 1e-300
    assert P[90] == FMAX and np.all(np.isfinite(P))
    assert idx[0] == 90 and val[0] == FMAX and npk == 1
    m = np.arange(181) != 90
    np.testing.assert_allclose(P[m].astype(np.float64), 1.0 / f[m], rtol=1e-6)


@pytest.mark.parametrize("lam,flag", [((1e-20, 0.5, 1.0), True), ((-1e-18, -1e-19, 0.0), True),
                                      ((0.25, 0.5, 1.0), False)])
def test_ev_clamp_matches_oracle(doa, lam, flag):
    lam = np.array(lam)
    V = np.eye(3, dtype=np.complex128)
    P, idx, val, npk, info = _inject(doa, "ev", 1, lam, V)
    f, oinfo = orc.spectrum("ev", 1, 0.5, lam, V, -90.0, 1.0, 181)
    assert bool(info & orc.INFO_DEGENERATE) == flag == bool(oinfo & orc.INFO_DEGENERATE)
    np.testing.assert_allclose(P.astype(np.float64), 1.0 / f, rtol=1e-6)
    assert npk == 0                                 # constant spectrum: no local maxima


@pytest.mark.parametrize("delta", [1e-9, 0.3])
def test_mn_degenerate_matches_oracle(doa, delta):
    s = np.sqrt(1.0 - delta * delta)
    V = _v3([[delta, s, 0.0], [0.0, 0.0, 1.0], [s, -delta, 0.0]])
    lam = np.array([0.1, 0.2, 3.0])
    P, idx, val, npk, info = _inject(doa, "mn", 1, lam, V)
    f, oinfo = orc.spectrum("mn", 1, 0.5, lam, V, -90.0, 1.0, 181)
    assert (info & orc.INFO_DEGENERATE) == (oinfo & orc.INFO_DEGENERATE)
    assert bool(info & orc.INFO_DEGENERATE) == (delta < 1e-3)
    np.testing.assert_allclose(P.astype(np.float64), 1.0 / f, rtol=1e-6)


@pytest.mark.parametrize("M,D", [(64, 2), (64, 8), (40, 3), (33, 1)])
@pytest.mark.parametrize("alg", ALGS)
def test_absolute_spectrum_large_K(doa, M, D, alg):
    """Oracle eigenpairs of a generated frame injected into doa_spectrum: P element-wise (absolute,
    not normalised) and the peak values, for K = M - D up to 63 noise vectors."""
    cfg = get_config("c2").with_(M=M, D=D, N=4 * M, sources=tuple(np.linspace(-40, 40, D)), dtheta=0.1)
    X = generate(cfg)[0]
    R = orc.covariance(X)
    lam, V, _, _ = orc.eig(R)
    P, idx, val, npk, info = _inject(doa, alg, D, lam, V, dtheta=0.1, L=1801)
    f, oinfo = orc.spectrum(alg, D, 0.5, lam, V, -90.0, 0.1, 1801)
    assert (info & orc.INFO_DEGENERATE) == (oinfo & orc.INFO_DEGENERATE)
    np.testing.assert_allclose(P.astype(np.float64), 1.0 / f, rtol=1e-6)
    Cm, _ = orc.projector(alg, D, lam, V)
    oidx, ofv, onpk, _ = orc.peaks(f, D)
    ok, ties, why = certify(idx, oidx, f, delta_bound(alg, M, D, R, lam, Cm, f), D)
    assert ok, why
    if np.array_equal(idx, oidx):
        np.testing.assert_allclose(val[:onpk].astype(np.float64), 1.0 / ofv[:onpk], rtol=1e-6)


def test_binding_rejects_mismatched_tensors(doa):
    plan = doa.Plan(16, 4, "music", 1.0, max_batch=8)
    X = torch.zeros((4, 32, 16), dtype=torch.complex64, device="cuda")
    R = torch.zeros((4, 16, 16), dtype=torch.complex128, device="cuda")
    with pytest.raises(ValueError):
        doa.doa_covariance(plan.h, X[..., :8].contiguous(), R)          # M mismatch
    with pytest.raises(ValueError):
        doa.doa_covariance(plan.h, X.to(torch.complex128), R)           # dtype
    with pytest.raises(ValueError):
        doa.doa_covariance(plan.h, X.cpu(), R)                          # host tensor
    with pytest.raises(ValueError):
        doa.doa_covariance(plan.h, X, R[:3])                            # B mismatch
    with pytest.raises(ValueError):
        plan.run(X.transpose(1, 2))                                     # not contiguous / wrong shape
    lam = torch.zeros((4, 16), dtype=torch.float64, device="cuda")
    V = torch.zeros((4, 16, 16), dtype=torch.complex128, device="cuda")
    info = torch.zeros((4,), dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):
        doa.doa_spectrum(plan.h, lam, V, info, P=torch.zeros((4, 10), device="cuda"))   # P too short
    with pytest.raises(ValueError):
        doa.doa_eig(plan.h, R, lam, V[:, :8].contiguous(), info)
    # the plan records its device
    pi = doa.binding.plan_info(plan.h)
    assert pi.device == torch.cuda.current_device() and pi.M == 16 and pi.D == 4 and pi.L == 181
    plan.close()


def test_plan_default_grid_ends_inside(doa):
    """the default L must keep the last grid point <= 90 deg for any step."""
    for dth in (0.13, 0.07, 0.3, 1.0, 0.01):
        plan = doa.Plan(16, 4, "music", dth, max_batch=1)
        assert -90.0 + (plan.L - 1) * dth <= 90.0 + 1e-9
        assert -90.0 + plan.L * dth > 90.0 + 1e-9
        plan.close()
