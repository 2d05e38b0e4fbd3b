"""doa_run_multi (several estimators of one batch in one call) and the small-batch direct scan.

* doa_run_multi equals per-plan doa_run bit for bit, for batches that take the direct scan
  (B <= 16: one launch evaluates all four estimators with the steering generated once per angle)
  and for batches that take the DMMA contraction.
* The direct scan against the oracle (peaks exact or certified, P within 1e-3 dB) on the paper's
  scan-range sweep (c3 down to 0.0001 deg, L = 1.8M), on one-sided (per-angle) grids, M = 2..64,
  and at the B = 16 / 17 regime boundary; and against the DMMA path on the same frames.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as orc  # noqa: E402
from synth import get_config, generate  # noqa: E402
from tiecert import certify, delta_bound, max_db_error  # noqa: E402

ALGS = ["phd", "music", "ev", "mn"]


@pytest.fixture(scope="module")
def doa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2007_14135_b200 as d
    return d


def _plans(doa, cfg, B, **kw):
    return [doa.Plan(cfg.M, cfg.D, a, cfg.dtheta, L=cfg.L, theta0=cfg.theta0, d_over_lambda=cfg.d_over_lambda,
                     max_batch=B, **kw) for a in ALGS]


def _oracle(X, alg, cfg):
    R = orc.covariance(X)
    lam, V, _, _ = orc.eig(R)
    f, _ = orc.spectrum(alg, cfg.D, cfg.d_over_lambda, lam, V, cfg.theta0, cfg.dtheta, cfg.L, threads=8)
    Cm, _ = orc.projector(alg, cfg.D, lam, V)
    return R, lam, f, Cm, orc.peaks(f, cfg.D)[0]


@pytest.mark.parametrize("B", [1, 5, 16, 17, 300])
def test_run_multi_equals_per_plan_run(doa, B):
    cfg = get_config("c4").with_(dtheta=0.05)
    X = torch.from_numpy(generate(cfg, frames=range(B))).cuda()
    plans = _plans(doa, cfg, B)
    idx, val, npk, info = doa.run_multi(plans, X)
    for a, p in enumerate(plans):
        i1, v1, n1, f1, _ = p.run(X)
        assert torch.equal(idx[a], i1) and torch.equal(val[a], v1)
        assert torch.equal(npk[a], n1) and torch.equal(info[a], f1)
    for p in plans:
        p.close()


@pytest.mark.parametrize("cfgname", ["c1", "c2", "c3_0.001", "c3_0.0001"])
def test_run_multi_single_frame_parity(doa, cfgname):
    cfg = get_config(cfgname)
    X = generate(cfg)
    plans = _plans(doa, cfg, 1)
    idx, val, npk, info = [t.cpu().numpy() for t in doa.run_multi(plans, torch.from_numpy(X).cuda())]
    for a, alg in enumerate(ALGS):
        R, lam, f, Cm, oidx = _oracle(X[0], alg, cfg)
        ok, ties, why = certify(idx[a, 0], oidx, f, delta_bound(alg, cfg.M, cfg.D, R, lam, Cm, f), cfg.D)
        assert ok, f"{cfgname} {alg}: {why}"
    for p in plans:
        p.close()


@pytest.mark.parametrize("M,D,theta0,dtheta,L,B", [
    (16, 3, -70.0, 0.07, 2286, 3),        # one-sided grid: per-angle direct scan
    (64, 8, -90.0, 0.05, 3601, 2),        # M = 64, mirrored
    (33, 5, -90.0, 0.1, 1801, 16),        # B = 16: the last direct batch size
    (2, 1, -90.0, 1.0, 181, 4),
    (9, 2, -60.0, 0.25, 481, 7)])
def test_direct_scan_parity(doa, M, D, theta0, dtheta, L, B):
    cfg = get_config("c2").with_(M=M, D=D, N=3 * M + 5, sources=tuple(np.linspace(-40, 40, D)), theta0=theta0,
                                 dtheta=dtheta)
    X = generate(cfg, frames=range(B))
    for alg in ALGS:
        plan = doa.Plan(M, D, alg, dtheta, L=L, theta0=theta0, max_batch=B)
        idx, val, npk, info, P = plan.run(torch.from_numpy(X).cuda(), want_P=True)
        idx, P = idx.cpu().numpy(), P.cpu().numpy()
        for b in range(B):
            R = orc.covariance(X[b])
            lam, V, _, _ = orc.eig(R)
            f, _ = orc.spectrum(alg, D, 0.5, lam, V, theta0, dtheta, L, threads=8)
            Cm, _ = orc.projector(alg, D, lam, V)
            ok, ties, why = certify(idx[b], orc.peaks(f, D)[0], f, delta_bound(alg, M, D, R, lam, Cm, f), D)
            assert ok, f"M={M} b={b} {alg}: {why}"
            assert max_db_error(P[b], 1.0 / f) <= 1e-3
            np.testing.assert_allclose(P[b].astype(np.float64), 1.0 / f, rtol=1e-6)
        plan.close()


def test_direct_and_dmma_paths_agree(doa):
    """The same 16 frames through the direct scan (B = 16) and inside a 64-frame batch (DMMA)."""
    cfg = get_config("c4")
    X = torch.from_numpy(generate(cfg, frames=range(64))).cuda()
    for alg in ALGS:
        plan = doa.Plan(cfg.M, cfg.D, alg, cfg.dtheta, max_batch=64)
        big = plan.run(X, want_P=True)
        small = plan.run(X[:16].contiguous(), want_P=True)
        Pb, Ps = big[4][:16].cpu().numpy().astype(np.float64), small[4].cpu().numpy().astype(np.float64)
        assert np.max(np.abs(Pb - Ps) / Pb) <= 1e-6
        for b in np.nonzero(np.any(big[0][:16].cpu().numpy() != small[0].cpu().numpy(), axis=1))[0]:
            R, lam, f, Cm, oidx = _oracle(X[b].cpu().numpy(), alg, cfg)
            for g in (big[0][b], small[0][b]):
                ok, _, why = certify(g.cpu().numpy(), oidx, f, delta_bound(alg, cfg.M, cfg.D, R, lam, Cm, f), cfg.D)
                assert ok, why
        plan.close()


def test_run_multi_rejects_bad_plan_sets(doa):
    cfg = get_config("c4")
    X = torch.zeros((4, 8, 16), dtype=torch.complex64, device="cuda")
    p16 = doa.Plan(16, 4, "music", 1.0, max_batch=4)
    p8 = doa.Plan(8, 2, "music", 1.0, max_batch=4)
    with pytest.raises(doa.DoaError):
        doa.run_multi([p16, p16], X)                      # repeated plan
    with pytest.raises((doa.DoaError, ValueError)):
        doa.run_multi([p16, p8], X)                       # different M
    small = doa.Plan(16, 4, "ev", 1.0, max_batch=2)
    with pytest.raises(doa.DoaError):
        doa.run_multi([p16, small], X)                    # B > max_batch of one plan
    for p in (p16, p8, small):
        p.close()


# ---------------------------------------------------------------------------------------------
# The frame kernel (eigendecomposition + S3 of every plan in one launch, M <= 16) and the four-plan
# scan launch: against the staged path (doa_eig -> doa_spectrum -> doa_peaks, which keeps the
# separate coefficient kernel), across the eig16s / eig16h boundary, and doa_scan_multi.

@pytest.mark.parametrize("M,D,B", [(16, 4, 300), (8, 2, 40), (12, 3, 2100)])
def test_frame_kernel_matches_staged_path(doa, M, D, B):
    cfg = get_config("c4").with_(M=M, D=D, dtheta=0.05)
    Xn = generate(cfg, frames=range(B))
    X = torch.from_numpy(Xn).cuda()
    plans = _plans(doa, cfg, B)
    idx, val, npk, info = [t.cpu().numpy() for t in doa.run_multi(plans, X)]
    R = plans[0].covariance(X)
    lam, V, einfo = plans[0].eig(R)
    for a, (alg, p) in enumerate(zip(ALGS, plans)):
        Ps, sinfo = p.spectrum(lam, V, info=einfo.clone(), want_P=True)
        si, sv, sn, sf = [t.cpu().numpy() for t in p.peaks(B, info=sinfo)]
        _, _, _, _, Pf = p.run(X, want_P=True)                   # fused path with P (single plan)
        Ps, Pf = Ps.cpu().numpy().astype(np.float64), Pf.cpu().numpy().astype(np.float64)
        assert np.max(np.abs(Pf - Ps) / Ps) <= 1e-6, alg        # same eigenpairs, S3 rounded differently
        diff = np.any(idx[a] != si, axis=1) | (npk[a] != sn)
        assert np.array_equal(info[a][~diff], sf[~diff]), alg
        for b in np.nonzero(diff)[0]:                            # differences only at certified ties
            Ro, lo, fo, Cm, oidx = _oracle(Xn[b], alg, cfg)
            for g in (idx[a, b], si[b]):
                ok, _, why = certify(g, oidx, fo, delta_bound(alg, M, D, Ro, lo, Cm, fo), D)
                assert ok, f"{alg} b={b}: {why}"
    for p in plans:
        p.close()


@pytest.mark.parametrize("M", [8, 16])
def test_frame_kernel_batch_invariant(doa, M):
    """B = 2047 runs eig16s (CTA per matrix), B = 2048 eig16h (two matrices per warp): the frame
    kernel's coefficients, hence every output, are bitwise the same for the common frames."""
    cfg = get_config("c4").with_(M=M, D=3, dtheta=0.5)
    X = torch.from_numpy(generate(cfg, frames=range(2048))).cuda()
    plans = _plans(doa, cfg, 2048)
    big = doa.run_multi(plans, X)
    small = doa.run_multi(plans, X[:2047].contiguous())
    for t_big, t_small in zip(big, small):
        assert torch.equal(t_big[:, :2047], t_small)
    for p in plans:
        p.close()


@pytest.mark.parametrize("B", [9, 1000])
def test_scan_multi_reproduces_run_multi(doa, B):
    cfg = get_config("c4").with_(dtheta=0.02)
    X = torch.from_numpy(generate(cfg, frames=range(B))).cuda()
    plans = _plans(doa, cfg, B)
    idx, val, npk, info = doa.run_multi(plans, X)
    doa.doa_scan_multi([p.h for p in plans], B)
    for a, p in enumerate(plans):
        i2, v2, n2, f2 = p.peaks(B, info=info[a].clone())
        assert torch.equal(i2, idx[a]) and torch.equal(v2, val[a]) and torch.equal(n2, npk[a])
        assert torch.equal(f2, info[a])
    doa.doa_scan_multi([p.h for p in plans[1:3]], B // 2)     # a subset, fewer frames
    with pytest.raises(doa.DoaError):
        doa.doa_scan_multi([p.h for p in plans], B + 1)      # more frames than the plans hold
    other = doa.Plan(cfg.M, cfg.D, "music", 0.5, max_batch=B)
    other.run(X)
    with pytest.raises(doa.DoaError):
        doa.doa_scan_multi([plans[0].h, other.h], B)          # different grid
    for p in plans + [other]:
        p.close()
