"""Pins for oracle.projector / oracle.spectrum — Table 3 Steps 3-4 and
Table 2 Step-5 on the ULA grid (EV weighting Q1; MN normalisation Q5).

Pins: projector invariants (MUSIC idempotent with trace M-D; PHD/MN rank one; MN w_0 = 1;
EV with a flat noise floor = MUSIC / sigma^2), LAPACK-built projectors, the V = I injection
(constant spectra), whole-spectrum closed forms for a noise-free single source (MUSIC and MN),
the exact null at the true angle, a 50-digit mpmath evaluation of a^H C a, the d = lambda/2
endpoint identity, the count of interior minima of a degree-(M-1) trigonometric polynomial,
and thread-count invariance.
"""
import mpmath as mp
import numpy as np
import pytest

from synth import get_config, generate

EPS = np.finfo(float).eps
ALGS = ["phd", "music", "ev", "mn"]


def _grid_theta(theta0, dtheta, L):
    """Q8 + Q26: theta0 + i*dtheta; a grid whose last point is exactly -theta0 is mirrored,
    theta_i = -theta_{L-1-i} for i >= ceil(L/2)."""
    th = theta0 + np.arange(L) * dtheta
    if L >= 2 and th[-1] == -theta0:
        H = (L + 1) // 2
        th[H:] = -th[: L - H][::-1]
    return th


def _grid_u(theta0, dtheta, L, dl=0.5):
    return 2 * dl * np.sin(np.deg2rad(_grid_theta(theta0, dtheta, L)))


def _noisy_R(orc, cfg, frame=0):
    return orc.covariance(generate(cfg, frames=[frame])[0])


def test_projector_invariants(orc):
    cfg = get_config("c2")
    R = _noisy_R(orc, cfg)
    lam, V, _, _ = orc.eig(R)
    M, D = cfg.M, cfg.D
    Cmu, _ = orc.projector("music", D, lam, V)
    assert np.linalg.norm(Cmu @ Cmu - Cmu) <= 1e-13
    assert abs(np.trace(Cmu).real - (M - D)) <= 1e-13
    assert np.linalg.norm(Cmu - Cmu.conj().T) <= 1e-14
    # MUSIC C = I - E_s E_s^H with E_s from LAPACK
    w, U = np.linalg.eigh(R)
    Es = U[:, M - D:]
    assert np.linalg.norm(Cmu - (np.eye(M) - Es @ Es.conj().T)) <= 1e-12
    for alg in ("phd", "mn"):
        Cx, _ = orc.projector(alg, D, lam, V)
        s = np.linalg.svd(Cx, compute_uv=False)
        assert s[1] <= 1e-14 * s[0], alg        # rank one
    Cmn, _ = orc.projector("mn", D, lam, V)
    assert abs(Cmn[0, 0] - 1.0) <= 1e-13       # w_0 = 1 (lambda' = (e1^H P_n e1)^-1)
    # MN from LAPACK's noise projector: valph = P_n e1 / (e1^H P_n e1)
    Pn = U[:, : M - D] @ U[:, : M - D].conj().T
    v = Pn[:, 0] / Pn[0, 0].real
    assert np.linalg.norm(Cmn - np.outer(v, v.conj())) <= 1e-11
    # EV = sum_k (1/lambda_k) e_k e_k^H with LAPACK's pairs
    Cev, _ = orc.projector("ev", D, lam, V)
    ref = (U[:, : M - D] / w[: M - D]) @ U[:, : M - D].conj().T
    assert np.linalg.norm(Cev - ref) <= 1e-11 * np.linalg.norm(ref)
    # PHD = e_min e_min^H
    Cp, _ = orc.projector("phd", D, lam, V)
    assert np.linalg.norm(Cp - np.outer(U[:, 0], U[:, 0].conj())) <= 1e-11


def test_ev_flat_noise_floor_equals_music_over_sigma2(orc):
    M, D, sig2 = 12, 2, 0.25
    m = np.arange(M)
    R = sig2 * np.eye(M, dtype=complex)
    for k in (1, 7):  # DFT-orthogonal sources: noise eigenvalues exactly sigma^2 up to rounding
        a = np.exp(-1j * np.pi * m * (-1 + 2 * k / M))
        R += np.outer(a, a.conj())
    lam, V, _, _ = orc.eig(R)
    Cev, _ = orc.projector("ev", D, lam, V)
    Cmu, _ = orc.projector("music", D, lam, V)
    assert np.linalg.norm(Cev - Cmu / sig2) <= 1e-12 / sig2


def test_identity_injection_constant_spectra(orc):
    # V = I: PHD f = |a_0|^2 = 1, MN f = |a_0|^2 = 1 exactly; MUSIC f = M - D, EV f = sum 1/lambda_k
    M, D, L = 16, 3, 1801
    lam = np.linspace(0.5, 4.0, M)
    V = np.eye(M, dtype=complex)
    for alg in ALGS:
        f, info = orc.spectrum(alg, D, 0.5, lam, V, -90.0, 0.1, L)
        ref = {"phd": 1.0, "mn": 1.0, "music": M - D, "ev": np.sum(1 / lam[: M - D])}[alg]
        assert np.max(np.abs(f - ref)) <= 4 * M * EPS * ref, alg
        if alg in ("phd", "mn"):
            assert np.all(f == 1.0)
            assert orc.peaks(f, D)[2] == 0          # constant spectrum: no peaks


@pytest.mark.parametrize("M,th0", [(8, 23.0), (16, -41.3), (16, 10.0), (64, 12.5)])
def test_noise_free_single_source_closed_forms(orc, M, th0):
    # R = a0 a0^H: MUSIC f = M - sin^2(M D/2) / (M sin^2(D/2)), D = pi (u - u0);
    # MN |w^H a|^2 = |1 - (1/M) sum_m e^{-j pi m (u - u0)}|^2 / (1 - 1/M)^2.
    m = np.arange(M)
    u0 = np.sin(np.deg2rad(th0))
    a0 = np.exp(-1j * np.pi * m * u0)
    R = np.outer(a0, a0.conj())
    lam, V, _, _ = orc.eig(R)
    L, dth = 3601, 0.05
    u = _grid_u(-90.0, dth, L)
    Dl = np.pi * (u - u0)
    with np.errstate(divide="ignore", invalid="ignore"):
        fej = np.where(np.abs(np.sin(Dl / 2)) < 1e-300, M,
                       np.sin(M * Dl / 2) ** 2 / (M * np.sin(Dl / 2) ** 2))
    f_mu, _ = orc.spectrum("music", 1, 0.5, lam, V, -90.0, dth, L)
    np.testing.assert_allclose(f_mu, np.maximum(M - fej, 1e-300), rtol=0, atol=1e-12 * M)
    s = np.exp(-1j * np.pi * np.outer(u - u0, m)).sum(axis=1) / M
    ref_mn = np.abs(1 - s) ** 2 / (1 - 1 / M) ** 2
    f_mn, _ = orc.spectrum("mn", 1, 0.5, lam, V, -90.0, dth, L)
    np.testing.assert_allclose(f_mn, np.maximum(ref_mn, 1e-300), rtol=0, atol=1e-11)


@pytest.mark.parametrize("alg", ["phd", "music", "mn", "ev"])
def test_exact_null_at_true_on_grid_angle(orc, alg):
    # north_star: "noise-free single source gives an exact null at the true theta" -> the
    # top-1 peak index is the true grid index.
    M, dth = 16, 0.01
    i_true = 13421
    th0 = -90.0 + i_true * dth
    m = np.arange(M)
    a0 = np.exp(-1j * np.pi * m * np.sin(th0 * np.pi / 180))
    R = np.outer(a0, a0.conj()) + 1e-3 * np.eye(M)      # sigma^2 > 0 keeps EV finite
    lam, V, _, _ = orc.eig(R)
    f, _ = orc.spectrum(alg, 1, 0.5, lam, V, -90.0, dth, 18001)
    idx, fv, npk, _ = orc.peaks(f, 1)
    assert npk == 1 and idx[0] == i_true
    assert fv[0] <= 1e-20 * np.max(f)


def test_sum_of_squares_equals_aHCa_and_mpmath(orc):
    cfg = get_config("c2")
    R = _noisy_R(orc, cfg)
    lam, V, _, _ = orc.eig(R)
    L, dth = 1801, 0.1
    u = _grid_u(-90.0, dth, L)
    M = cfg.M
    A = np.exp(-1j * np.pi * np.outer(np.arange(M), u))        # (M, L)
    mp.mp.dps = 40
    pick = [3, 200, 555, 901, 1200, 1799]
    for alg in ALGS:
        f, _ = orc.spectrum(alg, cfg.D, 0.5, lam, V, -90.0, dth, L)
        Cm, _ = orc.projector(alg, cfg.D, lam, V)
        q = np.einsum("ml,mn,nl->l", A.conj(), Cm, A).real
        scale = np.sum(np.abs(Cm)) * M
        assert np.max(np.abs(f - q)) <= 1e3 * EPS * scale, alg
        Cmp = mp.matrix([[mp.mpc(Cm[i, j].real, Cm[i, j].imag) for j in range(M)] for i in range(M)])
        for i in pick:
            th = mp.mpf(-90) + i * mp.mpf(dth)
            uu = mp.sin(th * mp.pi / 180)
            a = mp.matrix([mp.expj(-mp.pi * mm * uu) for mm in range(M)])
            ref = (a.H * Cmp * a)[0].real
            assert abs(float(ref) - f[i]) <= 1e-13 * scale, (alg, i)


def test_endpoint_symmetry_and_interior_minima(orc):
    cfg = get_config("c4")
    X = generate(cfg, frames=range(4))
    for b in range(4):
        lam, V, _, _ = orc.eig(orc.covariance(X[b]))
        for alg in ALGS:
            f, _ = orc.spectrum(alg, cfg.D, 0.5, lam, V, -90.0, 0.01, 18001)
            assert abs(f[0] - f[-1]) <= 1e-12 * max(f[0], f[-1])      # a(-90) = a(+90) at d = lambda/2
            assert np.all(f > 0)
            n = orc.peaks(f, cfg.D)[3]
            assert n <= cfg.M - 1                                       # degree M-1 trig polynomial


def test_thread_count_invariance(orc):
    cfg = get_config("c2")
    lam, V, _, _ = orc.eig(_noisy_R(orc, cfg))
    for alg in ALGS:
        f1, _ = orc.spectrum(alg, cfg.D, 0.5, lam, V, -90.0, 0.01, 18001, threads=1)
        f4, _ = orc.spectrum(alg, cfg.D, 0.5, lam, V, -90.0, 0.01, 18001, threads=5)
        assert np.array_equal(f1, f4)


def test_ev_degenerate_flag(orc):
    M = 8
    m = np.arange(M)
    a0 = np.exp(-1j * np.pi * m * 0.3)
    lam, V, _, _ = orc.eig(np.outer(a0, a0.conj()))       # noise eigenvalues ~ 0
    f, info = orc.spectrum("ev", 1, 0.5, lam, V, -90.0, 1.0, 181)
    assert info & orc.INFO_DEGENERATE
    assert np.all(np.isfinite(f))


@pytest.mark.parametrize("L,dth", [(18001, 0.01), (1801, 0.1), (180001, 0.001)])
def test_symmetric_grid_mirror_pin(orc, L, dth):
    # Q26: on a symmetric grid theta_{L-1-i} = -theta_i exactly, so for a REAL covariance
    # (a(-u) = conj a(u), real eigenvectors) f is exactly even: f[i] == f[L-1-i] bit for bit.
    # The plain formula theta0 + i*dtheta misses this in the last bits at thousands of indices.
    th_plain = -90.0 + np.arange(L) * dth
    assert np.any(th_plain != -th_plain[::-1])
    th = _grid_theta(-90.0, dth, L)
    assert np.array_equal(th, -th[::-1])
    cfg = get_config("c2")
    R = _noisy_R(orc, cfg).real.astype(complex)
    lam, V, _, _ = orc.eig(R)
    assert np.all(V.imag == 0)
    for alg in ALGS:
        f, _ = orc.spectrum(alg, cfg.D, 0.5, lam, V, -90.0, dth, L, threads=8)
        assert np.array_equal(f, f[::-1]), alg


def test_nonsymmetric_grid_is_plain(orc):
    # a grid that does not end at -theta0 keeps theta0 + i*dtheta everywhere: compare with the
    # brute-force a^H C a on that grid
    cfg = get_config("c2")
    lam, V, _, _ = orc.eig(_noisy_R(orc, cfg))
    L, dth, th0 = 1800, 0.1, -90.0
    assert th0 + (L - 1) * dth != -th0
    u = 2 * 0.5 * np.sin(np.deg2rad(th0 + np.arange(L) * dth))
    A = np.exp(-1j * np.pi * np.outer(np.arange(cfg.M), u))
    Cm, _ = orc.projector("music", cfg.D, lam, V)
    q = np.einsum("ml,mn,nl->l", A.conj(), Cm, A).real
    f, _ = orc.spectrum("music", cfg.D, 0.5, lam, V, th0, dth, L)
    assert np.max(np.abs(f - q)) <= 1e3 * EPS * np.sum(np.abs(Cm)) * cfg.M


# ------------------------------------------------------------------------------------------------
# Pins of the two guard branches (Q12 and G1) against closed forms.

def test_exact_zero_floor_and_fp32_saturation(orc):
    """Q12: f is floored at 1e-300 and the fp32 P = 1/f saturates at FLT_MAX.  M = 2, one snapshot
    x = (1, 1) (a noise-free source at broadside): R = [[1, 1], [1, 1]], the oracle's Jacobi gives
    e_min = (c, -c) with c = 1/sqrt(2) exactly (tau = 0 -> t = 1, s = t c = c), so at theta = 0
    (grid index 90 of -90:1:90) e_min^H a = c - c = 0 exactly: f = 0 -> 1e-300 -> P = FLT_MAX,
    the unique peak, val = FLT_MAX.  Elsewhere f = |c (1 - e^{-j pi u})|^2 = 1 - cos(pi u)."""
    X = np.array([[[1.0 + 0j, 1.0 + 0j]]], dtype=np.complex64)
    fmax = np.finfo(np.float32).max
    lam, V, _, _ = orc.eig(orc.covariance(X[0]))
    assert lam[0] == 0.0 and V[0, 0] == -V[1, 0]
    for alg in ("phd", "music"):                       # K = 1: the same C
        f, info = orc.spectrum(alg, 1, 0.5, lam, V, -90.0, 1.0, 181)
        assert f[90] == 1e-300                          # the floor (Q12), not 0
        u = np.sin(np.deg2rad(_grid_theta(-90.0, 1.0, 181)))
        ref = 1.0 - np.cos(np.pi * u)
        m = np.abs(u) > 1e-3
        assert np.max(np.abs(f[m] - ref[m]) / ref[m]) <= 1e-13
        r = orc.run_batch(alg, X, 1, 0.5, -90.0, 1.0, 181, want_P=True)
        assert r["P"][0, 90] == fmax                    # saturated, not inf
        assert np.all(np.isfinite(r["P"][0]))
        assert r["idx"][0, 0] == 90 and r["val"][0, 0] == fmax and r["npk"][0] == 1
        np.testing.assert_allclose(r["P"][0, m], (1.0 / ref[m]).astype(np.float32), rtol=1e-6)


def _v3(cols):
    return np.ascontiguousarray(np.array(cols, dtype=np.complex128).T)   # columns -> V[i][j]


def test_ev_degenerate_clamp_value(orc):
    """G1 (EV): a noise eigenvalue <= 100 eps lambda_max is clamped to that floor, i.e. weight
    1/(100 eps lambda_max), DEGENERATE; V = I makes |e_k^H a|^2 = 1, so f is the weight sum:
    lambda = (1e-20, 0.5, 1), K = 2 -> f = 1/(100 eps) + 2.  With lambda_max <= 0 the floor is 0
    and every weight is 1 -> f = K.  A clean spectrum (lambda = (0.25, 0.5, 1)) has no flag and
    f = 4 + 2."""
    V = np.eye(3, dtype=np.complex128)
    f, info = orc.spectrum("ev", 1, 0.5, np.array([1e-20, 0.5, 1.0]), V, -90.0, 1.0, 181)
    assert info & orc.INFO_DEGENERATE
    np.testing.assert_allclose(f, 1.0 / (100 * EPS) + 2.0, rtol=1e-14)
    f, info = orc.spectrum("ev", 1, 0.5, np.array([-1e-18, -1e-19, 0.0]), V, -90.0, 1.0, 181)
    assert info & orc.INFO_DEGENERATE
    np.testing.assert_allclose(f, 2.0, rtol=1e-14)
    f, info = orc.spectrum("ev", 1, 0.5, np.array([0.25, 0.5, 1.0]), V, -90.0, 1.0, 181)
    assert info == 0
    np.testing.assert_allclose(f, 6.0, rtol=1e-14)


def test_mn_degenerate_unnormalised(orc):
    """G1 (MN): with e1^H P_n e1 <= 100 eps the vector w = P_n e1 is kept unnormalised.  Noise
    vectors (delta, s, 0) and (0, 0, 1), s = sqrt(1 - delta^2), signal (s, -delta, 0): P_n e1 =
    delta (delta, s, 0), p0 = delta^2 = 1e-18 -> DEGENERATE and
    f = |w^H a|^2 = delta^2 (1 + 2 delta s cos(pi u))  (normalising would give f / delta^4).
    Above the threshold (delta = 0.3) w is normalised: f = (1 + 2 delta s cos(pi u)) / delta^2."""
    th = _grid_theta(-90.0, 1.0, 181)
    u = np.sin(np.deg2rad(th))
    for delta, degen in ((1e-9, True), (0.3, False)):
        s = np.sqrt(1.0 - delta * delta)
        V = _v3([[delta, s, 0.0], [0.0, 0.0, 1.0], [s, -delta, 0.0]])
        f, info = orc.spectrum("mn", 1, 0.5, np.array([0.1, 0.2, 3.0]), V, -90.0, 1.0, 181)
        base = 1.0 + 2.0 * delta * s * np.cos(np.pi * u)
        ref = delta ** 2 * base if degen else base / delta ** 2
        assert bool(info & orc.INFO_DEGENERATE) == degen
        np.testing.assert_allclose(f, ref, rtol=1e-12)
