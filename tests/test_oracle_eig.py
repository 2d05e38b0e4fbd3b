"""Pins for oracle.eig — Table 2 Step-2 `jsvd` (§3.2; Eigen JacobiSVD P:107)
read as the Hermitian eigendecomposition, eigenvalues ascending (Q2).

Pins: diagonal / identity inputs (no rotation), the 2x2 closed form, the asymptotic
covariance with DFT-orthogonal sources (eigenvalues P_i*M + sigma^2 and sigma^2 — the
north_star closed form), residual and orthonormality bounds, LAPACK (numpy.linalg.eigh)
agreement, and the paper's Eq. 5 residual magnitude (Table 6) as a ceiling.
"""
import os

import numpy as np
import pytest

EPS = np.finfo(float).eps


def _herm_psd(rng, M, scale=1.0):
    G = rng.standard_normal((M, 2 * M)) + 1j * rng.standard_normal((M, 2 * M))
    return scale * (G @ G.conj().T) / (2 * M)


def test_diagonal_input(orc):
    d = np.array([3.0, -1.0, 2.0, 0.5, 2.0])
    lam, V, sw, info = orc.eig(np.diag(d).astype(complex))
    assert info == 0 and sw == 0
    np.testing.assert_array_equal(lam, np.sort(d, kind="stable"))
    # V is the permutation of I that sorts d stably
    order = np.argsort(d, kind="stable")
    np.testing.assert_array_equal(V, np.eye(5)[:, order])


def test_identity(orc):
    lam, V, sw, info = orc.eig(np.eye(7, dtype=complex))
    np.testing.assert_array_equal(lam, np.ones(7))
    np.testing.assert_array_equal(V, np.eye(7))


@pytest.mark.parametrize("seed", range(20))
def test_2x2_closed_form(orc, seed):
    rng = np.random.default_rng(seed)
    a, d = rng.standard_normal(2) * 3
    b = complex(rng.standard_normal(), rng.standard_normal())
    R = np.array([[a, b], [np.conj(b), d]])
    lam, V, _, _ = orc.eig(R)
    h = np.hypot((a - d) / 2, abs(b))
    ref = np.array([(a + d) / 2 - h, (a + d) / 2 + h])
    np.testing.assert_allclose(lam, ref, rtol=0, atol=8 * EPS * (abs(a) + abs(d) + abs(b)))
    np.testing.assert_allclose(R @ V, V * lam, rtol=0, atol=1e-14 * np.linalg.norm(R))


@pytest.mark.parametrize("M,powers,uidx", [
    (16, (32.0, 16.0, 8.0), (0, 3, 9)),
    (8, (1.0, 4.0), (1, 6)),
    (64, (2.0, 1.0, 0.5, 0.25), (0, 16, 32, 50)),
])
def test_asymptotic_dft_orthogonal(orc, M, powers, uidx):
    # R = sum_i P_i a_i a_i^H + sigma^2 I with u_i - u_j in (2/M) Z: the steering vectors are
    # orthogonal with |a_i|^2 = M, so eigenvalues are {P_i M + sigma^2} U {sigma^2}^(M-D)
    # (north_star: "eigenvalues of R equal signal powers*M + sigma^2 in the ideal case").
    sig2 = 0.1
    m = np.arange(M)
    R = sig2 * np.eye(M, dtype=complex)
    for P, k in zip(powers, uidx):
        u = -1.0 + 2.0 * k / M
        a = np.exp(-1j * np.pi * m * u)
        R += P * np.outer(a, a.conj())
    lam, V, _, info = orc.eig(R)
    ref = np.sort(np.concatenate([np.array(powers) * M + sig2, np.full(M - len(powers), sig2)]))
    assert info == 0
    np.testing.assert_allclose(lam, ref, rtol=0, atol=50 * M * EPS * np.linalg.norm(R))


@pytest.mark.parametrize("M", [2, 3, 5, 8, 16, 31, 64])
def test_residual_orthonormality_and_lapack(orc, M):
    rng = np.random.default_rng(100 + M)
    for trial in range(5):
        R = _herm_psd(rng, M, scale=10.0 ** rng.uniform(-3, 3))
        lam, V, sw, info = orc.eig(R)
        nR = np.linalg.norm(R)
        assert info == 0 and sw <= 30
        assert np.all(np.diff(lam) >= 0)
        assert np.linalg.norm(R @ V - V * lam) <= 10 * M * EPS * nR
        assert np.linalg.norm(V.conj().T @ V - np.eye(M)) <= 10 * M * EPS
        ref = np.linalg.eigvalsh(R)
        assert np.max(np.abs(lam - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_subspace_matches_lapack(orc):
    # The noise-subspace projector (the only thing the estimators use) agrees with LAPACK's.
    rng = np.random.default_rng(7)
    M, D = 16, 4
    R = _herm_psd(rng, M)
    lam, V, _, _ = orc.eig(R)
    w, U = np.linalg.eigh(R)
    Pn = V[:, : M - D] @ V[:, : M - D].conj().T
    Pl = U[:, : M - D] @ U[:, : M - D].conj().T
    assert np.linalg.norm(Pn - Pl) <= 1e-12


def test_eq5_residual_below_paper_table6(orc):
    # Eq. 5 residual |A - U S V^H|; Table 6 prints 1.075e-14 for MATLAB fp64 on an
    # 8x8 matrix.  Over 200 random unit-norm 8x8 PSD matrices the oracle stays below that value.
    here = os.path.dirname(__file__)
    with open(os.path.join(here, "golden", "paper_table6_residuals.txt")) as fh:
        rows = dict(l.split()[:2] for l in fh if l.strip() and not l.startswith("#"))
    matlab = float(rows["MATLAB"])
    rng = np.random.default_rng(8)
    worst = 0.0
    for _ in range(200):
        R = _herm_psd(rng, 8)
        R /= np.linalg.norm(R)
        lam, V, _, _ = orc.eig(R)
        worst = max(worst, np.linalg.norm(R - (V * lam) @ V.conj().T))
    assert worst <= matlab


def test_sweep_counts_reasonable(orc):
    # cyclic-by-rows fp64 needs 6-8 sweeps at M=16 on sample covariances.
    from synth import get_config, generate
    cfg = get_config("c4")
    X = generate(cfg, frames=range(20))
    for b in range(20):
        lam, V, sw, info = orc.eig(orc.covariance(X[b]))
        assert info == 0 and 4 <= sw <= 10
