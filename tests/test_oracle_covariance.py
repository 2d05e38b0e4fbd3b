"""Pins for oracle.covariance — Eq. 3 (§3.1) / Table 2 Step-1.

Each check is fixed by the mathematics, not by re-typing the oracle's loop:
closed forms (N=1, X=0, rank-1 noiseless data), invariants (exact Hermitian symmetry,
trace = ||X||_F^2 / N), a 50-digit mpmath evaluation, and a BLAS cross-check.
"""
import mpmath as mp
import numpy as np
import pytest

from synth import get_config, generate, steering_ula


def _rand_X(rng, N, M):
    return (rng.standard_normal((N, M)) + 1j * rng.standard_normal((N, M))).astype(np.complex64)


def test_single_snapshot_is_outer_product(orc):
    # N = 1: R = x x^H exactly (fp32 products are exact in fp64; no summation).
    rng = np.random.default_rng(1)
    X = _rand_X(rng, 1, 7)
    x = X[0].astype(np.complex128)
    R = orc.covariance(X)
    assert np.array_equal(R, np.outer(x, np.conj(x)))


def test_zero_input(orc):
    R = orc.covariance(np.zeros((5, 6), np.complex64))
    assert np.array_equal(R, np.zeros((6, 6)))


def test_exact_hermitian_and_real_diagonal(orc):
    rng = np.random.default_rng(2)
    X = _rand_X(rng, 333, 16)
    R = orc.covariance(X)
    assert np.array_equal(R, R.conj().T)          # bitwise: conjugate products are exact mirrors
    assert np.all(np.imag(np.diag(R)) == 0.0)


def test_trace_is_frobenius_energy(orc):
    rng = np.random.default_rng(3)
    X = _rand_X(rng, 1000, 12)
    R = orc.covariance(X)
    e = np.sum(np.abs(X.astype(np.complex128)) ** 2) / 1000
    assert abs(np.trace(R).real - e) <= 1e-14 * e


def test_noiseless_rank_one(orc):
    # X = a s^T  =>  R = (||s||^2 / N) a a^H  (signal model Eq. 1 with W = 0, one source)
    cfg = get_config("c1").with_(D=1, sources=(23.0,), N=64)
    X = generate(cfg, noiseless=True)[0]            # complex64 rounding of a s^T
    R = orc.covariance(X)
    Xd = X.astype(np.complex128)
    # rank one up to the complex64 rounding of X
    w = np.linalg.eigvalsh(R)
    assert w[-2] <= 1e-12 * w[-1]
    a = steering_ula([23.0], cfg.M, cfg.d_over_lambda)[:, 0]
    s_energy = np.sum(np.abs(Xd[:, 0]) ** 2) / 64   # |a_0| = 1 so column 0 carries ||s||^2
    np.testing.assert_allclose(R, s_energy * np.outer(a, a.conj()), rtol=0, atol=1e-6 * s_energy)


def test_mpmath_small(orc):
    # M = 2, N = 3 evaluated with 50-digit arithmetic
    rng = np.random.default_rng(4)
    X = _rand_X(rng, 3, 2)
    R = orc.covariance(X)
    mp.mp.dps = 50
    for i in range(2):
        for j in range(2):
            acc = mp.mpc(0)
            for n in range(3):
                xi = mp.mpc(float(X[n, i].real), float(X[n, i].imag))
                xj = mp.mpc(float(X[n, j].real), float(X[n, j].imag))
                acc += xi * mp.conj(xj)
            ref = acc / 3
            assert abs(complex(ref) - R[i, j]) <= 2e-16 * (abs(complex(ref)) + 1e-300) + 1e-300


@pytest.mark.parametrize("M,N", [(8, 100), (16, 256), (16, 1024), (64, 257)])
def test_blas_cross_check(orc, M, N):
    rng = np.random.default_rng(M * 1000 + N)
    X = _rand_X(rng, N, M)
    R = orc.covariance(X)
    Xd = X.astype(np.complex128)
    ref = Xd.T @ Xd.conj() / N
    assert np.max(np.abs(R - ref)) <= 1e-14 * np.max(np.abs(ref))
