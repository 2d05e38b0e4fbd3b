"""The counter-based Eq. 1 generator in numpy (synth/philox.py), pinned to Philox4x32-10
known-answer vectors and to the statistics the signal model fixes (Eq. 1; Q13, Q14)."""
import os

import numpy as np

from synth.philox import generate, philox4x32_10, samples

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")


def test_philox_known_answers():
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        out = philox4x32_10(*v[:4], v[4], v[5])
        assert [int(o) for o in out] == v[6:], line


def test_samples_are_standard_complex_normal():
    z = samples(D=3, M=13, seed=12345, frames=range(40), N=500).ravel()
    assert abs(z.mean()) < 0.01
    assert abs(np.mean(np.abs(z) ** 2) - 1.0) < 0.01                 # E|z|^2 = 1
    assert abs(np.mean(z.real ** 2) - 0.5) < 0.01 and abs(np.mean(z.real * z.imag)) < 0.01
    assert abs(np.mean(z * z)) < 0.01                                 # circular: E z^2 = 0


def test_frames_are_independent_of_batch_and_order():
    a = samples(2, 5, 7, frames=[3, 9, 11], N=17)
    b = samples(2, 5, 7, frames=[11], N=17)
    assert np.array_equal(a[2], b[0])
    assert not np.array_equal(a[0], a[1])


def test_noise_free_single_source_is_a_steering_vector_times_signal():
    X = generate(M=8, d_over_lambda=0.5, D=1, theta_deg=[20.0], snr_db=400.0, seed=3, frames=[0], N=64)[0]
    u = np.sin(np.deg2rad(20.0))
    a = np.exp(-1j * np.pi * np.arange(8) * u)
    s = X[:, 0]                                                       # a_0 = 1
    assert np.allclose(X, s[:, None] * a[None, :], atol=1e-5)


def test_covariance_matches_model():
    M, D, snr = 6, 2, 5.0
    th = [-30.0, 25.0]
    X = generate(M, 0.5, D, th, snr, seed=99, frames=range(8), N=4000).astype(np.complex128)
    R = np.einsum("bnm,bnk->mk", X, X.conj()) / (8 * 4000)
    u = np.sin(np.deg2rad(th))
    A = np.exp(-1j * np.pi * np.arange(M)[:, None] * u[None, :])
    R0 = A @ A.conj().T + 10 ** (-snr / 10) * np.eye(M)
    assert np.max(np.abs(R - R0)) < 0.05
