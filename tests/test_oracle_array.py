"""Pins for the general-geometry oracle: Eq. 2 steering on an
azimuth x elevation grid and the 2-D peak rule (G2)."""
import os

import mpmath as mp
import numpy as np
import pytest
from scipy.ndimage import minimum_filter

from synth import get_config, generate
from synth.array import ARRAY_CONFIGS, generate_array, uca_positions

ALGS = ["phd", "music", "ev", "mn"]


def test_ula_as_array_matches_ula_oracle(orc):
    # ULA along x with spacing d (wavelengths), elevation 90 deg: Eq. 2 gives a_m = exp(+j 2 pi d m sin az),
    # the conjugate of the north-star ULA steering; so the array spectrum of X equals the ULA spectrum
    # of conj(X) (R -> conj(R), C -> conj(C), f real).
    cfg = get_config("c2").with_(dtheta=0.1)
    X = generate(cfg)[0]
    M, D = cfg.M, cfg.D
    pos = np.stack([0.5 * np.arange(M), np.zeros(M), np.zeros(M)], axis=1)
    lam_a, V_a, _, _ = orc.eig(orc.covariance(X))
    lam_u, V_u, _, _ = orc.eig(orc.covariance(np.conj(X)))
    for alg in ALGS:
        fa, _ = orc.spectrum_array(alg, D, pos, lam_a, V_a, -90.0, 0.1, cfg.L, 90.0, 1.0, 1)
        fu, _ = orc.spectrum(alg, D, 0.5, lam_u, V_u, -90.0, 0.1, cfg.L)
        assert np.max(np.abs(fa - fu)) <= 1e-9 * np.max(fu), alg
        assert np.array_equal(orc.peaks(fa, D)[0], orc.peaks(fu, D)[0])


def _uca_closed_form_phase(M, r, az, el):
    """UCA element phases in the closed form 2 pi r sin(el) sin(az + g_m), g_m = 2 pi m / M
    (x = r cos g, y = r sin g in Eq. 2)."""
    g = 2 * np.pi * np.arange(M) / M
    return 2 * np.pi * r * np.sin(np.deg2rad(el)) * np.sin(np.deg2rad(az) + g)


def test_uca_noise_free_music_closed_form_and_exact_null(orc):
    M, r = 8, 0.5                                   # radius in wavelengths
    pos = uca_positions(M, r * 299_792_458.0, 1.0)    # 1 Hz carrier: lambda = c, so positions = r
    az0, el0 = 123.0, 60.0
    a0 = np.exp(1j * _uca_closed_form_phase(M, r, az0, el0))
    lam, V, _, _ = orc.eig(np.outer(a0, a0.conj()))
    naz, nel = 360, 90
    f, _ = orc.spectrum_array("music", 1, pos, lam, V, 0.0, 1.0, naz, 1.0, 1.0, nel)
    AZ, EL = np.meshgrid(np.arange(naz) * 1.0, 1.0 + np.arange(nel) * 1.0, indexing="ij")
    g = 2 * np.pi * np.arange(M) / M
    phs = 2 * np.pi * r * np.sin(np.deg2rad(EL.reshape(-1)))[:, None] * np.sin(np.deg2rad(AZ.reshape(-1))[:, None] + g)
    ip = np.exp(1j * phs) @ a0.conj()
    ref = M - np.abs(ip) ** 2 / M
    np.testing.assert_allclose(f, np.maximum(ref, 1e-300), rtol=0, atol=1e-11 * M)
    p_true = int(round(az0)) * nel + int(round(el0 - 1.0))
    idx, fv, npk, _ = orc.peaks2d(f, naz, nel, True, 1)
    assert idx[0] == p_true and fv[0] <= 1e-20


def test_eq2_mpmath_single_point(orc):
    # f at one grid point against a 40-digit evaluation of Eq. 2 and a^H C a
    cfg = ARRAY_CONFIGS["e1"]
    X = generate_array(cfg)[0]
    lam, V, _, _ = orc.eig(orc.covariance(X))
    Cm, _ = orc.projector("music", cfg.D, lam, V)
    f, _ = orc.spectrum_array("music", cfg.D, cfg.pos, lam, V, 0.0, 1.0, 360, 90.0, 1.0, 1)
    mp.mp.dps = 40
    for ia in (0, 37, 200, 359):
        az, el = mp.radians(ia), mp.radians(90)
        a = [mp.expj(2 * mp.pi * (mp.mpf(x) * mp.sin(az) * mp.sin(el) + mp.mpf(y) * mp.cos(az) * mp.sin(el)
                                  + mp.mpf(z) * mp.cos(el))) for x, y, z in cfg.pos]
        q = mp.mpf(0)
        for p in range(cfg.M):
            for qq in range(cfg.M):
                q += (mp.conj(a[p]) * mp.mpc(Cm[p, qq].real, Cm[p, qq].imag) * a[qq]).real
        assert abs(float(q) - f[ia]) <= 1e-12 * cfg.M


def test_planar_symmetry_and_wrap(orc):
    cfg = ARRAY_CONFIGS["e1"]
    X = generate_array(cfg)[0]
    lam, V, _, _ = orc.eig(orc.covariance(X))
    # planar array (z = 0): f(az, el) = f(az, 180 - el); azimuth period 360
    f1, _ = orc.spectrum_array("mn", cfg.D, cfg.pos, lam, V, 0.0, 1.0, 360, 30.0, 1.0, 1)
    f2, _ = orc.spectrum_array("mn", cfg.D, cfg.pos, lam, V, 0.0, 1.0, 360, 150.0, 1.0, 1)
    f3, _ = orc.spectrum_array("mn", cfg.D, cfg.pos, lam, V, 360.0, 1.0, 360, 30.0, 1.0, 1)
    assert np.max(np.abs(f1 - f2)) <= 1e-12 * np.max(f1)
    assert np.max(np.abs(f1 - f3)) <= 1e-12 * np.max(f1)


def _cases():
    path = os.path.join(os.path.dirname(__file__), "golden", "peak2d_cases.txt")
    out = []
    for line in open(path):
        if not line.strip() or line.startswith("#"):
            continue
        head, f, idx, npk = [s.strip() for s in line.split("|")]
        naz, nel, wrap, D = [int(x) for x in head.split()]
        out.append((naz, nel, bool(wrap), D, [float(x) for x in f.split()], [int(x) for x in idx.split()], int(npk)))
    return out


@pytest.mark.parametrize("naz,nel,wrap,D,f,idx,npk", _cases())
def test_peak2d_golden(orc, naz, nel, wrap, D, f, idx, npk):
    gi, gf, gn, _ = orc.peaks2d(np.array(f), naz, nel, wrap, D)
    assert gi.tolist() == idx and gn == npk


@pytest.mark.parametrize("seed", range(20))
def test_peak2d_vs_minimum_filter(orc, seed):
    rng = np.random.default_rng(seed)
    naz, nel = int(rng.integers(3, 40)), int(rng.integers(1, 30))
    wrap = bool(seed % 2)
    f = rng.random((naz, nel)) + 0.01
    mode = ["wrap" if wrap else "constant", "constant"]
    mf = minimum_filter(f, size=3, mode=mode, cval=np.inf)
    cand = np.flatnonzero((f == mf).reshape(-1))
    D = 5
    order = sorted(cand.tolist(), key=lambda p: (f.reshape(-1)[p], p))
    exp = order[:D] + [-1] * max(0, D - len(order))
    gi, gf, gn, n = orc.peaks2d(f, naz, nel, wrap, D)
    assert n == len(cand) and gi.tolist() == exp


@pytest.mark.parametrize("alg", ["music", "ev", "mn"])
def test_e1_recovers_azimuths(orc, alg):
    cfg = ARRAY_CONFIGS["e1"]
    hits = 0
    for seed in range(10):
        c = cfg.with_(seed=100 + seed)
        X = generate_array(c)
        r = orc.run_array_batch(alg, X, c.D, c.pos, c.az0, c.daz, c.naz, c.el0, c.del_, c.nel, c.az_wrap)
        est = sorted((r["idx"][0] // c.nel) * c.daz + c.az0)
        hits += all(abs(e - t) <= 1.0 for e, t in zip(est, sorted(s[0] for s in c.sources)))
    assert hits == 10
