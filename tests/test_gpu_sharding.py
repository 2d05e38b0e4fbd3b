"""Frame-sharding invariance on one GPU ("the gathered peak lists are bitwise
identical for G in {1, 2, 4, 8}").  BASELINE configs[3]'s 65536-frame batch is split into G
contiguous shards exactly as bench.py's strong-scaling mode splits it across ranks
(dist.shard_range), every shard runs bench.py's step through its own plans (max_batch = shard
size, so every kernel's launch geometry changes with G), and the concatenated idx / val / npk /
info must equal the single-batch result bit for bit.  Uneven splits (G = 3, 7) are included."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth import get_config, generate  # noqa: E402

ALGS = ["phd", "music", "ev", "mn"]


@pytest.fixture(scope="module")
def doa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2007_14135_b200 as d
    return d


@pytest.fixture(scope="module")
def c4_frames():
    cfg = get_config("c4")
    return cfg, torch.from_numpy(generate(cfg)).cuda()


def _step(doa, cfg, X):
    B = X.shape[0]
    base = doa.Plan(cfg.M, cfg.D, "music", cfg.dtheta, L=cfg.L, max_batch=B)
    lam, V, info0 = base.eig(base.covariance(X))
    outs = []
    for alg in ALGS:
        plan = doa.Plan(cfg.M, cfg.D, alg, cfg.dtheta, L=cfg.L, max_batch=B)
        info = info0.clone()
        plan.spectrum(lam, V, info)
        idx, val, npk, info = plan.peaks(B, info)
        outs.append(torch.cat([idx, val.view(torch.int32), npk[:, None], info[:, None]], dim=1))
        plan.close()
    base.close()
    return torch.stack(outs)                       # (4, B, 2D+2) int32


def test_peak_lists_invariant_under_sharding(doa, c4_frames):
    from paper_2007_14135_b200 import dist as pd
    cfg, X = c4_frames
    ref = _step(doa, cfg, X)
    for G in (2, 3, 4, 7, 8):
        parts = []
        for r in range(G):
            fr = pd.shard_range(cfg.B, G, r)
            parts.append(_step(doa, cfg, X[fr.start:fr.stop]))
        got = torch.cat(parts, dim=1)
        assert torch.equal(got, ref), f"G={G}: {int((got != ref).any(-1).sum())} frame-alg rows differ"
