import sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2007_14135_b200 as doa
import oracle as orc
from synth import get_config, generate
from tiecert import max_db_error
cfg = get_config("c4").with_(dtheta=0.05)
B = 20
X = generate(cfg, frames=range(B))
for alg in ("music", "phd", "ev", "mn"):
    out = {}
    for eng in ("direct_fp32", "direct_tf32x3", "toeplitz_fp64"):
        p = doa.Plan(cfg.M, cfg.D, alg, cfg.dtheta, max_batch=B, engine=eng)
        idx, val, npk, info, P = p.run(torch.from_numpy(X).cuda(), want_P=True)
        torch.cuda.synchronize()
        out[eng] = (idx.cpu().numpy(), P.cpu().numpy().astype(np.float64))
        p.close()
    R = orc.covariance(X[0]); lam, V, _, _ = orc.eig(R)
    f, _ = orc.spectrum(alg, cfg.D, 0.5, lam, V, cfg.theta0, cfg.dtheta, cfg.L, threads=8)
    for eng, (idx, P) in out.items():
        print(alg, eng, "idx0", idx[0], "oracle", orc.peaks(f, cfg.D)[0], "dB err", round(max_db_error(P[0], 1.0 / f), 6),
              "rel vs fp32", float(np.max(np.abs(P - out["direct_fp32"][1]) / out["direct_fp32"][1])))
