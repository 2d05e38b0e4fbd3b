"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck / initcheck): every stage of
the ULA path at M = 8, 16, 33, 64 on symmetric and plain grids — single-plan doa_run (frame kernel
with one plan + P), doa_run_multi (frame kernel with four plans; eig16s below 2048 frames, eig16h at
2048), the small-batch direct scan and multi-CTA covariance (B <= 16, N > 256), doa_scan_multi, the
staged doa_eig/doa_spectrum path, the NEXT-2 fp32 engine and the general-array path (tiled 2-D peaks).
usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py [quick]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_14135_b200 as doa  # noqa: E402
from synth import get_config, generate  # noqa: E402
from synth.array import ARRAY_CONFIGS, generate_array  # noqa: E402

torch.cuda.set_device(0)
quick = len(sys.argv) > 1 and sys.argv[1] in ("quick", "tiny")
tiny = len(sys.argv) > 1 and sys.argv[1] == "tiny"
ALGS = ("phd", "music", "ev", "mn")
cases = [(16, 4, 0.5, 361, 37, 64), (16, 4, 0.07, 2572, 19, 64), (8, 2, 1.0, 181, 5, 64), (33, 5, 0.5, 361, 9, 64),
         (64, 8, 0.5, 361, 3, 64), (16, 3, 0.5, 361, 3, 1024)]
if not quick:
    cases.append((16, 4, 1.0, 181, 2048, 64))
if tiny:
    cases = [(16, 4, 0.5, 361, 37, 64), (16, 3, 0.5, 361, 3, 1024)]
for M, D, dth, L, B, N in cases:
    cfg = get_config("c2").with_(M=M, D=D, N=N, sources=tuple(np.linspace(-40, 40, D)), dtheta=dth)
    X = torch.from_numpy(generate(cfg, frames=range(B))).cuda()
    plans = [doa.Plan(M, D, a, dth, L=L, max_batch=B) for a in ALGS]
    for p in plans:
        p.run(X, want_P=True)
    doa.run_multi(plans, X)
    doa.doa_scan_multi([p.h for p in plans], B)
    R = plans[0].covariance(X)
    lam, V, info = plans[0].eig(R)
    plans[1].spectrum(lam, V, info=info.clone(), want_P=True)
    plans[1].peaks(B, info=info.clone())
    if M <= 16:
        plans[2].set_engine("direct_fp32")
        plans[2].run(X, want_P=True)
        plans[3].set_engine("direct_tf32x3")
        plans[3].run(X, want_P=True)
    torch.cuda.synchronize()
    for p in plans:
        p.close()
    print("ok", M, L, B, N, flush=True)
acfg = ARRAY_CONFIGS["e1_360x90"]
Xa = torch.from_numpy(generate_array(acfg)).cuda()
for alg in ALGS:
    ap = doa.Plan.array(acfg.pos, acfg.D, alg, acfg.az0, acfg.daz, acfg.naz, acfg.el0, acfg.del_, acfg.nel,
                        acfg.az_wrap, max_batch=1)
    ap.run(Xa, want_P=True)
    torch.cuda.synchronize()
    ap.close()
print("ok array")
print("sanitize run done")
