"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck / initcheck): every stage of
the ULA path at M = 8, 16, 33, 64 on symmetric and plain grids, plus the general-array path.
usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_14135_b200 as doa  # noqa: E402
from synth import get_config, generate  # noqa: E402

torch.cuda.set_device(0)
for M, D, dth, L, B in [(16, 4, 0.5, 361, 37), (16, 4, 0.07, 2572, 19), (8, 2, 1.0, 181, 5), (33, 5, 0.5, 361, 9),
                        (64, 8, 0.5, 361, 3)]:
    cfg = get_config("c2").with_(M=M, D=D, N=64, sources=tuple(np.linspace(-40, 40, D)), dtheta=dth)
    X = torch.from_numpy(generate(cfg, frames=range(B))).cuda()
    for alg in ("phd", "music", "ev", "mn"):
        plan = doa.Plan(M, D, alg, dth, L=L, max_batch=B)
        out = plan.run(X, want_P=True)
        torch.cuda.synchronize()
        plan.close()
    print("ok", M, L, flush=True)
print("sanitize run done")
