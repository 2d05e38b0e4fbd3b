"""One doa_eig call on the c4 covariances (for ncu captures): python tools/eig_once.py [B]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2007_14135_b200 as doa  # noqa: E402
from synth import get_config, generate  # noqa: E402

cfg = get_config("c4")
B = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.B
X = torch.from_numpy(generate(cfg, frames=range(B))).cuda()
p = doa.Plan(cfg.M, cfg.D, "music", cfg.dtheta, max_batch=B)
R = p.covariance(X)
for _ in range(2):
    p.eig(R)
torch.cuda.synchronize()
