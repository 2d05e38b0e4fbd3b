import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import collections, torch, numpy as np
import paper_2007_14135_b200 as doa
from synth import get_config, generate
cfg=get_config("c4")
X=torch.from_numpy(generate(cfg, frames=range(4096))).cuda()
p=doa.Plan(16,4,"music",0.01,max_batch=4096)
R=p.covariance(X); lam,V,info=p.eig(R)
sw=(info.cpu().numpy()>>8)
print(collections.Counter(sw.tolist()), sw.mean())
