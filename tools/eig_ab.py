"""A/B timing of doa_eig on the c4 covariances (65536 M = 16 matrices): python tools/eig_ab.py
[lib ...] — each libdoa variant (DOA_LIB) is timed in its own subprocess; prints ms per call and
whether the eigenpairs are bitwise equal to the first variant's."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, sys, torch
sys.path.insert(0, ROOT)
import paper_2007_14135_b200 as doa
from synth import get_config, generate
cfg = get_config("c4")
B = int(os.environ.get("EIG_AB_B", cfg.B))
X = torch.from_numpy(generate(cfg, frames=range(B))).cuda()
p = doa.Plan(cfg.M, cfg.D, "music", cfg.dtheta, max_batch=B)
R = p.covariance(X)
lam, V, info = p.eig(R)
torch.cuda.synchronize()
ts = []
for _ in range(12):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); p.eig(R); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
ts = sorted(ts[2:])
torch.save({"lam": lam.cpu(), "V": V.cpu(), "info": info.cpu()}, OUT)
print(json.dumps({"lib": os.environ.get("DOA_LIB", "default"), "ms_median": ts[len(ts) // 2], "ms_min": ts[0],
                  "noconv": int((info & 1).sum())}))
'''


def main():
    libs = sys.argv[1:] or [os.path.join(ROOT, "paper_2007_14135_b200", "libdoa.so")]
    ref = None
    for i, lib in enumerate(libs):
        out = f"/tmp/eig_ab_{i}.pt"
        env = dict(os.environ, DOA_LIB=lib)
        code = CHILD.replace("ROOT", repr(ROOT)).replace("OUT", repr(out))
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        if r.returncode != 0:
            print(lib, "FAILED", r.stderr[-2000:])
            continue
        line = json.loads(r.stdout.strip().splitlines()[-1])
        import torch
        d = torch.load(out)
        if ref is None:
            ref = d
        line["bitwise_equal_to_first"] = all(torch.equal(d[k], ref[k]) for k in d)
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
