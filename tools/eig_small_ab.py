"""Small-batch eigensolver latency A/B: python tools/eig_small_ab.py lib1 [lib2 ...] — per library
(DOA_LIB, own subprocess) the time per doa_eig call for B = 1, 4, 64, 512 c2-shaped matrices
(M = 16, n launches captured in a CUDA graph and replayed), and bitwise equality of the eigenpairs with the first library."""
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
res = {}
outs = {}
for B in (1, 4, 64, 512):
    X = torch.from_numpy(generate(cfg, frames=range(B))).cuda()
    p = doa.Plan(cfg.M, cfg.D, "music", cfg.dtheta, max_batch=B)
    R = p.covariance(X)
    lam, V, info = p.eig(R)
    torch.cuda.synchronize()
    n = 50
    lam2, V2, info2 = p.eig(R)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):                 # n launches, replayed without host overhead
        for _ in range(n):
            doa.doa_eig(p.h, R, lam2, V2, info2, s.cuda_stream)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        g.replay()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    res[B] = e0.elapsed_time(e1) / n * 1e3
    outs[B] = (lam.cpu(), V.cpu(), info.cpu())
torch.save(outs, OUT)
print(json.dumps({"lib": os.environ.get("DOA_LIB"), "us_per_call": res}))
'''
ref = None
for i, lib in enumerate(sys.argv[1:]):
    out = f"/tmp/eig_small_{i}.pt"
    r = subprocess.run([sys.executable, "-c", CHILD.replace("ROOT", repr(ROOT)).replace("OUT", repr(out))],
                       env=dict(os.environ, DOA_LIB=lib), capture_output=True, text=True)
    if r.returncode:
        print(lib, "FAILED", r.stderr[-1500:])
        continue
    d = json.loads(r.stdout.strip().splitlines()[-1])
    import torch
    o = torch.load(out)
    ref = ref or o
    d["bitwise_equal_to_first"] = all(torch.equal(a, b) for B in o for a, b in zip(o[B], ref[B]))
    print(json.dumps(d), flush=True)
