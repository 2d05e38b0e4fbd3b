import json, os, subprocess, sys
ROOT = "/root/repo"
CHILD = r'''
import json, os, sys, torch
sys.path.insert(0, "/root/repo")
import paper_2007_14135_b200 as doa
from synth import get_config, generate
cfg = get_config("c5")
B = 1024
X = torch.from_numpy(generate(cfg.with_(N=256), frames=range(B))).cuda()
p = doa.Plan(cfg.M, cfg.D, "music", 0.5, max_batch=B)
R = p.covariance(X)
lam, V, info = p.eig(R)
torch.cuda.synchronize()
ts = []
for _ in range(6):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); p.eig(R); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
torch.save({"lam": lam.cpu(), "V": V.cpu()}, OUT)
print(json.dumps({"lib": os.environ.get("DOA_LIB", "default"), "ms": sorted(ts)[len(ts)//2]}))
'''
ref = None
for i, lib in enumerate(sys.argv[1:]):
    out = f"/tmp/eign_{i}.pt"
    env = dict(os.environ, DOA_LIB=os.path.join(ROOT, lib))
    r = subprocess.run([sys.executable, "-c", CHILD.replace("OUT", repr(out))], env=env, capture_output=True, text=True)
    if r.returncode: print(lib, "FAIL", r.stderr[-1500:]); continue
    import torch
    d = torch.load(out)
    line = json.loads(r.stdout.strip().splitlines()[-1])
    if ref is None: ref = d
    line["bitwise_equal_to_first"] = all(torch.equal(d[k], ref[k]) for k in d)
    print(json.dumps(line))
