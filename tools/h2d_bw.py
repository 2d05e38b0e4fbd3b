"""Host->device bandwidth from pinned memory (the e2e ceiling): one 2 GiB copy, and 16 x 128 MiB
chunks on one stream.  python tools/h2d_bw.py"""
import json

import torch

n = 2 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
out = {}
for name, chunk in (("one_copy", n), ("chunks_128MiB", 128 << 20), ("chunks_512MiB", 512 << 20)):
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record()
            for o in range(0, n, chunk):
                d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
            e1.record()
        torch.cuda.synchronize()
        out[name] = n / (e0.elapsed_time(e1) / 1e3) / 1e9
print(json.dumps({"h2d_GBps": out}))
