"""NEXT-3 measurement: the on-device Eq. 1 generator (doa_generate) alone and the streaming step
'generate the batch on the device, then the whole hot path for the four estimators', c4 shape
(65536 frames x M=16 x N=256, D=4 random DOAs per frame, 0.01 deg grid).  CUDA events on the
launching stream, warm-up first.  Prints one JSON line.
usage: python tools/gen_stream.py [--frames B] [--steps K]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_14135_b200 as doa  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=65536)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--dtheta", type=float, default=0.01)
args = ap.parse_args()
M, D, N, B = 16, 4, 256, args.frames
L = int(round(180 / args.dtheta)) + 1
torch.cuda.set_device(0)
s = torch.cuda.current_stream()
rng = np.random.default_rng(4)
th = torch.from_numpy(np.sort(rng.uniform(-60, 60, size=(B, D)), axis=1)).cuda()
X = torch.empty((B, N, M), dtype=torch.complex64, device="cuda")
plans = [doa.Plan(M, D, a, args.dtheta, L=L, max_batch=B) for a in ("phd", "music", "ev", "mn")]
R = torch.empty((B, M, M), dtype=torch.complex128, device="cuda")
lam = torch.empty((B, M), dtype=torch.float64, device="cuda")
V = torch.empty((B, M, M), dtype=torch.complex128, device="cuda")
info0 = torch.empty(B, dtype=torch.int32, device="cuda")
outs = [(torch.empty((B, D), dtype=torch.int32, device="cuda"), torch.empty((B, D), dtype=torch.float32, device="cuda"),
         torch.empty(B, dtype=torch.int32, device="cuda"), torch.empty(B, dtype=torch.int32, device="cuda"))
        for _ in plans]


def gen(step):
    doa.doa_generate(M, 0.5, D, th, 10.0, 2026, step * B, X)


def hot():
    doa.doa_covariance(plans[0].h, X, R)
    doa.doa_eig(plans[0].h, R, lam, V, info0)
    for p, (idx, val, npk, info) in zip(plans, outs):
        info.copy_(info0)
        doa.doa_spectrum(p.h, lam, V, info)
        doa.doa_peaks(p.h, B, idx, val, npk, info)


def timed(fn):
    for w in range(3):
        fn(w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for k in range(args.steps):
        fn(k)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / args.steps


g_ms = timed(gen)
h_ms = timed(lambda k: hot())
gh_ms = timed(lambda k: (gen(k), hot()))
print(json.dumps({"what": "NEXT-3 on-device Eq. 1 generator (doa_generate) + streaming step", "frames": B, "M": M,
                  "N": N, "D": D, "L": L, "generate_ms": g_ms, "generate_GBps_written": B * N * M * 8 / g_ms / 1e6,
                  "hot_path_ms": h_ms, "stream_step_ms": gh_ms, "stream_frames_per_s": B / (gh_ms / 1e3),
                  "note": "generate + S1-S7 for 4 estimators per step, no host traffic; compare the PCIe-bound e2e"}))
