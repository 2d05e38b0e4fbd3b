"""Probe: does splitting the c4 batch into chunks on two streams (S1-S2 of chunk k+1 overlapping
S3-S7 of chunk k) beat the serial step?  Separate plan sets per stream (plan workspaces are per
call).  Prints ms per step for serial and overlapped schedules."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2007_14135_b200 as doa  # noqa: E402
from synth import get_config, generate  # noqa: E402

cfg = get_config("c4")
B, M, D, N, dth = cfg.B, cfg.M, cfg.D, cfg.N, cfg.dtheta
X = torch.from_numpy(generate(cfg)).cuda()
ALGS = ("phd", "music", "ev", "mn")
nchunks = int(sys.argv[1]) if len(sys.argv) > 1 else 2
Bc = B // nchunks
streams = [torch.cuda.Stream() for _ in range(2)]
sets = []
for k in range(2):
    plans = [doa.Plan(M, D, a, dth, max_batch=Bc) for a in ALGS]
    R = torch.empty((Bc, M, M), dtype=torch.complex128, device="cuda")
    lam = torch.empty((Bc, M), dtype=torch.float64, device="cuda")
    V = torch.empty((Bc, M, M), dtype=torch.complex128, device="cuda")
    info0 = torch.empty(Bc, dtype=torch.int32, device="cuda")
    outs = [(torch.empty((Bc, D), dtype=torch.int32, device="cuda"), torch.empty((Bc, D), dtype=torch.float32, device="cuda"),
             torch.empty(Bc, dtype=torch.int32, device="cuda"), torch.empty(Bc, dtype=torch.int32, device="cuda"))
            for _ in ALGS]
    sets.append((plans, R, lam, V, info0, outs))


def chunk(c, k, st):
    plans, R, lam, V, info0, outs = sets[k]
    Xc = X[c * Bc:(c + 1) * Bc]
    doa.doa_covariance(plans[0].h, Xc, R, stream=st)
    doa.doa_eig(plans[0].h, R, lam, V, info0, stream=st)
    for p, (idx, val, npk, info) in zip(plans, outs):
        with torch.cuda.stream(st):
            info.copy_(info0)
        doa.doa_spectrum(p.h, lam, V, info, stream=st)
        doa.doa_peaks(p.h, Bc, idx, val, npk, info, stream=st)


def step_overlap():
    main = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(main)
    for st in streams:
        st.wait_event(ev)
    for c in range(nchunks):
        k = c % 2
        chunk(c, k, streams[k])
    for st in streams:
        e = torch.cuda.Event()
        e.record(st)
        main.wait_event(e)


def step_serial():
    st = torch.cuda.current_stream()
    for c in range(nchunks):
        chunk(c, 0, st)


def timeit(fn, reps=5):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


print("chunks", nchunks, "serial", round(timeit(step_serial), 3), "overlap", round(timeit(step_overlap), 3))
