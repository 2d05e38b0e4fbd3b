#!/usr/bin/env python
"""Benchmark of the DOA hot path (BASELINE.json metric: "DOA frames/s and spectrum points/s
(M=16 ULA, 4 algs) at 1/2/4/8 B200").

One step = one batch of synthetic frames through the whole hot path for all four estimators:
S1 covariance + S2 eigendecomposition once per frame, then S3-S7 (coefficients, scan, peaks) for
PHD, MUSIC, EV and MN — all through the C ABI (include/doa.h) on device-resident inputs.  For
N > 1 (torchrun) every rank owns its own batch of frames (weak scaling: frames are independent),
and the per-frame peak lists are gathered to every rank with one NCCL all_gather per step (the
only collective; north_star).  Rank 0 prints one JSON line.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c4|ns|c2|...] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ALGS = ("phd", "music", "ev", "mn")
METRIC = "DOA frames/s and spectrum points/s (M=16 ULA, 4 algs) at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--frames", type=int, default=0, help="override frames per GPU (default: config B)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the step as a CUDA graph (auto: single-GPU runs)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target oracle CPU time for cpu_baseline")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def peaks_json():
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
        return json.load(fh)


# ------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.dev), "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for n, v in zip(names, s[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        under = [x for x in sm if x > 500] or sm
        return {"sm_mhz": statistics.median(under) if under else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------------ CPU baseline
def oracle_baseline(cfg, seconds: float, frames_start: int = 0):
    """Time the oracle as it stands on this host's cores on a bounded sample of the workload."""
    import numpy as np

    import oracle
    from synth import generate

    cores = os.cpu_count() or 1
    # calibrate with one frame x 4 algs on one thread
    X1 = generate(cfg, frames=[frames_start])
    t0 = time.perf_counter()
    for a in ALGS:
        oracle.run_batch(a, X1, cfg.D, cfg.d_over_lambda, cfg.theta0, cfg.dtheta, cfg.L, threads=1)
    t1 = time.perf_counter() - t0
    n = int(max(cores, min(cfg.B, seconds * cores / max(t1, 1e-6))))
    n = max(cores, (n // cores) * cores)
    frames = list(range(frames_start, frames_start + n))
    X = generate(cfg, frames=frames)
    t0 = time.perf_counter()
    for a in ALGS:
        oracle.run_batch(a, X, cfg.D, cfg.d_over_lambda, cfg.theta0, cfg.dtheta, cfg.L, threads=cores)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "frames/s", "cores": cores, "kind": "oracle",
            "sample": f"{n} frames of {cfg.name} (frames {frames[0]}..{frames[-1]}), all 4 algorithms, "
                      f"{dt:.1f} s wall on {cores} threads; frames/s extrapolates to the full batch",
            "seconds": dt, "frames": n}


def run_reference(args, cfg):
    """--impl reference: the oracle (this tier's reference arm) on a bounded sample per step."""
    ws, rank, _ = dist_env()
    if ws > 1 and rank != 0:
        return
    import oracle
    from synth import generate
    cores = os.cpu_count() or 1
    # size each step to ~ (150 s / (steps + warmup)) of CPU time
    X1 = generate(cfg, frames=[0])
    t0 = time.perf_counter()
    for a in ALGS:
        oracle.run_batch(a, X1, cfg.D, cfg.d_over_lambda, cfg.theta0, cfg.dtheta, cfg.L, threads=1)
    t1 = time.perf_counter() - t0
    per_step = max(2.0, 150.0 / (args.steps + args.warmup))
    n = int(max(cores, per_step * cores / max(t1, 1e-6)))
    n = min(n, cfg.B)
    X = generate(cfg, frames=range(n))

    def step():
        for a in ALGS:
            oracle.run_batch(a, X, cfg.D, cfg.d_over_lambda, cfg.theta0, cfg.dtheta, cfg.L, threads=cores)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    v = n / dt
    line = {"metric": METRIC, "value": v, "unit": "frames/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(cfg, n, args.gpus),
            "points_per_s": v * cfg.L * len(ALGS),
            "cpu_baseline": {"value": v, "unit": "frames/s", "cores": cores, "kind": "oracle",
                             "sample": f"{n} frames of {cfg.name} per step, all 4 algorithms, {cores} threads"},
            "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(cfg, frames_per_gpu, n_gpus):
    if hasattr(cfg, "naz"):                        # general array (NEXT-1)
        return {"workload": cfg.name, "frames_per_gpu": frames_per_gpu, "global_batch": frames_per_gpu * n_gpus,
                "M": cfg.M, "N": cfg.N, "D": cfg.D, "geometry": "UCA r=10 m @ 15 MHz (Eq. 2)" if cfg.M == 8 else "array",
                "grid": f"{cfg.naz} az x {cfg.nel} el", "L": cfg.L, "snr_db": cfg.snr_db, "algs": list(ALGS),
                "parallelism": f"frames sharded dp{n_gpus}"}
    return {"workload": cfg.name, "frames_per_gpu": frames_per_gpu, "global_batch": frames_per_gpu * n_gpus,
            "M": cfg.M, "N": cfg.N, "D": cfg.D, "L": cfg.L, "dtheta_deg": cfg.dtheta, "d_over_lambda": cfg.d_over_lambda,
            "snr_db": cfg.snr_db, "algs": list(ALGS), "parallelism": f"frames sharded dp{n_gpus}",
            "l2": "inputs larger than L2 (X is %.2f GiB per GPU vs 126 MB L2); no flush" %
                  (frames_per_gpu * cfg.N * cfg.M * 8 / 2 ** 30)}


# ------------------------------------------------------------------------------------ our arm
def main():
    args = parse()
    from synth import get_config
    from synth.array import ARRAY_CONFIGS, generate_array
    is_array = args.workload in ARRAY_CONFIGS       # general geometry (NEXT-1: the paper's UCA workload)
    cfg = ARRAY_CONFIGS[args.workload] if is_array else get_config(args.workload)
    if is_array and os.environ.get("DOA_BENCH_NEL"):   # the paper's 360 x {1, 30, 60, 90} sweep
        nel = int(os.environ["DOA_BENCH_NEL"])
        cfg = cfg.with_(name=f"e1_360x{nel}", el0=90.0 if nel == 1 else 1.0, nel=nel)
    if args.impl == "reference":
        if is_array:
            print(json.dumps({"impl": "reference", "unavailable": "reference arm implemented for ULA workloads"}))
            return
        return run_reference(args, cfg)

    ws, rank, local = dist_env()
    B = args.frames or cfg.B
    frames = range(rank * B, (rank + 1) * B)      # == dist.weak_range(B, rank): own batch per rank
    # generate this rank's frames BEFORE touching CUDA (the generator forks worker processes)
    from synth import generate
    t0 = time.perf_counter()
    Xh_np = generate_array(cfg, frames=frames) if is_array else generate(cfg, frames=frames)
    gen_s = time.perf_counter() - t0

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_2007_14135_b200 as doa
    from paper_2007_14135_b200 import binding as bd
    from paper_2007_14135_b200 import dist as pdist

    Xh = torch.from_numpy(Xh_np).pin_memory()
    del Xh_np
    X = Xh.to(dev)
    M, D, L = cfg.M, cfg.D, cfg.L
    if is_array:
        plans = [doa.Plan.array(cfg.pos, D, a, cfg.az0, cfg.daz, cfg.naz, cfg.el0, cfg.del_, cfg.nel, cfg.az_wrap,
                                max_batch=B, device=dev) for a in ALGS]
    else:
        plans = [doa.Plan(M, D, a, cfg.dtheta, L=L, theta0=cfg.theta0, d_over_lambda=cfg.d_over_lambda,
                          max_batch=B, device=dev) for a in ALGS]
    R = torch.empty((B, M, M), dtype=torch.complex128, device=dev)
    lam = torch.empty((B, M), dtype=torch.float64, device=dev)
    V = torch.empty((B, M, M), dtype=torch.complex128, device=dev)
    info_eig = torch.empty((B,), dtype=torch.int32, device=dev)
    info = torch.empty((len(ALGS), B), dtype=torch.int32, device=dev)
    idx = torch.empty((len(ALGS), B, D), dtype=torch.int32, device=dev)
    val = torch.empty((len(ALGS), B, D), dtype=torch.float32, device=dev)
    npk = torch.empty((len(ALGS), B), dtype=torch.int32, device=dev)
    gathered = None
    if ws > 1:
        gathered = torch.empty((ws, len(ALGS), B, 2 * D + 2), dtype=torch.int32, device=dev)
        packed = torch.empty((len(ALGS), B, 2 * D + 2), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    s = stream.cuda_stream
    spec_ev = []   # (start, end) events around each doa_spectrum call (coefficients + scan kernel)

    def step(sh, record=False):
        """One step on stream handle `sh`; returns the number of libdoa kernel launches."""
        launches = 0
        bd.doa_covariance(plans[0].h, X, R, sh)
        launches += bd.doa_last_launch_count()
        bd.doa_eig(plans[0].h, R, lam, V, info_eig, sh)
        launches += bd.doa_last_launch_count()
        for a, p in enumerate(plans):
            info[a].copy_(info_eig)
            if record:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            bd.doa_spectrum(p.h, lam, V, info[a], None, sh)
            launches += bd.doa_last_launch_count()
            if record:
                e1.record(stream)
                spec_ev.append((e0, e1))
            bd.doa_peaks(p.h, B, idx[a], val[a], npk[a], info[a], sh)
            launches += bd.doa_last_launch_count()
        if ws > 1:
            pdist.pack_peaks(idx, val, npk, info, out=packed)
            pdist.gather_peaks(packed, out=gathered)
        return launches

    # CUDA graph: the step is a fixed sequence of async ABI calls on one stream, so it can be
    # captured once and replayed (removes the ~10 us per-launch CPU overhead that dominates
    # single-frame workloads).  Default: on for single-GPU runs.
    use_graph = args.graph == "on" or (args.graph == "auto" and ws == 1)
    for _ in range(max(3, args.warmup)):
        step(s)
    torch.cuda.synchronize()
    graph = None
    launches_per_step = 0
    if use_graph:
        for _ in range(min(args.steps, 5)):           # per-launch timing of doa_spectrum, outside the graph
            step(s, record=True)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            launches_per_step = step(torch.cuda.current_stream().cuda_stream)
        for _ in range(max(3, args.warmup)):
            graph.replay()
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    launches = 0
    for _ in range(args.steps):
        if graph is not None:
            graph.replay()
            launches += launches_per_step
        else:
            launches += step(s, record=True)
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    if ws > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    ms_step = ms / args.steps
    total_frames = B * ws
    value = total_frames / (ms_step / 1e3)

    # roofline of the dominant kernel: the scan (S4-S6) inside doa_spectrum.  On a symmetric grid
    # (Q26) the scan evaluates each mirrored angle pair with one contraction, so the
    # algorithmic work per angle is half that of the per-angle form.
    mirrored = (not is_array and cfg.theta0 + float(L - 1) * cfg.dtheta == -cfg.theta0
                and os.environ.get("DOA_SCAN_MIRROR", "1") != "0")
    spec_ms = statistics.mean(e0.elapsed_time(e1) for e0, e1 in spec_ev)
    if is_array:                                   # K - 1 = M(M-1) fp64 FMAs per (frame, grid point)
        scan_flops = 2.0 * M * (M - 1) * L * B
    elif mirrored:                                 # per mirrored pair: E and O (2(M-1) FMAs), E +- O (2 adds)
        scan_flops = (2.0 * (M - 1) + 1.0) * L * B
    else:                                          # 2(M-1) fp64 FMAs per (frame, angle)
        scan_flops = 4.0 * (M - 1) * L * B
    pk = peaks_json()
    fp64_peak = 148 * 64 * 2 * float(pk.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12   # TFLOP/s, guide unit counts
    achieved = scan_flops / (spec_ms / 1e3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath) and cfg.name == "c4":
        with open(tpath) as fh:
            traffic = json.load(fh).get("scan", {}).get("traffic_bytes")
    roofline = {"bound": "alu", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": achieved / fp64_peak, "traffic": traffic,
                "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum of one scan launch, ncu --set full "
                                  "(profiles/traffic.json); algorithmic operand bytes per launch: coef 16.8 MB",
                "kernel": "doa_spectrum = coef_kernel + scan kernel (FP64 DMMA mma.sync m8n8k4); events "
                          "bracket both, so the scan's own fraction is higher",
                "algorithmic_flops_per_point": scan_flops / (L * B), "mirrored_scan": mirrored,
                "kernel_ms": spec_ms, "share_of_step": spec_ms * len(ALGS) / ms_step,
                "peak_source": "148 SMs x 64 FP64 lanes x 2 flop x sm_max_mhz (guide unit counts; "
                               "measured DMMA 37.18 / DFMA 34.19 TFLOP/s in profiles/fp64_peaks_r01.txt)"}

    # end to end: host (pinned) -> device copies + the step + peak lists back, via doa_run_host
    e2e = None
    if not args.no_e2e:
        n_alg = len(ALGS)
        hidx = torch.empty((n_alg, B, D), dtype=torch.int32)
        hval = torch.empty((n_alg, B, D), dtype=torch.float32)
        hnpk = torch.empty((n_alg, B), dtype=torch.int32)
        hinfo = torch.empty((n_alg, B), dtype=torch.int32)
        hs = [p.h for p in plans]
        for _ in range(2):
            bd.doa_run_host(hs, Xh, hidx, hval, hnpk, hinfo, s)
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        k2 = max(2, min(args.steps, 5))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k2):
            bd.doa_run_host(hs, Xh, hidx, hval, hnpk, hinfo, s)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if ws > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        ems /= k2
        # consistency: the host path returns the device path's peak lists
        same = bool(torch.equal(hidx, idx.cpu()))
        e2e = {"value": total_frames / (ems / 1e3), "unit": "frames/s", "ms_per_step": ems,
               "h2d_bytes_per_step": int(Xh.numel() * 8),
               "d2h_bytes_per_step": int(hidx.numel() * 4 + hval.numel() * 4 + hnpk.numel() * 4 + hinfo.numel() * 4),
               "api": "doa_run_host (4 plans)", "matches_device_path": same}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and not is_array:
        cpu = oracle_baseline(cfg, args.cpu_seconds)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": ws, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": config_dict(cfg, B, ws),
                "points_per_s": value * L * len(ALGS),
                "roofline": roofline, "cpu_baseline": cpu, "clocks": clk, "e2e": e2e,
                "gpu_launches": launches, "cuda_graph": bool(use_graph), "gen_seconds": gen_s}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
