#!/usr/bin/env python
"""Benchmark of the DOA hot path (BASELINE.json metric: "DOA frames/s and spectrum points/s
(M=16 ULA, 4 algs) at 1/2/4/8 B200").

One step = one batch of synthetic frames through the whole hot path for all four estimators:
S1 covariance + S2 eigendecomposition once per frame, then S3-S7 (coefficients, scan, peaks) for
PHD, MUSIC, EV and MN — all through the C ABI (include/doa.h) on device-resident inputs.  For
N > 1 (torchrun) the config's batch (c4: 65536 frames) is split into contiguous shards, one per
rank (strong scaling, BASELINE configs[3]; `--scaling weak` gives every rank a full batch), and
the per-frame peak lists are gathered to every rank in frame order with one NCCL all_gather per
step (the only collective; north_star).  The compute part of the step is replayed as a CUDA graph;
the gather runs after it.  The default c4 run also measures the north-star workload (c4's frames
on the 0.001-degree grid) and reports it under "north_star".  Rank 0 prints one JSON line.

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
                    help="replay the compute part of the step as a CUDA graph (auto: on)")
    ap.add_argument("--scaling", default="auto", choices=["auto", "strong", "weak"],
                    help="strong (default for batched workloads): the config's batch is split across the GPUs; "
                         "weak: every GPU owns a full batch")
    ap.add_argument("--no-north-star", dest="north_star", action="store_false",
                    help="skip the north-star (ns) measurement that the default c4 run adds")
    ap.add_argument("--engine", default="toeplitz_fp64", choices=["toeplitz_fp64", "direct_fp32", "direct_tf32x3"],
                    help="scan engine of the ULA plans (doa_plan_set_engine): the product's fp64 Toeplitz DMMA "
                         "contraction, or the NEXT-2 FP32-pipe direct form (A/B evidence)")
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
            "scaling": "strong" if cfg.B > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(cfg, n, args.gpus),
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
# Mean Jacobi sweeps of the M = 16 eigensolver on c4/ns frames (tools/eig_sweep_count.py, the
# DOA_EIG_COUNT diagnostic build): the S2 term of the step roofline.
EIG_SWEEPS_M16 = 7.72


class Workload:
    """Plans + buffers + the step of one ULA/array workload on this rank's frames."""

    def __init__(self, cfg, is_array, X, B, dev, doa, engine="toeplitz_fp64"):
        import torch
        self.cfg, self.B, self.X, self.is_array = cfg, B, X, is_array
        M, D = cfg.M, cfg.D
        if is_array:
            self.plans = [doa.Plan.array(cfg.pos, D, a, cfg.az0, cfg.daz, cfg.naz, cfg.el0, cfg.del_, cfg.nel,
                                         cfg.az_wrap, max_batch=B, device=dev) for a in ALGS]
        else:
            self.plans = [doa.Plan(M, D, a, cfg.dtheta, L=cfg.L, theta0=cfg.theta0, d_over_lambda=cfg.d_over_lambda,
                                   max_batch=B, device=dev, engine=engine) for a in ALGS]
        self.engine = "toeplitz_fp64" if is_array else engine
        self.R = torch.empty((B, M, M), dtype=torch.complex128, device=dev)
        self.lam = torch.empty((B, M), dtype=torch.float64, device=dev)
        self.V = torch.empty((B, M, M), dtype=torch.complex128, device=dev)
        self.info_eig = torch.empty((B,), dtype=torch.int32, device=dev)
        self.info = torch.empty((len(ALGS), B), dtype=torch.int32, device=dev)
        self.idx = torch.empty((len(ALGS), B, D), dtype=torch.int32, device=dev)
        self.val = torch.empty((len(ALGS), B, D), dtype=torch.float32, device=dev)
        self.npk = torch.empty((len(ALGS), B), dtype=torch.int32, device=dev)
        self.packed = torch.empty((len(ALGS), B, 2 * D + 2), dtype=torch.int32, device=dev)
        self.spec_ev = []

    def compute(self, sh, stream=None, record=False):
        """S1-S7 for the four estimators (doa_run_multi: covariance, then the frame kernel —
        eigendecomposition + the four estimators' coefficients — then one scan launch over the four
        plans and the peak selection) + packing of the peak lists; returns the number of libdoa
        kernel launches.  record=True additionally times the dominant kernel on the step's data:
        the four-plan scan launch (doa_scan_multi on the coefficients doa_run_multi left in the
        plans — one scan_cta_kernel launch per plan; general-array workloads: each plan's
        doa_spectrum), for the roofline."""
        import torch
        from paper_2007_14135_b200 import binding as bd
        from paper_2007_14135_b200 import dist as pdist
        if self.B == 0:
            return 0
        hs = [p.h for p in self.plans]
        bd.doa_run_multi(hs, self.X, self.idx, self.val, self.npk, self.info, sh)
        n = bd.doa_last_launch_count()
        if record and not self.is_array:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            bd.doa_scan_multi(hs, self.B, sh)             # S4-S6 of the four plans: 4 scan launches
            e1.record(stream)
            self.spec_ev.append((e0, e1))
            bd.doa_run_multi(hs, self.X, self.idx, self.val, self.npk, self.info, sh)   # restore the outputs
        elif record:
            bd.doa_covariance(hs[0], self.X, self.R, sh)
            bd.doa_eig(hs[0], self.R, self.lam, self.V, self.info_eig, sh)
            for a, h in enumerate(hs):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                bd.doa_spectrum(h, self.lam, self.V, self.info_eig, None, sh)
                e1.record(stream)
                self.spec_ev.append((e0, e1))
            bd.doa_run_multi(hs, self.X, self.idx, self.val, self.npk, self.info, sh)   # restore the outputs
        pdist.pack_peaks(self.idx, self.val, self.npk, self.info, out=self.packed)
        return n


def timed_steps(args, wl, ws, dev, stream, use_graph, gather):
    """Warm up, optionally capture the compute part of the step in a CUDA graph, then time exactly
    args.steps steps between CUDA events on `stream` (barrier + synchronize on both sides) and take
    the max over ranks.  gather() is the step's one collective (NCCL all_gather of the peak lists,
    ws > 1), run eagerly after the replayed compute.  Returns (ms_per_step, launches, graph, clocks)."""
    import torch
    import torch.distributed as dist
    s = stream.cuda_stream
    for _ in range(max(3, args.warmup)):
        wl.compute(s)
        gather(wl)
    torch.cuda.synchronize()
    graph, per = None, 0
    for _ in range(min(args.steps, 5)):               # per-launch timing of doa_spectrum, outside the timed steps
        wl.compute(s, stream, record=True)
    torch.cuda.synchronize()
    if use_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            per = wl.compute(stream.cuda_stream)
        for _ in range(max(3, args.warmup)):
            graph.replay()
            gather(wl)
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev.index)
    clocks.start()
    time.sleep(0.3)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    launches = 0
    for _ in range(args.steps):
        if graph is not None:
            graph.replay()
            launches += per
        else:
            launches += wl.compute(s, stream)
        gather(wl)
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    if ws > 1:
        ms = max_over_ranks(ms, dev)
        dist.barrier()
    return ms / args.steps, launches, graph, clk


def max_over_ranks(x: float, dev) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def scan_roofline(wl, is_array, mirrored):
    """Roofline of the dominant kernel (the scan inside doa_spectrum) from its CUDA-event time."""
    cfg = wl.cfg
    M, L, B = cfg.M, cfg.L, wl.B
    spec_ms = statistics.mean(e0.elapsed_time(e1) for e0, e1 in wl.spec_ev)
    if not is_array:                               # doa_scan_multi: the four plans' launches back to back
        spec_ms /= len(ALGS)
    if wl.engine == "direct_tf32x3":               # tcgen05 GEMM: 3 tf32 products of (128 angles x 256 cols x K 32)
        # algorithmic work of the direct form (as for the FP32-pipe engine); peak = dense tf32 (MEASURED_PEAKS
        # bf16 x the guide's tf32:bf16 ratio 1/2)
        nv = [(M - cfg.D) if a in ("music", "ev") else 1 for a in ALGS]
        scan_flops = sum(n * (8.0 * M + 4.0) for n in nv) / len(nv) * L * B
        pk = peaks_json()
        tf32_peak = float(pk.get("bf16_tflops", pk.get("cublas_bf16_tflops", 2250.0))) / 2.0
        return spec_ms, scan_flops, scan_flops / (spec_ms / 1e3) / 1e12, tf32_peak
    if wl.engine == "direct_fp32":                 # per vector x_j: 4M FFMA for x_j^H a, 2 for |.|^2; mean over plans
        nv = [(M - cfg.D) if a in ("music", "ev") else 1 for a in ALGS]
        scan_flops = sum(n * (8.0 * M + 4.0) for n in nv) / len(nv) * L * B
        pk = peaks_json()
        fp32_peak = 148 * 128 * 2 * float(pk.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
        return spec_ms, scan_flops, scan_flops / (spec_ms / 1e3) / 1e12, fp32_peak
    if is_array:                                   # K - 1 = M(M-1) fp64 FMAs per (frame, grid point)
        scan_flops = 2.0 * M * (M - 1) * L * B
    elif mirrored:                                 # per mirrored pair: E and O (2(M-1) FMAs), E +- O (2 adds)
        scan_flops = (2.0 * (M - 1) + 1.0) * L * B
    else:                                          # 2(M-1) fp64 FMAs per (frame, angle)
        scan_flops = 4.0 * (M - 1) * L * B
    pk = peaks_json()
    fp64_peak = 148 * 64 * 2 * float(pk.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12   # TFLOP/s, guide unit counts
    achieved = scan_flops / (spec_ms / 1e3) / 1e12
    return spec_ms, scan_flops, achieved, fp64_peak


def step_roofline_ms(cfg, B, mirrored, fp64_peak_tflops):
    """SURVEY §8(d) step roofline (T_roof = sum over stages of max(bytes/BW, flops/F64)) with the
    scan's algorithmic work as the kernel does it (mirrored: 2(M-1)+1 flops per (frame, angle))."""
    M, N, L = cfg.M, cfg.N, cfg.L
    hbm = float(peaks_json().get("hbm_gbs", 6446.9)) * 1e9
    f64 = fp64_peak_tflops * 1e12
    cov = max(8.0 * M * N * B / hbm, 4.0 * M * M * N * B / f64)
    jac = 24.0 * M * M * (M - 1) * EIG_SWEEPS_M16 * B / f64
    per = (2.0 * (M - 1) + 1.0) if mirrored else 4.0 * (M - 1)
    scan = len(ALGS) * per * L * B / f64
    return 1e3 * (cov + jac + scan)


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
    from paper_2007_14135_b200 import dist as pdist_
    # Strong scaling (default for batched workloads): BASELINE configs[3] fixes the batch (65536
    # frames) and shards it across the GPUs; weak: every rank owns its own full batch; single-frame
    # configs run as independent replicas (nothing to shard).
    total = args.frames or cfg.B
    scaling = args.scaling if args.scaling != "auto" else ("strong" if total > 1 else "weak")
    if scaling == "strong":
        frames = pdist_.shard_range(total, ws, rank)
        total_frames = total
    else:
        frames = pdist_.weak_range(total, rank)
        total_frames = total * ws
    B = len(frames)
    # generate this rank's frames BEFORE touching CUDA (the generator forks worker processes)
    from synth import generate
    t0 = time.perf_counter()
    Xh_np = generate_array(cfg, frames=frames) if is_array else generate(cfg, frames=frames)
    gen_s = time.perf_counter() - t0

    import torch
    import torch.distributed as dist
    # DOA_BENCH_ONE_GPU / DOA_BENCH_BACKEND=gloo: test hooks that run the multi-rank path as several
    # processes on one GPU (NCCL refuses two ranks on one device); the driver's runs use neither
    if os.environ.get("DOA_BENCH_ONE_GPU"):
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        backend = os.environ.get("DOA_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")    # communicator log (NVLS / NVLink paths) on stderr
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    import paper_2007_14135_b200 as doa
    from paper_2007_14135_b200 import binding as bd

    Xh = torch.from_numpy(Xh_np).pin_memory()
    del Xh_np
    X = Xh.to(dev)
    D, L = cfg.D, cfg.L
    wl = Workload(cfg, is_array, X, B, dev, doa, engine=args.engine)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)

    if ws > 1:
        gbuf = torch.empty((ws, len(ALGS), max(pdist_.shard_sizes(total_frames if scaling == "strong" else B * ws, ws)),
                            2 * D + 2), dtype=torch.int32, device=dev)
        gout = torch.empty((len(ALGS), total_frames, 2 * D + 2), dtype=torch.int32, device=dev)

        def gather(w):
            if scaling == "strong":
                pdist_.gather_sharded(w.packed, total_frames, out=gout, buf=gbuf)
            else:
                pdist_.gather_peaks(w.packed, out=gbuf)
    else:
        def gather(w):
            return None

    use_graph = args.graph in ("on", "auto")
    ms_step, launches, graph, clk = timed_steps(args, wl, ws, dev, stream, use_graph, gather)
    value = total_frames / (ms_step / 1e3)

    mirrored = (not is_array and cfg.theta0 + float(L - 1) * cfg.dtheta == -cfg.theta0
                and os.environ.get("DOA_SCAN_MIRROR", "1") != "0")
    spec_ms, scan_flops, achieved, fp64_peak = scan_roofline(wl, is_array, mirrored)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath) and cfg.name == "c4" and B == cfg.B:
        with open(tpath) as fh:
            rec = json.load(fh).get("scan", {})
            traffic = rec.get("traffic_bytes")
    roofline = {"bound": "alu", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": achieved / fp64_peak, "traffic": traffic if wl.engine == "toeplitz_fp64" else None,
                "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum of one scan launch, ncu --set full "
                                  "(profiles/traffic.json); algorithmic operand bytes per launch: coef 16.8 MB",
                "kernel": ("doa_spectrum per plan (coefficient + array scan kernels)" if is_array else
                           "scan_cta_kernel (S4-S6, FP64 DMMA mma.sync m8n8k4), one launch per estimator, "
                           "timed via doa_scan_multi on the step's coefficients (mean per launch)"),
                "algorithmic_flops_per_point": scan_flops / (L * B), "mirrored_scan": mirrored,
                "kernel_ms": spec_ms, "launches_per_step": len(ALGS),
                "share_of_step": spec_ms * len(ALGS) / ms_step,
                "peak_source": "148 SMs x 64 FP64 lanes x 2 flop x sm_max_mhz (guide unit counts; "
                               "measured DMMA 37.18 / DFMA 34.19 TFLOP/s in profiles/fp64_peaks_r01.txt)"}
    if wl.engine == "direct_tf32x3":
        roofline.update({"bound": "tensor", "kernel": "scan_tc_kernel (NEXT-2 direct form on tcgen05 kind::tf32, 3xTF32, "
                                   "TMEM accumulators), one launch per estimator, timed via doa_scan_multi",
                         "algorithmic_flops_per_point": scan_flops / (L * B),
                         "peak_source": "MEASURED_PEAKS.json bf16 dense x 1/2 (tf32:bf16 ratio of the guide)"})
    if wl.engine == "direct_fp32":
        roofline.update({"kernel": "scan_f32_kernel (NEXT-2 FP32-pipe direct form), one launch per estimator, "
                                   "timed via doa_scan_multi (mean per launch)",
                         "algorithmic_flops_per_point": scan_flops / (L * B),
                         "peak_source": "148 SMs x 128 FP32 lanes x 2 flop x sm_max_mhz (guide unit counts; "
                                        "measured FFMA 72.4 TFLOP/s in profiles/fp64_peaks_r01.txt)"})
    if not is_array:
        roofline["step_roofline_ms"] = step_roofline_ms(cfg, B, mirrored, fp64_peak)
        roofline["step_frac"] = roofline["step_roofline_ms"] / ms_step

    # north-star workload (c4's frames on the 0.001-degree grid) measured in the same run
    north = None
    if args.north_star and cfg.name == "c4" and not is_array:
        ncfg = get_config("ns")
        if ws == 1 or scaling == "strong":
            nwl = Workload(ncfg, False, X, B, dev, doa)
            nargs = argparse.Namespace(**vars(args))
            nargs.steps = max(2, min(args.steps, 5))
            n_ms, _, ngraph, nclk = timed_steps(nargs, nwl, ws, dev, stream, use_graph, gather)
            n_spec, _, n_ach, _ = scan_roofline(nwl, False, mirrored)
            n_roof = step_roofline_ms(ncfg, B, mirrored, fp64_peak)
            north = {"workload": "ns", "L": ncfg.L, "dtheta_deg": ncfg.dtheta, "frames": total_frames,
                     "value": total_frames / (n_ms / 1e3), "unit": "frames/s", "ms_per_step": n_ms,
                     "steps": nargs.steps, "points_per_s": total_frames / (n_ms / 1e3) * ncfg.L * len(ALGS),
                     "step_roofline_ms": n_roof, "step_frac": n_roof / n_ms,
                     "doa_spectrum_ms": n_spec, "doa_spectrum_frac": n_ach / fp64_peak, "clocks": nclk}
            del ngraph, nwl

    # end to end: host (pinned) -> device copies + the step + peak lists back, via doa_run_host
    e2e = None
    if not args.no_e2e and B > 0:
        n_alg = len(ALGS)
        hidx = torch.empty((n_alg, B, D), dtype=torch.int32)
        hval = torch.empty((n_alg, B, D), dtype=torch.float32)
        hnpk = torch.empty((n_alg, B), dtype=torch.int32)
        hinfo = torch.empty((n_alg, B), dtype=torch.int32)
        hs = [p.h for p in wl.plans]
        s = stream.cuda_stream
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
            ems = max_over_ranks(ems, dev)
        ems /= k2
        # consistency: the host path returns the device path's peak lists
        same = bool(torch.equal(hidx, wl.idx.cpu()))
        e2e = {"value": total_frames / (ems / 1e3), "unit": "frames/s", "ms_per_step": ems,
               "h2d_bytes_per_step": int(Xh.numel() * 8) * (ws if scaling == "strong" else 1),
               "d2h_bytes_per_step": int(hidx.numel() * 4 + hval.numel() * 4 + hnpk.numel() * 4 + hinfo.numel() * 4)
               * (ws if scaling == "strong" else 1),
               "api": "doa_run_host (4 plans)", "matches_device_path": same,
               "bytes_note": "whole job (all ranks' shards)" if scaling == "strong" else "per rank"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and not is_array:
        cpu = oracle_baseline(cfg, args.cpu_seconds)

    if rank == 0:
        cfgd = config_dict(cfg, B, ws)
        cfgd["global_batch"] = total_frames
        cfgd["scaling_split"] = (f"{total_frames} frames split into {ws} contiguous shards (dist.shard_range)"
                                 if scaling == "strong" else f"{B} frames per rank")
        if wl.engine != "toeplitz_fp64":
            cfgd["engine"] = wl.engine
        line = {"metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": ws, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None, "dtype": "f64" if wl.engine == "toeplitz_fp64" else "f32",
                "data": "synthetic",
                "config": cfgd,
                "points_per_s": value * L * len(ALGS),
                "roofline": roofline, "north_star": north, "cpu_baseline": cpu, "clocks": clk, "e2e": e2e,
                "gpu_launches": launches, "cuda_graph": graph is not None, "gen_seconds": gen_s}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
