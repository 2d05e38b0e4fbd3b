"""Multi-process (world_size 2-3, gloo, CPU) tests of the frame-sharding / peak-gather host logic
(paper_2007_14135_b200/dist.py) that bench.py runs over NCCL on GPUs.  The strong-scaling test
shards a real batch with shard_range, lets every rank compute its shard's peak lists (with the
oracle standing in for the GPU path, which needs a device), gathers them with gather_sharded and
checks the result equals the single-process batch bitwise."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fake_peaks(frames, D):
    """Deterministic per-frame stand-in for a rank's peak lists (depends only on the frame index)."""
    f = torch.tensor(list(frames), dtype=torch.int64)
    idx = ((f[:, None] * 7919 + torch.arange(D)[None, :] * 104729) % 18001).to(torch.int32)
    val = (f[:, None].double() * 0.5 + torch.arange(D)[None, :]).to(torch.float32)
    npk = (f % (D + 1)).to(torch.int32)
    info = (f % 16).to(torch.int32)
    return idx, val, npk, info


def _worker(rank, world, port, per_rank, D, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2007_14135_b200 import dist as pd
        frames = pd.weak_range(per_rank, rank)
        idx, val, npk, info = _fake_peaks(frames, D)
        packed = pd.pack_peaks(idx, val, npk, info)
        out = pd.gather_peaks(packed)
        if rank == 0:
            q.put(out.clone())
    finally:
        dist.destroy_process_group()


def _strong_worker(rank, world, port, total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2007_14135_b200 import dist as pd
        from synth import get_config, generate
        cfg = get_config("c4").with_(dtheta=0.5, N=64)
        packs = []
        frames = pd.shard_range(total, world, rank)
        X = generate(cfg, frames=frames) if len(frames) else None
        for alg in ("phd", "music", "ev", "mn"):
            if X is None:
                t = torch.zeros((0, 2 * cfg.D + 2), dtype=torch.int32)
            else:
                r = oracle.run_batch(alg, X, cfg.D, 0.5, cfg.theta0, cfg.dtheta, cfg.L)
                t = pd.pack_peaks(torch.from_numpy(r["idx"]), torch.from_numpy(r["val"]),
                                  torch.from_numpy(r["npk"]), torch.from_numpy(r["info"]))
            packs.append(t)
        out = pd.gather_sharded(torch.stack(packs), total)
        if rank == 0:
            q.put(out.clone())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total,world", [(13, 2), (13, 3), (2, 3)])
def test_strong_sharded_gather_equals_single_batch(total, world):
    """Contiguous shards of a c4-like batch (uneven when world does not divide it, including an
    empty shard), each rank's peak lists computed on its shard only, gathered in frame order:
    bitwise equal to the whole batch computed in one process."""
    import oracle
    from paper_2007_14135_b200 import dist as pd
    from synth import get_config, generate
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_strong_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = get_config("c4").with_(dtheta=0.5, N=64)
    X = generate(cfg, frames=range(total))
    assert out.shape == (4, total, 2 * cfg.D + 2)
    for a, alg in enumerate(("phd", "music", "ev", "mn")):
        r = oracle.run_batch(alg, X, cfg.D, 0.5, cfg.theta0, cfg.dtheta, cfg.L)
        ref = pd.pack_peaks(torch.from_numpy(r["idx"]), torch.from_numpy(r["val"]),
                            torch.from_numpy(r["npk"]), torch.from_numpy(r["info"]))
        assert torch.equal(out[a], ref), alg


def test_weak_sharded_gather_equals_single_process():
    world, per_rank, D = 2, 37, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, per_rank, D, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2007_14135_b200 import dist as pd
    assert out.shape == (world, per_rank, 2 * D + 2)
    idx, val, npk, info = pd.unpack_peaks(out.reshape(world * per_rank, 2 * D + 2), D)
    ridx, rval, rnpk, rinfo = _fake_peaks(range(world * per_rank), D)
    assert torch.equal(idx, ridx) and torch.equal(val, rval)
    assert torch.equal(npk, rnpk) and torch.equal(info, rinfo)


@pytest.mark.parametrize("total,world", [(65536, 8), (10, 3), (3, 4), (0, 2)])
def test_shard_range_partitions(total, world):
    from paper_2007_14135_b200 import dist as pd
    seen = []
    for r in range(world):
        seen.extend(pd.shard_range(total, world, r))
    assert seen == list(range(total))


def test_pack_roundtrip():
    from paper_2007_14135_b200 import dist as pd
    idx, val, npk, info = _fake_peaks(range(5), 3)
    out = pd.unpack_peaks(pd.pack_peaks(idx, val, npk, info), 3)
    for a, b in zip(out, (idx, val, npk, info)):
        assert torch.equal(a, b)
