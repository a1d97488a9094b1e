"""Multi-rank host path on CPU (gloo, world_size 2): GOP-range and stream sharding reassemble the
single-device output exactly, and the max-over-ranks timing reduction behaves.  The per-rank
encode here is the oracle (CPU stand-in for the device kernel; the device kernel's GOP-range call
is covered by tests/test_gpu_parity.py::test_batch_gop_range_host_paths_agree_bitwise)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1311_1419_b200 import dist as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gather_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.CONFIGS["C2"].with_(T=21, W=48, H=32)
    frames = synth.gen_stream(cfg, 0)
    phi = synth.phi_from_seed(5, cfg.M, cfg.B ** 2)
    g0, g1 = pdist.shard_gops(cfg.T, cfg.G, world, rank)
    y_local, _ = oracle.encode_stream(frames[g0 * cfg.G:min(g1 * cfg.G, cfg.T)], phi, cfg.G, cfg.B, with_scale=False)
    got = pdist.gather_measurements(torch.from_numpy(y_local), dst=0)
    if rank == 0:
        y_all, _ = oracle.encode_stream(frames, phi, cfg.G, cfg.B, with_scale=False)
        q.put(bool(np.array_equal(got.numpy(), y_all)))
    else:
        q.put(got is None)
    dist.destroy_process_group()


def test_gather_measurements_two_ranks():
    """dist.gather_measurements reassembles GOP-range shards (uneven sizes) on rank 0."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(res), res


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.CONFIGS["C2"].with_(T=27, W=64, H=48)
    frames = synth.gen_stream(cfg, 0)
    phi = synth.phi_from_seed(3, cfg.M, cfg.B ** 2)
    # GOP-range shard of one stream
    g0, g1 = pdist.shard_gops(cfg.T, cfg.G, world, rank)
    f0, f1 = g0 * cfg.G, min(g1 * cfg.G, cfg.T)
    y_local, _ = oracle.encode_stream(frames[f0:f1], phi, cfg.G, cfg.B, with_scale=False)
    n_local = torch.tensor([y_local.shape[0]])
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, n_local)
    mx = int(max(s.item() for s in sizes))
    buf = torch.zeros((mx,) + y_local.shape[1:], dtype=torch.float64)
    buf[: y_local.shape[0]] = torch.from_numpy(y_local)
    gathered = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(gathered, buf)
    full = torch.cat([g[: int(s.item())] for g, s in zip(gathered, sizes)]).numpy()
    # max-over-ranks timing reduction (bench.py)
    t = torch.tensor([1.0 + rank])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        ref, _ = oracle.encode_stream(frames, phi, cfg.G, cfg.B, with_scale=False)
        q.put((bool(np.array_equal(full, ref)), float(t.item()),
               [pdist.cs_offset(cfg.T, cfg.G, world, r) for r in range(world)]))
    dist.barrier()
    dist.destroy_process_group()


def test_gop_sharding_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, tmax, offs = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok
    assert tmax == 2.0
    assert offs[0] == 0 and offs[1] > 0


@pytest.mark.parametrize("T,G,world", [(27, 8, 2), (240, 8, 8), (300, 8, 3), (9, 8, 4), (128, 32, 8), (5, 1, 2)])
def test_shard_gops_partition(T, G, world):
    ranges = [pdist.shard_gops(T, G, world, r) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == pdist.n_gops(T, G)
    for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
        assert a1 == b0 and a0 <= a1
    counts = [pdist.cs_frames_in_gops(T, G, a, b) for a, b in ranges]
    assert sum(counts) == oracle.cs_frame_count(T, G)
    offs = [pdist.cs_offset(T, G, world, r) for r in range(world)]
    assert offs == list(np.cumsum([0] + counts[:-1]))
    if G > 1 and pdist.n_gops(T, G) >= world:
        assert max(counts) - min(counts) <= G - 1   # balanced to one GOP


@pytest.mark.parametrize("n,world", [(64, 8), (64, 3), (1, 2), (5, 5)])
def test_shard_streams(n, world):
    rs = [pdist.shard_streams(n, world, r) for r in range(world)]
    assert rs[0][0] == 0 and rs[-1][1] == n
    assert all(a1 == b0 for (_, a1), (b0, _) in zip(rs, rs[1:]))
    sizes = [b - a for a, b in rs]
    assert max(sizes) - min(sizes) <= 1
