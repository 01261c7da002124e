"""Multi-process (world_size 2, gloo on CPU) coverage of the frame-parallel
sharding: shards partition the clip, noise is keyed by global frame so the
union of the ranks' outputs is byte-identical to a single-process run, and the
end-of-run statistics reduce as documented. The per-frame compute here is the
oracle (CPU test infrastructure); on GPUs each rank runs the same plan."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from paper_2511_04261_b200 import shard as sh


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _frames_payloads(frame0, F, M, N, C, b, n):
    frames = oracle.synth_frames(frame0, F, M, N, C)
    masks = oracle.synth_masks(frame0, F, M, N)
    p = oracle.make_privacy_params(0.5, 16, b, n)
    out = []
    for f in range(F):
        seeds = [oracle.derive_plane_seed(42, frame0 + f, k) for k in range(C)]
        pl, img = oracle.pixelize_adaptive(frames[f], masks[f], b, n, p.sigma, p.sigma_sub,
                                           "keyed", seeds)
        out.append((pl, img.tobytes()))
    return out


def _worker(rank, world, port, total, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = sh.strong_shard(rank, world, total)
    res = _frames_payloads(s.frame0, s.frames, 40, 72, 3, 8, 2)
    gathered = [None] * world
    dist.all_gather_object(gathered, (s.frame0, s.frames, res))
    stats = sh.reduce_run_stats(dist, torch.device("cpu"), s.frames, 100 * (rank + 1),
                                1.5 + rank)
    if rank == 0:
        q.put((gathered, stats))
    dist.barrier()
    dist.destroy_process_group()


def test_partitions():
    for total in (1, 5, 600, 100000):
        for world in (1, 2, 4, 8):
            shards = [sh.strong_shard(r, world, total) for r in range(world)]
            assert sum(s.frames for s in shards) == total
            assert [s.frame0 for s in shards] == [sum(x.frames for x in shards[:r]) for r in range(world)]
    w = [sh.weak_shard(r, 4, 600) for r in range(4)]
    assert [s.frame0 for s in w] == [0, 600, 1200, 1800]


def test_two_rank_run_is_byte_identical_to_one():
    total = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, stats = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    union = [x for (_, _, res) in sorted(gathered) for x in res]
    single = _frames_payloads(0, total, 40, 72, 3, 8, 2)
    assert union == single
    assert stats == {"frames": total, "bytes": 300, "max_ms": 2.5}
