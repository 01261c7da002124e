"""Frame-parallel sharding across GPUs (one process per GPU).

Frames are independent (paper Theorem; the reference's
run_batch already treats files independently, cli.cpp:194-211), so a clip is
split into contiguous frame blocks with NO collective on the data path. Noise
is keyed by the GLOBAL frame index (plane seeds derived from (seed, frame,
channel)), never by rank, so outputs are byte-identical for any world size --
the multi-GPU analogue of the reference's schedule-independence criterion
(acceptance_main.cpp:356-401). A collective is used only once, at the end, to
reduce run statistics (frames, bytes, max device time).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    frame0: int   # global index of this rank's first frame
    frames: int   # frames owned by this rank


def strong_shard(rank: int, world: int, total_frames: int) -> Shard:
    """Contiguous block partition of a fixed clip (strong scaling)."""
    base, extra = divmod(total_frames, world)
    frames = base + (1 if rank < extra else 0)
    frame0 = rank * base + min(rank, extra)
    return Shard(rank, world, frame0, frames)


def weak_shard(rank: int, world: int, frames_per_rank: int) -> Shard:
    """Each rank owns its own block of `frames_per_rank` frames (weak scaling)."""
    return Shard(rank, world, rank * frames_per_rank, frames_per_rank)


def plane_seed_list(seed: int, shard: Shard, channels: int):
    """Per-plane seeds of a shard, keyed by global frame index."""
    from . import plane_seeds
    return plane_seeds(seed, shard.frames, channels, frame0=shard.frame0)


def reduce_run_stats(dist, device, frames: int, bytes_moved: int, ms: float) -> dict:
    """One small all-reduce at end of run: sums of frames/bytes, max of time."""
    import torch
    t = torch.tensor([float(frames), float(bytes_moved)], dtype=torch.float64, device=device)
    m = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
    return {"frames": int(t[0].item()), "bytes": int(t[1].item()), "max_ms": float(m[0].item())}
