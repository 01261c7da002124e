"""Multi-rank check of the frame-parallel path through the GPU (run under
torchrun; tests/test_gpu_multi.py). Every rank pixelizes its strong shard of a
clip (global frame indices key the noise, paper_2511_04261_b200/shard.py);
rank 0 gathers per-frame digests and compares them with one context over the
whole clip. DPPX_FORCE_DEVICE pins every rank to one GPU (single-GPU pools);
DPPX_DIST_BACKEND selects the plumbing backend (gloo there)."""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: synthetic frames)
import paper_2511_04261_b200 as dp  # noqa: E402
from paper_2511_04261_b200 import shard as sh  # noqa: E402

TOTAL, M, N, C, B, NSUB = 9, 72, 136, 3, 16, 4


def digests(ctx, frame0, frames):
    if frames == 0:
        return []
    fr = oracle.synth_frames(frame0, frames, M, N, C)
    mk = oracle.synth_masks(frame0, frames, M, N)
    p = dp.make_privacy_params(0.5, 16, B, NSUB)
    seeds = dp.plane_seeds(42, frames, C, frame0=frame0)
    pls, img = ctx.pixelize_adaptive(fr, mk, p, dp.NOISE_KEYED, seeds)
    return [hashlib.sha256(b"".join(pls[f * C:(f + 1) * C]) + img[f].tobytes()).hexdigest()
            for f in range(frames)]


def main():
    out = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    gpu = int(os.environ.get("DPPX_FORCE_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    backend = os.environ.get("DPPX_DIST_BACKEND", "nccl")
    torch.cuda.set_device(gpu)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
    else:
        dist.init_process_group(backend)
    ctx = dp.Context(gpu)
    s = sh.strong_shard(rank, world, TOTAL)
    mine = digests(ctx, s.frame0, s.frames)
    gathered = [None] * world
    dist.all_gather_object(gathered, (s.frame0, s.frames, mine))
    if rank == 0:
        union = [d for (_, _, ds) in sorted(gathered) for d in ds]
        single = digests(ctx, 0, TOTAL)
        with open(out, "w") as f:
            json.dump({"world": world, "frames": [g[1] for g in sorted(gathered)],
                       "identical": union == single}, f)
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
