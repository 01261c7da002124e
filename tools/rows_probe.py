#!/usr/bin/env python3
"""One K1r launch (1080p RGB, given b n, 120 frames) for ncu captures."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2511_04261_b200 as dp
    b, n = int(sys.argv[1]), int(sys.argv[2])
    F, M, N, C = 120, 1080, 1920, 3
    dev = torch.device("cuda:0")
    ctx = dp.Context(0)
    img = torch.empty((F, M, N * C), dtype=torch.uint8, device=dev)
    out = torch.empty_like(img)
    mask = torch.empty((F, M, N), dtype=torch.uint8, device=dev)
    d = dp._desc(M, N, C, F)
    ctx.synth_frames_dev(d, 101, 0, img, mask)
    nz, keep = dp.Context._noise(dp.NOISE_KEYED, dp.plane_seeds(42, F, C))
    p = dp.make_privacy_params(0.5, 16, b, n)
    cap = dp.adaptive_payload_capacity(M, N, b, n)
    st = (cap + 15) // 16 * 16
    stats = torch.zeros((F * C, st), dtype=torch.uint8, device=dev)
    lens = torch.zeros(F * C, dtype=torch.int32, device=dev)
    for _ in range(2):
        if n > 1:
            ctx.pixelize_adaptive_dev(d, img, mask, p, nz, stats, st, lens, out)
        else:
            ctx.pixelize_uniform_dev(d, img, p, nz, stats, out)
    ctx.synchronize()


if __name__ == "__main__":
    main()
