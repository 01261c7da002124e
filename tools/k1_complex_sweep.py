#!/usr/bin/env python3
"""K1 time vs fraction of complex cells (mask mode, device-resident).

The statistics kernel is HBM-bound while few cells are complex and becomes
draw-bound (n*n Laplace draws per complex cell) as the fraction grows; this
measures where, for the venice shape (1080p RGB, b16 n4, 600 frames).

usage (GPU box): python tools/k1_complex_sweep.py [--frames 600]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=600)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--b", type=int, default=16)
    ap.add_argument("--n", type=int, default=4)
    args = ap.parse_args()
    import torch

    import paper_2511_04261_b200 as dp
    F, M, N, C, b, n = args.frames, 1080, 1920, 3, args.b, args.n
    dev = torch.device("cuda:0")
    ctx = dp.Context(0)
    img = torch.empty((F, M, N * C), dtype=torch.uint8, device=dev)
    out = torch.empty_like(img)
    mask = torch.empty((F, M, N), dtype=torch.uint8, device=dev)
    d = dp._desc(M, N, C, F)
    ctx.synth_frames_dev(d, 101, 0, img, mask)
    p = dp.make_privacy_params(0.5, 16, b, n)
    cap = dp.adaptive_payload_capacity(M, N, b, n)
    stride = (cap + 15) & ~15
    payload = torch.zeros((F * C, stride), dtype=torch.uint8, device=dev)
    lens = torch.zeros(F * C, dtype=torch.int32, device=dev)
    nz, keep = dp.Context._noise(dp.NOISE_KEYED, dp.plane_seeds(42, F, C))
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    GR, GC = (M + b - 1) // b, (N + b - 1) // b
    gen = torch.Generator(device=dev).manual_seed(7)
    rows = []
    for frac in (0.0, 0.1, 0.25, 0.5, 0.75, 1.0):
        cells = (torch.rand((F, GR, GC), generator=gen, device=dev) >= frac).to(torch.uint8)
        full = cells.repeat_interleave(b, 1).repeat_interleave(b, 2)[:, :M, :N]
        mask.copy_(full)
        for _ in range(2):
            ctx.pixelize_adaptive_dev(d, img, mask, p, nz, payload, stride, lens, out)
        ctx.synchronize()
        ctx.reset_stats()
        ctx.set_timing(True)
        for _ in range(args.steps):
            ctx.pixelize_adaptive_dev(d, img, mask, p, nz, payload, stride, lens, out)
        ctx.synchronize()
        st = ctx.stats()
        ctx.set_timing(False)
        k1 = st["device_ms"]["stats_tma"] / max(1, st["launches"]["stats_tma"])
        alg = F * M * N * C * 2 + int(lens.sum().item())
        rows.append({"complex_frac": frac, "k1_ms": round(k1, 4),
                     "k1_frac_of_hbm": round(alg / (k1 / 1e3) / 1e9 / peak, 4),
                     "draws_per_frame": int(C * GR * GC * ((1 - frac) + frac * n * n))})
    print(json.dumps({"workload": f"{F} x {N}x{M} RGB adaptive b{b} n{n}, random cell masks",
                      "rows": rows}))


if __name__ == "__main__":
    main()
