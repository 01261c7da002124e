#!/usr/bin/env python3
"""Per-b K1 time of the padding sweep workload (60 x 1917x1083 RGB, uniform)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2511_04261_b200 as dp
    F, M, N, C = 60, 1083, 1917, 3
    dev = torch.device("cuda:0")
    ctx = dp.Context(0)
    pitch = (N * C + 15) // 16 * 16
    img = torch.empty((F, M, pitch), dtype=torch.uint8, device=dev)
    out = torch.empty_like(img)
    d = dp._desc(M, N, C, F, pitch=pitch, opitch=pitch)
    ctx.synth_frames_dev(d, 101, 0, img, None)
    nz, keep = dp.Context._noise(dp.NOISE_KEYED, dp.plane_seeds(42, F, C))
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    rows = []
    for b in (4, 8, 16, 32):
        for eps in (0.1, 1.0):
            p = dp.make_privacy_params(eps, 16, b)
            G = dp.grid_dims(M, N, b).grid_count()
            means = torch.zeros((F * C, G), dtype=torch.uint8, device=dev)
            for _ in range(3):
                ctx.pixelize_uniform_dev(d, img, p, nz, means, out)
            ctx.synchronize()
            ctx.reset_stats()
            ctx.set_timing(True)
            for _ in range(10):
                ctx.pixelize_uniform_dev(d, img, p, nz, means, out)
            ctx.synchronize()
            st = ctx.stats()
            ctx.set_timing(False)
            ms = st["device_ms"]["stats_tma"] / max(1, st["launches"]["stats_tma"])
            alg = F * M * N * C * 2 + F * C * G
            rows.append({"b": b, "eps": eps, "k1_ms": round(ms, 4),
                         "frac": round(alg / (ms / 1e3) / 1e9 / peak, 4),
                         "draws_per_frame": C * G})
    print(json.dumps(rows))


if __name__ == "__main__":
    main()
