#!/usr/bin/env python3
"""K2 broadcast (broadcast_means_dev) per grid side on the sweep shape
(60 x 1917x1083 RGB, padded rows), with and without output pad scratch."""
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
    out = torch.empty((F, M, pitch), dtype=torch.uint8, device=dev)
    d = dp._desc(M, N, C, F, pitch=pitch, opitch=pitch)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    rows = []
    for pad in (True, False):
        ctx.set_out_pad_scratch(pad)
        for b in (4, 8, 16, 32):
            G = dp.grid_dims(M, N, b).grid_count()
            means = torch.randint(0, 256, (F * C, G), dtype=torch.uint8, device=dev)
            for _ in range(3):
                ctx.broadcast_means_dev(d, means, b, out)
            ctx.synchronize()
            ctx.reset_stats()
            ctx.set_timing(True)
            for _ in range(10):
                ctx.broadcast_means_dev(d, means, b, out)
            ctx.synchronize()
            st = ctx.stats()
            ctx.set_timing(False)
            ms = st["device_ms"]["expand"] / max(1, st["launches"]["expand"])
            alg = F * M * N * C + F * C * G
            rows.append({"pad_scratch": pad, "b": b, "k2_ms": round(ms, 4),
                         "frac": round(alg / (ms / 1e3) / 1e9 / peak, 4)})
    print(json.dumps(rows))


if __name__ == "__main__":
    main()
