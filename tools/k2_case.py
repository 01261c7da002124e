#!/usr/bin/env python3
"""One K2 reassemble configuration (device resident), for ncu captures and
A/B: python tools/k2_case.py M N F b n   (launch 1 warms up, then 3 timed)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2511_04261_b200 as dp
    M, N, F, b, n = (int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (2160, 3840, 32, 32, 8)))
    C = 3
    ctx = dp.Context(0)
    dev = torch.device("cuda:0")
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
    ctx.pixelize_adaptive_dev(d, img, mask, p, nz, stats, st, lens, out)
    ctx.reassemble_dev(d, stats, st, lens, b, n, out)
    ctx.synchronize()
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
    ctx.reset_stats()
    ctx.set_timing(True)
    for _ in range(3):
        ctx.reassemble_dev(d, stats, st, lens, b, n, out)
    ctx.synchronize()
    s = ctx.stats()
    k2 = s["device_ms"]["expand"] / s["launches"]["expand"]
    alg = F * M * N * C + int(lens.sum().item())
    print(json.dumps({"M": M, "N": N, "F": F, "b": b, "n": n, "k2_ms": round(k2, 4),
                      "frac": round(alg / (k2 / 1e3) / 1e9 / peak, 4)}))


if __name__ == "__main__":
    main()
