#!/usr/bin/env python3
"""K1 time and roofline fraction across grid sizes the paper recommends
(PAPER.md: b = 8, 12, 16, 24 for PETS; 12, 24, 30, 40 for Venice-2; up to
b = 128, n <= 128 for PPM-100), device-resident 1080p RGB, 120 frames.
usage: b_sweep.py [frames] [uniform]   (uniform: b = 2..20, 30, 128 with n = 1)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = [(12, 1), (12, 3), (16, 4), (16, 8), (32, 8), (20, 1), (20, 5), (24, 1), (24, 3), (24, 4), (30, 5), (40, 1),
         (40, 2), (40, 4), (40, 5), (64, 1), (64, 4), (64, 8), (64, 16), (128, 1), (128, 8), (128, 16),
         (128, 32), (128, 128), (128, 2), (128, 4), (30, 2), (30, 3), (30, 6), (30, 10),
         (4, 4), (8, 8), (16, 16), (32, 32)]  # n = b: 1-px subcells


def main():
    import torch

    import paper_2511_04261_b200 as dp
    F, M, N, C = int(sys.argv[1]) if len(sys.argv) > 1 else 120, 1080, 1920, 3
    cases = CASES
    if len(sys.argv) > 2 and sys.argv[2] == "uniform":  # the paper's b = 2..20 sweep (+ 30, 128)
        cases = [(b, 1) for b in list(range(2, 21)) + [30, 128]]
    dev = torch.device("cuda:0")
    ctx = dp.Context(0)
    img = torch.empty((F, M, N * C), dtype=torch.uint8, device=dev)
    out = torch.empty_like(img)
    mask = torch.empty((F, M, N), dtype=torch.uint8, device=dev)
    d = dp._desc(M, N, C, F)
    ctx.synth_frames_dev(d, 101, 0, img, mask)
    nz, keep = dp.Context._noise(dp.NOISE_KEYED, dp.plane_seeds(42, F, C))
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    rows = []
    for b, n in cases:
        p = dp.make_privacy_params(0.5, 16, b, n)
        G = dp.grid_dims(M, N, b).grid_count()
        adaptive = n > 1
        if adaptive:
            cap = dp.adaptive_payload_capacity(M, N, b, n)
            st = (cap + 15) // 16 * 16
            stats = torch.zeros((F * C, st), dtype=torch.uint8, device=dev)
            lens = torch.zeros(F * C, dtype=torch.int32, device=dev)
            call = lambda: ctx.pixelize_adaptive_dev(d, img, mask, p, nz, stats, st, lens, out)
        else:
            stats = torch.zeros((F * C, G), dtype=torch.uint8, device=dev)
            call = lambda: ctx.pixelize_uniform_dev(d, img, p, nz, stats, out)
        for _ in range(2):
            call()
        ctx.synchronize()
        ctx.reset_stats()
        ctx.set_timing(True)
        for _ in range(5):
            call()
        ctx.synchronize()
        s = ctx.stats()
        ctx.set_timing(False)
        fam = ("stats_tma" if s["launches"]["stats_tma"] else
               "stats_rows" if s["launches"]["stats_rows"] else "stats_generic")
        ms = s["device_ms"][fam] / max(1, s["launches"][fam])
        pay = int(lens.sum().item()) if adaptive else F * C * G
        alg = F * M * N * C * 2 + pay
        # reconstruction from the statistics (K0 on the payload + K2 / K2r);
        # one untimed call first (lazy module loading of the expand kernel)
        if adaptive:
            ctx.reassemble_dev(d, stats, st, lens, b, n, out)
        else:
            ctx.broadcast_means_dev(d, stats, b, out)
        ctx.synchronize()
        ctx.reset_stats()
        ctx.set_timing(True)
        for _ in range(3):
            if adaptive:
                ctx.reassemble_dev(d, stats, st, lens, b, n, out)
            else:
                ctx.broadcast_means_dev(d, stats, b, out)
        ctx.synchronize()
        s2 = ctx.stats()
        ctx.set_timing(False)
        k2 = s2["device_ms"]["expand"] / max(1, s2["launches"]["expand"])
        k0 = s["device_ms"]["classify"] / max(1, s["launches"]["classify"])
        rows.append({"b": b, "n": n, "kernel": fam, "k1_ms": round(ms, 4), "k0_ms": round(k0, 4),
                     "k0_frac": round(F * M * N / (k0 / 1e3) / 1e9 / peak, 4) if adaptive else None,
                     "frac": round(alg / (ms / 1e3) / 1e9 / peak, 4),
                     "k2_ms": round(k2, 4),
                     "k2_frac": round((F * M * N * C + pay) / (k2 / 1e3) / 1e9 / peak, 4)})
    print(json.dumps(rows))


if __name__ == "__main__":
    main()
