#!/usr/bin/env python3
"""The paper's PPM-100 (b, n) grid (b in {1, 2, 4, ..., 128},
n in {1, 2, 4, ..., b}), adaptive, on 4K RGB frames (config 4's shape),
device resident: K1 (and K0) time, kernel family, K1 fraction of HBM."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2511_04261_b200 as dp
    F, M, N, C = int(sys.argv[1]) if len(sys.argv) > 1 else 8, 2160, 3840, 3
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    dev = torch.device("cuda:0")
    ctx = dp.Context(0)
    ctx.set_out_pad_scratch(True)
    img = torch.empty((F, M, N * C), dtype=torch.uint8, device=dev)
    out = torch.empty_like(img)
    mask = torch.empty((F, M, N), dtype=torch.uint8, device=dev)
    d = dp._desc(M, N, C, F)
    ctx.synth_frames_dev(d, 101, 0, img, mask)
    nz, keep = dp.Context._noise(dp.NOISE_KEYED, dp.plane_seeds(42, F, C))
    rows = []
    b = 1
    while b <= 128:
        n = 1
        while n <= b:
            p = dp.make_privacy_params(0.5, 32, b, n)
            cap = dp.adaptive_payload_capacity(M, N, b, n)
            st = (cap + 15) // 16 * 16
            stats = torch.zeros((F * C, st), dtype=torch.uint8, device=dev)
            lens = torch.zeros(F * C, dtype=torch.int32, device=dev)
            ctx.pixelize_adaptive_dev(d, img, mask, p, nz, stats, st, lens, out)
            ctx.synchronize()
            ctx.reset_stats()
            ctx.set_timing(True)
            ctx.pixelize_adaptive_dev(d, img, mask, p, nz, stats, st, lens, out)
            ctx.synchronize()
            s = ctx.stats()
            ctx.set_timing(False)
            fam = [k for k, v in s["launches"].items() if v and k != "classify"]
            k1 = sum(s["device_ms"][k] for k in fam)
            pay = int(lens.sum().item())
            alg = F * M * N * C * 2 + pay
            # reconstruction (reassemble: K0 on the payload means + K2)
            ctx.reassemble_dev(d, stats, st, lens, b, n, out)
            ctx.synchronize()
            ctx.reset_stats()
            ctx.set_timing(True)
            ctx.reassemble_dev(d, stats, st, lens, b, n, out)
            ctx.synchronize()
            s2 = ctx.stats()
            ctx.set_timing(False)
            k2 = s2["device_ms"]["expand"]
            rows.append({"b": b, "n": n, "kernel": fam, "k1_ms": round(k1, 3),
                         "k0_ms": round(s["device_ms"]["classify"], 3),
                         "k1_frac": round(alg / (k1 / 1e3) / 1e9 / peak, 3),
                         "k2_ms": round(k2, 3),
                         "k2_frac": round((pay + F * M * N * C) / (k2 / 1e3) / 1e9 / peak, 3) if k2 else None})
            del stats, lens
            n *= 2
        b *= 2
    print(json.dumps(rows))


if __name__ == "__main__":
    main()
