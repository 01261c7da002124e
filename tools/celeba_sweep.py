#!/usr/bin/env python3
"""The paper's CelebA face experiment grid: adaptive
pixelization of 178x218 RGB faces at b in {4,8,12,16,20} (n = 4) and
n in {1,2,4,8,16} (b = 16), device resident, 20 000 frames: K0 + K1 time,
the kernel family used, and the K1 fraction of measured HBM."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2511_04261_b200 as dp
    F, M, N, C = int(sys.argv[1]) if len(sys.argv) > 1 else 20000, 218, 178, 3
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    dev = torch.device("cuda:0")
    ctx = dp.Context(0)
    ctx.set_out_pad_scratch(True)
    pitch = (N * C + 15) // 16 * 16
    img = torch.empty((F, M, pitch), dtype=torch.uint8, device=dev)
    out = torch.empty_like(img)
    mask = torch.empty((F, M, N), dtype=torch.uint8, device=dev)
    d = dp._desc(M, N, C, F, pitch=pitch, opitch=pitch)
    ctx.synth_frames_dev(d, 101, 0, img, mask)
    nz, keep = dp.Context._noise(dp.NOISE_KEYED, dp.plane_seeds(42, F, C))
    rows = []
    for b, n in [(4, 4), (8, 4), (12, 4), (16, 4), (20, 4), (16, 1), (16, 2), (16, 8), (16, 16)]:
        p = dp.make_privacy_params(5.0, 16, b, n)
        cap = dp.adaptive_payload_capacity(M, N, b, n)
        st = (cap + 15) // 16 * 16
        stats = torch.zeros((F * C, st), dtype=torch.uint8, device=dev)
        lens = torch.zeros(F * C, dtype=torch.int32, device=dev)
        ctx.pixelize_adaptive_dev(d, img, mask, p, nz, stats, st, lens, out)
        ctx.synchronize()
        ctx.reset_stats()
        ctx.set_timing(True)
        for _ in range(3):
            ctx.pixelize_adaptive_dev(d, img, mask, p, nz, stats, st, lens, out)
        ctx.synchronize()
        s = ctx.stats()
        ctx.set_timing(False)
        fams = {k: v for k, v in s["launches"].items() if v}
        k1f = [k for k in fams if k != "classify"]
        k1 = sum(s["device_ms"][k] for k in k1f) / 3
        k0 = s["device_ms"]["classify"] / max(1, s["launches"]["classify"])
        alg = F * M * N * C * 2 + int(lens.sum().item())
        # reassembly (K0 from the payloads + K2)
        ctx.reassemble_dev(d, stats, st, lens, b, n, out)
        ctx.synchronize()
        ctx.reset_stats()
        ctx.set_timing(True)
        for _ in range(3):
            ctx.reassemble_dev(d, stats, st, lens, b, n, out)
        ctx.synchronize()
        s2 = ctx.stats()
        ctx.set_timing(False)
        k2 = s2["device_ms"]["expand"] / max(1, s2["launches"]["expand"])
        k0r = s2["device_ms"]["classify"] / max(1, s2["launches"]["classify"])
        k2alg = F * M * N * C + int(lens.sum().item())
        rows.append({"b": b, "n": n, "kernels": fams, "k1_ms": round(k1, 4), "k0_ms": round(k0, 4),
                     "k1_frac": round(alg / (k1 / 1e3) / 1e9 / peak, 4), "k2_ms": round(k2, 4),
                     "k0r_ms": round(k0r, 4), "k2_frac": round(k2alg / (k2 / 1e3) / 1e9 / peak, 4)})
        del stats, lens
    print(json.dumps(rows))


if __name__ == "__main__":
    main()
