#!/usr/bin/env python3
"""Device-resident throughput of the variance-classification extension
(no mask input): fused single pass (K1 VAR + K0 mode 3 + gather) vs the
2-pass path (K0 mode 2 reads the frames, then K1), on the venice shape.

usage (GPU box): python tools/variance_bench.py [--frames 600] [--tau 5000]
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
    ap.add_argument("--tau", type=float, default=5000.0)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--b", type=int, default=16)
    ap.add_argument("--n", type=int, default=4)
    args = ap.parse_args()
    import torch

    import paper_2511_04261_b200 as dp
    F, M, N, C, b, n = args.frames, 1080, 1920, 3, args.b, args.n
    dev = torch.device("cuda:0")
    ctx = dp.Context(0)
    pitch = N * C
    img = torch.empty((F, M, pitch), dtype=torch.uint8, device=dev)
    out = torch.empty_like(img)
    d = dp._desc(M, N, C, F)
    ctx.synth_frames_dev(d, 101, 0, img, None)
    p = dp.make_privacy_params(0.5, 16, b, n)
    cap = dp.adaptive_payload_capacity(M, N, b, n)
    stride = (cap + 15) & ~15
    payload = torch.zeros((F * C, stride), dtype=torch.uint8, device=dev)
    lens = torch.zeros(F * C, dtype=torch.int32, device=dev)
    nz, keep = dp.Context._noise(dp.NOISE_KEYED, dp.plane_seeds(42, F, C))
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    res = {}
    for mode in ("1", "0"):
        os.environ["DPPX_VAR_FUSED"] = mode
        for _ in range(3):
            ctx.pixelize_adaptive_variance_dev(d, img, args.tau, p, nz, payload, stride, lens, out)
        ctx.synchronize()
        ctx.reset_stats()
        ctx.set_timing(True)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        evs[0].record(stream)
        for i in range(args.steps):
            ctx.pixelize_adaptive_variance_dev(d, img, args.tau, p, nz, payload, stride, lens, out)
            evs[i + 1].record(stream)
        e0, e1 = evs[0], evs[-1]
        e1.synchronize()
        per = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
        st = ctx.stats()
        ctx.set_timing(False)
        ms = e0.elapsed_time(e1) / args.steps
        pay = int(lens.sum().item())
        alg = F * M * N * C * 2 + pay  # frames read once + image written + payloads
        res["fused" if mode == "1" else "two_pass"] = {
            "ms_per_step": round(ms, 4),
            "step_ms_min_max": [round(min(per), 4), round(max(per), 4)],
            "MP_per_s": round(F * M * N / 1e6 / (ms / 1e3), 1),
            "fps": round(F / (ms / 1e3), 1),
            "algorithmic_GB": round(alg / 1e9, 3),
            "step_frac_of_hbm": round(alg / (ms / 1e3) / 1e9 / peak, 4),
            "kernel_ms": {k: round(v / args.steps, 4) for k, v in st["device_ms"].items() if v},
            "launches": {k: v // args.steps for k, v in st["launches"].items() if v},
        }
    del os.environ["DPPX_VAR_FUSED"]
    S = int.from_bytes(payload[0, 4 * dp.grid_dims(M, N, b).grid_count():][:4].cpu().numpy()
                       .tobytes(), "little")
    print(json.dumps({"workload": f"{F} x {N}x{M} RGB, variance classification b{b} n{n} "
                      f"tau={args.tau}", "simple_cells_plane0": S,
                      "peak_gbs": peak, **res}))


if __name__ == "__main__":
    main()
