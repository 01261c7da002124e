"""One K1 configuration on 1080p RGB frames, device resident, for ncu captures
of the draw-bound kernels (launch 1 is a warm-up, launch 2 the capture):

  ncu --set full -k regex:k_stats_tma -s 1 -c 1 python tools/k1_case.py --b 4 --n 1
  ncu --set full -k regex:k_stats_tma -s 1 -c 1 python tools/k1_case.py --b 16 --n 4 --complex 0.5
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=120)
    ap.add_argument("--b", type=int, default=4)
    ap.add_argument("--n", type=int, default=1)
    ap.add_argument("--eps", type=float, default=0.5)
    ap.add_argument("--complex", type=float, default=-1.0, help="random cell mask; < 0: ellipse")
    ap.add_argument("--launches", type=int, default=2)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--width", type=int, default=1920)
    args = ap.parse_args()
    import torch

    import paper_2511_04261_b200 as dp
    F, M, N, C, b, n = args.frames, args.height, args.width, 3, args.b, args.n
    dev = torch.device("cuda:0")
    ctx = dp.Context(0)
    img = torch.empty((F, M, N * C), dtype=torch.uint8, device=dev)
    out = torch.empty_like(img)
    mask = torch.empty((F, M, N), dtype=torch.uint8, device=dev)
    d = dp._desc(M, N, C, F)
    ctx.synth_frames_dev(d, 101, 0, img, mask)
    GR, GC = (M + b - 1) // b, (N + b - 1) // b
    if args.complex >= 0:
        gen = torch.Generator(device=dev).manual_seed(7)
        cells = (torch.rand((F, GR, GC), generator=gen, device=dev) >= args.complex).to(torch.uint8)
        mask.copy_(cells.repeat_interleave(b, 1).repeat_interleave(b, 2)[:, :M, :N])
    p = dp.make_privacy_params(args.eps, 16, b, n)
    nz, keep = dp.Context._noise(dp.NOISE_KEYED, dp.plane_seeds(42, F, C))
    adaptive = n > 1 or args.complex >= 0
    if adaptive:
        cap = dp.adaptive_payload_capacity(M, N, b, n)
        stride = (cap + 15) & ~15
        payload = torch.zeros((F * C, stride), dtype=torch.uint8, device=dev)
        lens = torch.zeros(F * C, dtype=torch.int32, device=dev)
        run = lambda: ctx.pixelize_adaptive_dev(d, img, mask, p, nz, payload, stride, lens, out)
    else:
        means = torch.zeros((F * C, GR * GC), dtype=torch.uint8, device=dev)
        run = lambda: ctx.pixelize_uniform_dev(d, img, p, nz, means, out)
    ctx.set_timing(True)
    for _ in range(args.launches):
        run()
    ctx.synchronize()
    st = ctx.stats()
    fam = max(("stats_tma", "stats_rows", "stats_generic"), key=lambda k: st["launches"].get(k, 0))
    k1 = st["device_ms"][fam] / max(1, st["launches"][fam])
    print(json.dumps({"b": b, "n": n, "complex": args.complex, "family": fam, "k1_ms_mean": round(k1, 4)}))


if __name__ == "__main__":
    main()
