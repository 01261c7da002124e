#!/usr/bin/env python3
"""Randomized stress of the device entry points against the oracle (GPU box).

Each case draws a geometry (tiny to 1080p-wide, narrow frames, ragged sizes),
channels, frames, (b, n), noise, and a strided device layout: random row
pitch, frame stride and base misalignment for the frames, the mask and the
output, so every kernel variant (TMA fast path, packed slots, generic path)
and every alignment branch is exercised. Checks pixelize (uniform, adaptive),
then reassemble / broadcast back into another strided buffer.

usage: python tools/fuzz_gpu.py [--cases 500] [--seed 1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

FAST_BN = [(4, 1), (8, 1), (8, 2), (16, 1), (16, 2), (16, 4), (32, 1), (32, 2), (32, 4), (32, 8)]


def strided(torch, dev, rng, F, M, row, fill=0):
    """A device buffer holding F frames of M rows x `row` bytes at a random
    pitch / frame stride / base offset; returns (view_base_tensor, pitch, fstride)."""
    aligned = rng.random() < 0.6
    pitch = row + (0 if aligned and row % 16 == 0 else int(rng.integers(0, 24)))
    if aligned:
        pitch = (pitch + 15) // 16 * 16
    fstride = pitch * M + (0 if aligned else int(rng.integers(0, 40)))
    if aligned:
        fstride = (fstride + 15) // 16 * 16
    off = 0 if aligned else int(rng.integers(0, 16))
    buf = torch.full((off + fstride * F + 64,), fill, dtype=torch.uint8, device=dev)
    return buf[off:], pitch, fstride


def scatter(torch, view, frames, pitch, fstride):
    F, M, N, C = frames.shape
    host = view.cpu().numpy()
    for f in range(F):
        for i in range(M):
            host[f * fstride + i * pitch: f * fstride + i * pitch + N * C] = frames[f, i].reshape(-1)
    view.copy_(torch.from_numpy(host))


def gather(view, shape, pitch, fstride):
    import numpy as np
    F, M, N, C = shape
    host = view.cpu().numpy()
    out = np.zeros(shape, np.uint8)
    for f in range(F):
        for i in range(M):
            out[f, i] = host[f * fstride + i * pitch: f * fstride + i * pitch + N * C].reshape(N, C)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=500)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    import numpy as np
    import torch

    import oracle
    import paper_2511_04261_b200 as dp
    dev = torch.device("cuda:0")
    ctx = dp.Context(0)
    ctx.set_timing(True)  # per-family launch counts
    rng = np.random.default_rng(args.seed)
    fails = 0
    counts = {}
    for case in range(args.cases):
        u01 = rng.random()
        if u01 < 0.55:
            b, n = FAST_BN[rng.integers(len(FAST_BN))]
        else:
            b = int(rng.choice([12, 20, 24, 30, 40, 64, 128])) if u01 < 0.8 else int(rng.integers(1, 20))
            divs = [d for d in range(1, b + 1) if b % d == 0]
            n = int(rng.choice(divs))
        C = int(rng.choice([1, 3, 3, 4]))
        F = int(rng.integers(1, 5))
        wide = rng.random() < 0.2
        M = int(rng.integers(b, (1100 if wide else 3 * b + 40) + 1))
        N = int(rng.integers(b, (1950 if wide else 3 * b + 200) + 1))
        adaptive = n > 1 or rng.random() < 0.5
        kind = "keyed" if rng.random() < 0.8 else "none"
        p = dp.make_privacy_params(float(rng.choice([0.1, 0.5, 1.0])), 16, b, n)
        frames = rng.integers(0, 256, (F, M, N, C), np.uint8)
        masks = (rng.random((F, M, N)) < rng.random()).astype(np.uint8)
        seeds = dp.plane_seeds(int(rng.integers(0, 2**62)), F, C)
        nz, keep = dp.Context._noise(dp.NOISE_KEYED if kind == "keyed" else dp.NOISE_NONE,
                                     seeds if kind == "keyed" else None)
        img_v, pitch, fstride = strided(torch, dev, rng, F, M, N * C)
        scatter(torch, img_v, frames, pitch, fstride)
        out_v, opitch, ofstride = strided(torch, dev, rng, F, M, N * C, fill=7)
        ctx.reset_stats()
        tag = dict(case=case, M=M, N=N, C=C, F=F, b=b, n=n, adaptive=adaptive, kind=kind,
                   pitch=pitch, opitch=opitch)
        try:
            if adaptive:
                mask_v, mpitch, mfstride = strided(torch, dev, rng, F, M, N)
                scatter(torch, mask_v, masks[..., None], mpitch, mfstride)
                d = dp._desc(M, N, C, F, pitch, fstride, mpitch, mfstride, opitch, ofstride)
                cap = dp.adaptive_payload_capacity(M, N, b, n)
                sstride = (cap + 15) // 16 * 16
                payload = torch.zeros((F * C, sstride), dtype=torch.uint8, device=dev)
                lens = torch.zeros(F * C, dtype=torch.int32, device=dev)
                ctx.pixelize_adaptive_dev(d, img_v, mask_v, p, nz, payload, sstride, lens, out_v)
                ctx.synchronize()
                got = gather(out_v, frames.shape, opitch, ofstride)
                pl = payload.cpu().numpy()
                ln = lens.cpu().numpy()
                for f in range(F):
                    rp, ri = oracle.pixelize_adaptive(
                        frames[f], masks[f], b, n, p.sigma, p.sigma_sub, kind,
                        seeds[f * C:(f + 1) * C] if kind == "keyed" else None, frame=f)
                    assert [bytes(pl[f * C + c, :ln[f * C + c]]) for c in range(C)] == rp, "payload"
                    assert np.array_equal(got[f], ri), "image"
                # reassemble into a fresh strided buffer
                r_v, rpitch, rfstride = strided(torch, dev, rng, F, M, N * C, fill=3)
                dr = dp._desc(M, N, C, F, opitch=rpitch, ofstride=rfstride)
                ctx.reassemble_dev(dr, payload, sstride, lens, b, n, r_v)
                ctx.synchronize()
                assert np.array_equal(gather(r_v, frames.shape, rpitch, rfstride), got), "reassemble"
            else:
                d = dp._desc(M, N, C, F, pitch, fstride, opitch=opitch, ofstride=ofstride)
                G = dp.grid_dims(M, N, b).grid_count()
                means = torch.zeros((F * C, G), dtype=torch.uint8, device=dev)
                ctx.pixelize_uniform_dev(d, img_v, p, nz, means, out_v)
                ctx.synchronize()
                got = gather(out_v, frames.shape, opitch, ofstride)
                mh = means.cpu().numpy()
                for f in range(F):
                    rm, ri = oracle.pixelize_uniform(
                        frames[f], b, p.sigma, kind,
                        seeds[f * C:(f + 1) * C] if kind == "keyed" else None, frame=f)
                    assert np.array_equal(mh[f * C:(f + 1) * C], rm), "means"
                    assert np.array_equal(got[f], ri), "image"
                r_v, rpitch, rfstride = strided(torch, dev, rng, F, M, N * C, fill=3)
                dr = dp._desc(M, N, C, F, opitch=rpitch, ofstride=rfstride)
                ctx.broadcast_means_dev(dr, means, b, r_v)
                ctx.synchronize()
                assert np.array_equal(gather(r_v, frames.shape, rpitch, rfstride), got), "broadcast"
            st = ctx.stats()
            for k, v in st["launches"].items():
                counts[k] = counts.get(k, 0) + (1 if v else 0)
        except AssertionError as e:
            fails += 1
            print("FAIL", e, tag, flush=True)
        except (ValueError, RuntimeError) as e:
            fails += 1
            print("ERROR", e, tag, flush=True)
    print(f"fuzz: {args.cases} cases, {fails} failures, seed {args.seed}, kernels {counts}")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
