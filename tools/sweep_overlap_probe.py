#!/usr/bin/env python3
"""Does the one-read sweep overlap its draws with its broadcasts? Times (CUDA
events on the ctx stream, 60 x 1917x1083 RGB, 12 runs): the whole step, the
step without images (sums + draws), and the 12 broadcasts alone."""
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
    ctx.set_out_pad_scratch(True)
    pitch = (N * C + 15) // 16 * 16
    img = torch.empty((F, M, pitch), dtype=torch.uint8, device=dev)
    d = dp._desc(M, N, C, F, pitch=pitch, opitch=pitch)
    ctx.synth_frames_dev(d, 7, 0, img, None)
    nz, keep = dp.Context._noise(dp.NOISE_KEYED, dp.plane_seeds(42, F, C))
    bl, el = [4, 8, 16, 32], [0.1, 0.5, 1.0]
    means = [torch.zeros((F * C, dp.grid_dims(M, N, b).grid_count()), dtype=torch.uint8, device=dev)
             for b in bl for _ in el]
    outs = [torch.empty_like(img) for _ in range(12)]
    s = torch.cuda.ExternalStream(ctx.stream) if ctx.stream else torch.cuda.current_stream()

    def timed(fn, reps=10):
        for _ in range(3):
            fn()
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps

    full = timed(lambda: ctx.pixelize_uniform_sweep_dev(d, img, bl, el, 16, nz, means, outs))
    noimg = timed(lambda: ctx.pixelize_uniform_sweep_dev(d, img, bl, el, 16, nz, means, None))

    def bcast():
        k = 0
        for b in bl:
            for _ in el:
                ctx.broadcast_means_dev(d, means[k], b, outs[k])
                k += 1
    bc = timed(bcast)
    # the same two halves from two contexts (two streams), forced concurrent
    ctx2 = dp.Context(0)
    ctx2.set_out_pad_scratch(True)
    s2 = torch.cuda.ExternalStream(ctx2.stream)

    def bcast2():
        k = 0
        for b in bl:
            for _ in el:
                ctx2.broadcast_means_dev(d, means[k], b, outs[k])
                k += 1

    def both():
        ev = torch.cuda.Event()
        ev.record(s)
        s2.wait_event(ev)
        bcast2()
        ctx.pixelize_uniform_sweep_dev(d, img, bl, el, 16, nz, means, None)
        ev2 = torch.cuda.Event()
        ev2.record(s2)
        s.wait_event(ev2)
    conc = timed(both)
    print(json.dumps({"concurrent_two_ctx_ms": round(conc, 4)}))
    print(json.dumps({"step_ms": round(full, 4), "sums_draws_ms": round(noimg, 4), "broadcasts_ms": round(bc, 4),
                      "serial_sum_ms": round(noimg + bc, 4), "overlap_ms": round(noimg + bc - full, 4),
                      "l0_ctas": os.environ.get("DPPX_SWEEP_L0_CTAS", "3")}))


if __name__ == "__main__":
    main()
