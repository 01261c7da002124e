"""Which bytes outside [0, N*C) of each output row does each writer store, and
what values (diagnostic for tests/test_gpu_parity.py::test_default_stores_are_window_safe)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_04261_b200 as dp  # noqa: E402

ctx = dp.Context(0)
dev = torch.device("cuda:0")
cases = [(100, 301, 1, 4, 1, True), (100, 301, 1, 4, 1, False), (100, 301, 3, 4, 1, True),
         (100, 301, 1, 8, 2, True), (64, 250, 3, 30, 5, True), (100, 1000, 1, 4, 1, True)]
for (M, N, C, b, n, adaptive) in cases:
    F = 2
    row = N * C
    pitch = (row + 15) // 16 * 16
    mpitch = (N + 15) // 16 * 16
    left = 16
    opitch = (left + row + 7 + 15) // 16 * 16
    d = dp._desc(M, N, C, F, pitch=pitch, mpitch=mpitch, opitch=opitch)
    img = torch.empty((F, M, pitch), dtype=torch.uint8, device=dev)
    mask = torch.empty((F, M, mpitch), dtype=torch.uint8, device=dev)
    ctx.synth_frames_dev(d, 9, 0, img, mask)
    p = dp.make_privacy_params(0.5, 16, b, n if adaptive else 1)
    nz, keep = dp.Context._noise(dp.NOISE_KEYED, dp.plane_seeds(42, F, C))
    G = dp.grid_dims(M, N, b).grid_count()
    for pad in (False, True):
        ctx.set_out_pad_scratch(pad)
        for k in range(2):
            parent = torch.full((F, M, opitch), 0xA5, dtype=torch.uint8, device=dev)
            win = parent.view(-1)[left:]
            ctx.reset_stats()
            ctx.set_timing(True)
            if adaptive:
                cap = dp.adaptive_payload_capacity(M, N, b, n)
                stride = (cap + 15) // 16 * 16
                if k == 0:
                    payload = torch.zeros((F * C, stride), dtype=torch.uint8, device=dev)
                    lens = torch.zeros(F * C, dtype=torch.int32, device=dev)
                    ctx.pixelize_adaptive_dev(d, img, mask, p, nz, payload, stride, lens, win)
                else:
                    ctx.reassemble_dev(d, payload, stride, lens, b, n, win)
            else:
                if k == 0:
                    means = torch.zeros((F * C, G), dtype=torch.uint8, device=dev)
                    ctx.pixelize_uniform_dev(d, img, p, nz, means, win)
                else:
                    ctx.broadcast_means_dev(d, means, b, win)
            ctx.synchronize()
            st = {kk: v for kk, v in ctx.stats()["launches"].items() if v}
            ctx.set_timing(False)
            par = parent.cpu().numpy().reshape(F * M, opitch)
            after = par[:, left + row:]
            before = par[:, :left].copy()
            w = np.nonzero((after != 0xA5).any(axis=0))[0]
            vals = after[0, w].tolist() if len(w) else []
            pix = par[0, left + row - 4: left + row].tolist()
            print((M, N, C, b, n, "ad" if adaptive else "un"), "pad" if pad else "def",
                  "K1" if k == 0 else "K2", st, "after-row bytes written:", w.tolist()[:12],
                  "values", vals[:8], "last pixels", pix, "before-window written:",
                  int((before != 0xA5).sum()), flush=True)
ctx.set_out_pad_scratch(False)
