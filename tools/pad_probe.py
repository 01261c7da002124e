"""Which output padding bytes do the kernels write? (pitch slack diagnostics)"""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
import paper_2511_04261_b200 as dp
ctx = dp.Context(0)
dev = torch.device('cuda:0')
for (M, N, C, b, n) in [(100, 301, 1, 4, 1), (64, 250, 3, 30, 5), (218, 178, 3, 16, 4), (83, 1917, 3, 8, 2)]:
    F = 7
    row = N * C
    pitch = (row + 15) // 16 * 16
    opitch = (row + 63) // 64 * 64 + 64
    mpitch = (N + 15) // 16 * 16
    d = dp._desc(M, N, C, F, pitch=pitch, mpitch=mpitch, opitch=opitch)
    img = torch.empty((F, M, pitch), dtype=torch.uint8, device=dev)
    mask = torch.empty((F, M, mpitch), dtype=torch.uint8, device=dev)
    ctx.synth_frames_dev(d, 5, 0, img, mask)
    p = dp.make_privacy_params(0.5, 16, b, n)
    cap = dp.adaptive_payload_capacity(M, N, b, n)
    stride = (cap + 15) // 16 * 16
    nz, keep = dp.Context._noise(dp.NOISE_KEYED, dp.plane_seeds(42, F, C))
    for on in (False, True):
        ctx.set_out_pad_scratch(on)
        payload = torch.zeros((F * C, stride), dtype=torch.uint8, device=dev)
        lens = torch.zeros(F * C, dtype=torch.int32, device=dev)
        o1 = torch.full((F, M, opitch), 0xA5, dtype=torch.uint8, device=dev)
        o2 = torch.full_like(o1, 0xA5)
        ctx.reset_stats(); ctx.set_timing(True)
        ctx.pixelize_adaptive_dev(d, img, mask, p, nz, payload, stride, lens, o1)
        ctx.synchronize(); s1 = {k: v for k, v in ctx.stats()['launches'].items() if v}
        ctx.reset_stats()
        ctx.reassemble_dev(d, payload, stride, lens, b, n, o2)
        ctx.synchronize(); s2 = {k: v for k, v in ctx.stats()['launches'].items() if v}
        ctx.set_timing(False)
        for name, o, s in (("K1", o1, s1), ("K2", o2, s2)):
            pad = o.cpu().numpy()[:, :, row:]
            w = np.nonzero((pad != 0xA5).any(axis=(0, 1)))[0]
            print((M, N, C, b, n), "on" if on else "off", name, s, "row", row,
                  "written pad offsets", (int(w.min()), int(w.max())) if len(w) else None, flush=True)
ctx.set_out_pad_scratch(False)
