"""Memory-safety and race checks of every kernel family without
compute-sanitizer (closed on this GPU pool: profiles/r02_sanitizer.txt).

* Reads: every input (frames, masks, payload slots) lives inside a larger
  device buffer whose bytes outside the described extents -- guard bands
  before and after, pitch slack, gaps between frames and slots -- are filled
  with a poison byte. Each case runs twice with different poison; any read of
  a byte the descriptor does not cover that influences a result shows up as a
  difference (and as a mismatch with the oracle).
* Writes: outputs (image windows, payload slots, means) sit in canary-filled
  parent buffers; every byte outside the described extents must keep its
  canary, and payload slot bytes past each plane's length too.
* Races: each case runs three times (different poison, the persistent K1's
  dynamic unit claims land differently) and must give identical bytes.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

import paper_2511_04261_b200 as dp

CASES = [  # (M, N, C, b, n, adaptive) -- one or more per kernel family
    (72, 136, 3, 16, 4, True), (64, 128, 1, 16, 4, True), (67, 131, 3, 8, 2, True),      # K1 / K2
    (40, 96, 3, 12, 3, True), (57, 131, 3, 24, 4, True), (57, 131, 1, 16, 8, True),      # LPW, split
    (64, 250, 3, 30, 5, True), (150, 301, 3, 128, 32, True),                            # K1a / K2a
    (150, 301, 3, 128, 8, True), (61, 253, 3, 40, 8, True),                             # K1r / K2r
    (218, 178, 3, 16, 4, True), (218, 178, 3, 16, 1, False), (20, 7, 3, 4, 2, True),    # packed, K1g
    (83, 1917, 3, 4, 1, False), (61, 253, 3, 7, 1, False), (150, 253, 1, 128, 1, False),  # K1 / K1u
    (33, 45, 3, 5, 1, False), (100, 301, 1, 4, 1, True), (70, 203, 3, 64, 16, True),
    (70, 203, 3, 16, 16, True), (57, 131, 3, 8, 4, True), (40, 150, 1, 32, 16, True),  # in-lane 1-2 px
    (218, 178, 3, 16, 8, True), (218, 178, 3, 8, 4, True), (218, 178, 1, 16, 16, True),  # packed STR / 1 px
    (20, 77, 3, 16, 2, True),                                                          # K0 per frame
]
GUARD = 4096


class Region:
    """A described 3-D byte region (F x rows x width, pitch, frame stride)
    inside a poisoned / canaried parent buffer."""

    def __init__(self, torch, dev, F, rows, width, pitch, fstride, fill):
        self.F, self.rows, self.width, self.pitch, self.fstride = F, rows, width, pitch, fstride
        self.size = GUARD + F * fstride + GUARD
        self.parent = torch.full((self.size,), fill, dtype=torch.uint8, device=dev)
        self.view = self.parent[GUARD:]

    def inside(self):
        m = np.zeros(self.size, bool)
        for f in range(self.F):
            for i in range(self.rows):
                o = GUARD + f * self.fstride + i * self.pitch
                m[o:o + self.width] = True
        return m

    def put(self, arr):  # arr: F x rows x width
        host = self.parent.cpu().numpy()
        for f in range(self.F):
            for i in range(self.rows):
                o = GUARD + f * self.fstride + i * self.pitch
                host[o:o + self.width] = arr[f, i]
        self.parent.copy_(self.parent.new_tensor(host))

    def get(self):
        host = self.parent.cpu().numpy()
        out = np.empty((self.F, self.rows, self.width), np.uint8)
        for f in range(self.F):
            for i in range(self.rows):
                o = GUARD + f * self.fstride + i * self.pitch
                out[f, i] = host[o:o + self.width]
        return out, host


def _geometry(M, N, C):
    row = N * C
    pitch = (row + 15) // 16 * 16 + 16       # slack that is not the kernels' own padding
    fstride = M * pitch + 48                 # gap between frames (16-B aligned)
    mpitch = (N + 15) // 16 * 16 + 16
    mfstride = M * mpitch + 32
    return row, pitch, fstride, mpitch, mfstride


@pytest.mark.parametrize("M,N,C,b,n,adaptive", CASES)
@pytest.mark.parametrize("pad_scratch", [False, True])
def test_poisoned_inputs_and_canaried_outputs(ctx, M, N, C, b, n, adaptive, pad_scratch):
    import torch
    dev = torch.device("cuda:0")
    F = 3
    row, pitch, fstride, mpitch, mfstride = _geometry(M, N, C)
    frames = oracle.synth_frames(21, F, M, N, C)
    masks = oracle.synth_masks(21, F, M, N)
    p = dp.make_privacy_params(0.5, 16, b, n if adaptive else 1)
    seeds = dp.plane_seeds(7, F, C)
    nz, keep = dp.Context._noise(dp.NOISE_KEYED, seeds)
    G = dp.grid_dims(M, N, b).grid_count()
    d = dp._desc(M, N, C, F, pitch=pitch, fstride=fstride, mpitch=mpitch, mfstride=mfstride,
                 opitch=pitch, ofstride=fstride)
    if adaptive:
        cap = dp.adaptive_payload_capacity(M, N, b, n)
        sstride = (cap + 15) // 16 * 16 + 16
    else:
        sstride = G
    CANARY = 0x5A
    runs = []
    ctx.set_out_pad_scratch(pad_scratch)
    try:
        for poison in (0x00, 0xFF, 0x81):
            img = Region(torch, dev, F, M, row, pitch, fstride, poison)
            img.put(frames.reshape(F, M, row))
            msk = Region(torch, dev, F, M, N, mpitch, mfstride, poison ^ 1)
            msk.put(masks)
            out = Region(torch, dev, F, M, row, pitch, fstride, CANARY)
            stats = Region(torch, dev, 1, F * C, sstride, sstride, F * C * sstride, CANARY)
            lens = torch.zeros(F * C, dtype=torch.int32, device=dev)
            if adaptive:
                ctx.pixelize_adaptive_dev(d, img.view, msk.view, p, nz, stats.view, sstride, lens,
                                          out.view)
            else:
                ctx.pixelize_uniform_dev(d, img.view, p, nz, stats.view, out.view)
            ctx.synchronize()
            o, ohost = out.get()
            s, shost = stats.get()
            ln = lens.cpu().numpy()
            # writes stay inside the output windows (pad scratch: up to the sector end)
            allowed = out.inside()
            if pad_scratch:
                for f in range(F):
                    for i in range(M):
                        a = GUARD + f * fstride + i * pitch
                        allowed[a:a + min(pitch, (row + 31) // 32 * 32)] = True
            assert (ohost[~allowed] == CANARY).all(), "K1 image store outside its window"
            sin = np.zeros(stats.size, bool)
            for q in range(F * C):
                used = int(ln[q]) if adaptive else G
                sin[GUARD + q * sstride:GUARD + q * sstride + used] = True
            assert (shost[~sin] == CANARY).all(), "statistics store outside the payloads"
            # K2 from the poisoned statistics (slot slack past each length poisoned)
            src = Region(torch, dev, 1, F * C, sstride, sstride, F * C * sstride, poison)
            sarr = s.copy()
            if adaptive:
                for q in range(F * C):
                    sarr[0, q, int(ln[q]):] = poison
            src.put(sarr)
            out2 = Region(torch, dev, F, M, row, pitch, fstride, CANARY)
            if adaptive:
                ctx.reassemble_dev(d, src.view, sstride, lens, b, n, out2.view)
            else:
                ctx.broadcast_means_dev(d, src.view, b, out2.view)
            ctx.synchronize()
            o2, o2host = out2.get()
            assert (o2host[~allowed] == CANARY).all(), "K2 store outside its window"
            assert np.array_equal(o2, o), "K2 != K1 image"
            payloads = [bytes(s[0, q, :int(ln[q])]) for q in range(F * C)] if adaptive else s
            runs.append((o, payloads))
    finally:
        ctx.set_out_pad_scratch(False)
    for o, pl in runs[1:]:  # independent of the poison and of the unit schedule
        assert np.array_equal(o, runs[0][0])
        assert (pl == runs[0][1]) if adaptive else np.array_equal(pl, runs[0][1])
    o, pl = runs[0]
    for f in range(F):
        sd = seeds[f * C:(f + 1) * C]
        if adaptive:
            rp, ri = oracle.pixelize_adaptive(frames[f], masks[f], b, n, p.sigma, p.sigma_sub, "keyed", sd)
            assert pl[f * C:(f + 1) * C] == rp
        else:
            rm, ri = oracle.pixelize_uniform(frames[f], b, p.sigma, "keyed", sd)
            assert np.array_equal(pl[0, f * C:(f + 1) * C], rm)
        assert np.array_equal(o[f].reshape(M, N, C), ri)
