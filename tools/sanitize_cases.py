"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family on aligned, padded, packed-slot, split-strip
and rows shapes, out-pad-scratch off and on, the host pipeline (pinned and
pageable, dense re-pitch, row bands), the fused variance path, metrics, a
malformed reassemble payload. Each result is checked against the oracle, so a
sanitizer-clean run is also a parity run.

usage (under gpurun): compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (checker only)
import paper_2511_04261_b200 as dp  # noqa: E402

QUICK = os.environ.get("SAN_QUICK") == "1"


def adaptive_case(ctx, M, N, C, b, n, F=2, kind="keyed"):
    frames = oracle.synth_frames(3, F, M, N, C)
    masks = oracle.synth_masks(3, F, M, N)
    p = dp.make_privacy_params(0.5, 16, b, n)
    seeds = dp.plane_seeds(77, F, C)
    pls, img = ctx.pixelize_adaptive(frames, masks, p, dp.NOISE_KEYED if kind == "keyed" else dp.NOISE_NONE,
                                     seeds if kind == "keyed" else None)
    for f in range(F):
        rp, ri = oracle.pixelize_adaptive(frames[f], masks[f], b, n, p.sigma, p.sigma_sub, kind,
                                          seeds[f * C:(f + 1) * C] if kind == "keyed" else None)
        assert pls[f * C:(f + 1) * C] == rp and np.array_equal(img[f], ri), ("adaptive", M, N, C, b, n)
    back = ctx.reassemble(pls, M, N, b, n, channels=C, frames=F)
    assert np.array_equal(back, img), ("reassemble", M, N, C, b, n)
    return ctx.stats()["launches"]


def uniform_case(ctx, M, N, C, b, F=2):
    frames = oracle.synth_frames(4, F, M, N, C)
    p = dp.make_privacy_params(0.5, 16, b)
    seeds = dp.plane_seeds(5, F, C)
    means, img = ctx.pixelize_uniform(frames, p, dp.NOISE_KEYED, seeds)
    for f in range(F):
        rm, ri = oracle.pixelize_uniform(frames[f], b, p.sigma, "keyed", seeds[f * C:(f + 1) * C])
        assert np.array_equal(means[f * C:(f + 1) * C], rm) and np.array_equal(img[f], ri), \
            ("uniform", M, N, C, b)
    back = ctx.broadcast_means(means, M, N, b, channels=C, frames=F)
    assert np.array_equal(back, img), ("broadcast", M, N, C, b)


def main():
    ctx = dp.Context(0)
    cases_ad = [
        (72, 136, 3, 16, 4), (64, 128, 1, 16, 4), (67, 131, 3, 8, 2), (40, 96, 3, 12, 3),   # K1
        (57, 131, 3, 24, 4), (57, 131, 1, 16, 8),                                           # split strips
        (64, 250, 3, 30, 5), (150, 301, 3, 128, 32),                                        # K1a / K2a
        (150, 301, 3, 128, 8), (61, 253, 3, 40, 8),                                         # K1r / K2r
        (218, 178, 3, 16, 4), (20, 7, 3, 4, 2),                                             # packed, generic
        (300, 299, 1, 64, 16),
    ]
    cases_un = [(83, 1917, 3, 4), (83, 1917, 3, 32), (61, 253, 3, 7), (61, 253, 3, 30),
                (61, 253, 1, 128), (218, 178, 3, 16), (33, 45, 3, 5)]
    if QUICK:
        cases_ad, cases_un = cases_ad[:4] + cases_ad[6:8], cases_un[:3]
    for pad in (False, True):
        ctx.set_out_pad_scratch(pad)
        for c in cases_ad:
            adaptive_case(ctx, *c)
        for c in cases_un:
            uniform_case(ctx, *c)
    ctx.set_out_pad_scratch(False)
    # Algorithm 1
    frames = oracle.synth_frames(6, 1, 61, 99, 1)
    p = dp.make_privacy_params(0.5, 16, 16)
    _, img = ctx.pixelize_reference(frames, p, dp.NOISE_KEYED, [11])
    ri = oracle.pixelize_reference(frames[0][..., 0], 16, p.sigma, 11)
    assert np.array_equal(img[0][..., 0], ri)
    # host pipeline: many frames (chunks), pageable, dense 534-byte rows (re-pitch)
    adaptive_case(ctx, 218, 178, 3, 16, 4, F=9)
    uniform_case(ctx, 218, 178, 3, 16, F=9)
    # single-frame row bands (>= 4 MB frame, pinned buffers)
    M, N, C = 1080, 1920, 3
    fr = dp.pinned_empty((1, M, N, C))
    fr[:] = oracle.synth_frames(8, 1, M, N, C)
    mk = dp.pinned_empty((1, M, N))
    mk[:] = oracle.synth_masks(8, 1, M, N)
    out = dp.pinned_empty((1, M, N, C))
    p = dp.make_privacy_params(0.5, 16, 16, 4)
    seeds = dp.plane_seeds(42, 1, C)
    pls, img = ctx.pixelize_adaptive(fr, mk, p, dp.NOISE_KEYED, seeds, out=out)
    rp, ri = oracle.pixelize_adaptive(fr[0], mk[0], 16, 4, p.sigma, p.sigma_sub, "keyed", seeds)
    assert pls == rp and np.array_equal(img[0], ri), "bands"
    # fused variance classification
    frames = oracle.synth_frames(2, 2, 64, 128, 3)
    p = dp.make_privacy_params(0.5, 16, 16, 4)
    pls, img = ctx.pixelize_adaptive_variance(frames, 800.0, p, dp.NOISE_KEYED, dp.plane_seeds(3, 2, 3))
    # metrics
    a = oracle.synth_frames(1, 1, 80, 90, 3)
    b = oracle.synth_frames(2, 1, 80, 90, 3)
    ctx.metrics(a, b, "both")
    # malformed reassemble payload: RecordError, no out-of-bounds read
    M, N, b_, n_ = 150, 301, 16, 4
    G = dp.grid_dims(M, N, b_).grid_count()
    bad = [bytes(5 * G + 4)] * 3
    try:
        ctx.reassemble(bad, M, N, b_, n_, channels=3, frames=1, check_lengths=False)
        raise AssertionError("malformed payload accepted")
    except dp.RecordError:
        pass
    ctx.synchronize()
    print("sanitize cases ok:", ctx.stats()["launches"])
    ctx.close()


if __name__ == "__main__":
    main()
