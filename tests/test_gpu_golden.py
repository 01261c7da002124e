"""The GPU path reproduces the fixtures generated from the reference itself
(tests/golden/, see make_golden.py): small random cases through the
reference-shaped API, BASELINE shapes as RGB batches with derived plane seeds."""
import hashlib
import os

import numpy as np
import pytest

import oracle
import paper_2511_04261_b200 as dp

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_device_noise_equals_reference_golden_draws(ctx):
    """Laplace doubles drawn on the device == the reference's laplace_at values
    recorded in noise.json (bit for bit, incl. the log1p evaluation)."""
    import json
    d = json.load(open(os.path.join(G, "noise.json")))
    for v in d["draws"]:
        got = ctx.device_laplace(int(v["seed"]), np.array([v["key"]], np.uint32), v["sigma"])[0]
        assert got == float.fromhex(v["laplace"]), v


def test_small_cases_through_dropin_api(ctx):
    z = np.load(os.path.join(G, "small_cases.npz"))
    for k in sorted({k.split("_")[0] for k in z.files}):
        M, N, b, n, m, has = (int(x) for x in z[f"{k}_params"])
        eps = float(z[f"{k}_eps"][0])
        seed = None if has < 0 else int(z[f"{k}_seed"][0])
        u = dp.pixelize_parallel(z[f"{k}_img"], dp.make_privacy_params(eps, m, b), seed)
        assert np.array_equal(u.means.values, z[f"{k}_umeans"]) and np.array_equal(u.image, z[f"{k}_uimg"]), k
        a = dp.pixelize_adaptive(z[f"{k}_img"], z[f"{k}_mask"], dp.make_privacy_params(eps, m, b, n), seed)
        assert a.means.payload() == z[f"{k}_payload"].tobytes() and np.array_equal(a.image, z[f"{k}_aimg"]), k
        assert np.array_equal(dp.reassemble(a.means, M, N), a.image)
        assert np.array_equal(dp.broadcast_means(u.means, M, N), u.image)


def test_shaped_cases_rgb(ctx):
    z = np.load(os.path.join(G, "shaped_cases.npz"))
    for name in sorted({k.rsplit("_", 1)[0] for k in z.files if k.endswith("_spec")}):
        M, N, b, n, m = (int(x) for x in z[f"{name}_spec"])
        eps = float(z[f"{name}_eps"][0])
        frames = oracle.synth_frames(3, 1, M, N, 3)
        masks = oracle.synth_masks(3, 1, M, N)
        seeds = dp.plane_seeds(42, 1, 3, frame0=3)
        if f"{name}_ch0_payload" in z.files:
            pls, img = ctx.pixelize_adaptive(frames, masks, dp.make_privacy_params(eps, m, b, n),
                                             dp.NOISE_KEYED, seeds)
            for ch in range(3):
                assert pls[ch] == z[f"{name}_ch{ch}_payload"].tobytes(), (name, ch)
        else:
            means, img = ctx.pixelize_uniform(frames, dp.make_privacy_params(eps, m, b),
                                              dp.NOISE_KEYED, seeds)
            for ch in range(3):
                assert np.array_equal(means[ch], z[f"{name}_ch{ch}_means"]), (name, ch)
        for ch in range(3):
            plane = np.ascontiguousarray(img[0, :, :, ch])
            assert hashlib.sha256(plane.tobytes()).digest() == z[f"{name}_ch{ch}_imgsha"].tobytes()


def test_algorithm1_reference_path(ctx):
    """pixelize_reference (Algorithm 1, partial border grids) vs the reference
    itself on the 40 golden cases, and == pixelize_parallel when b | M, N."""
    z = np.load(os.path.join(G, "small_cases.npz"))
    for k in sorted({k.split("_")[0] for k in z.files}):
        M, N, b, n, m, has = (int(x) for x in z[f"{k}_params"])
        eps = float(z[f"{k}_eps"][0])
        seed = None if has < 0 else int(z[f"{k}_seed"][0])
        out = dp.pixelize_reference(z[f"{k}_img"], dp.make_privacy_params(eps, m, b), seed)
        assert np.array_equal(out, z[f"{k}_refimg"]), k
    rng = np.random.default_rng(21)  # test_pixelize.cpp:92-106
    for _ in range(10):
        b = 1 << int(rng.integers(0, 4))
        M, N = b * int(rng.integers(1, 13)), b * int(rng.integers(1, 13))
        img = rng.integers(0, 256, (M, N), dtype=np.uint8)
        p = dp.make_privacy_params(0.5, 16, b)
        s = int(rng.integers(0, 2**62))
        assert np.array_equal(dp.pixelize_reference(img, p, s), dp.pixelize_parallel(img, p, s).image)


def test_metrics_bit_identical_to_reference(ctx):
    """mse / ssim on the GPU == the reference's metrics.cpp (via the oracle,
    pinned to the reference in tests/test_oracle_vs_ref.py), bit for bit."""
    rng = np.random.default_rng(17)
    for M, N in [(7, 7), (19, 33), (218, 178), (576, 768)]:
        a = rng.integers(0, 256, (M, N), dtype=np.uint8)
        b = np.clip(a.astype(int) + rng.integers(-40, 40, (M, N)), 0, 255).astype(np.uint8)
        assert dp.mse(a, b) == oracle.mse(a, b)
        assert dp.ssim(a, b) == oracle.ssim(a, b)
        assert dp.ssim(a, a) == 1.0
    # RGB batches: per channel plane
    frames = oracle.synth_frames(0, 2, 64, 96, 3)
    p = dp.make_privacy_params(0.5, 16, 8, 2)
    masks = oracle.synth_masks(0, 2, 64, 96)
    _, out = ctx.pixelize_adaptive(frames, masks, p, dp.NOISE_KEYED, dp.plane_seeds(1, 2, 3))
    s = ctx.metrics(frames, out, "ssim")
    m = ctx.metrics(frames, out, "mse")
    m2, s2 = ctx.metrics(frames, out, "both")
    assert np.array_equal(m2, m) and np.array_equal(s2, s)
    for f in range(2):
        for c in range(3):
            assert s[f * 3 + c] == oracle.ssim(frames[f, :, :, c], out[f, :, :, c])
            assert m[f * 3 + c] == oracle.mse(frames[f, :, :, c], out[f, :, :, c])
    with pytest.raises(ValueError):
        dp.ssim(np.zeros((6, 9), np.uint8), np.zeros((6, 9), np.uint8))


@pytest.mark.gpu
@pytest.mark.parametrize("C", [1, 3])
def test_ssim_ragged_bands_and_chunks(ctx, C):
    """The band SSIM kernel (8 window rows x 128-column chunks per CTA) on
    shapes whose window rows / columns end inside a band or a chunk, and
    saturated planes (window sums at their maximum, 49 * 255^2): every plane
    bit-identical to the oracle (metrics.cpp:144-182)."""
    rng = np.random.default_rng(23 + C)
    for M, N in [(7, 7), (8, 134), (14, 135), (15, 262), (22, 263), (7, 390), (40, 9), (13, 1000)]:
        F = 3
        a = rng.integers(0, 256, (F, M, N, C), dtype=np.uint8)
        b = np.clip(a.astype(int) + rng.integers(-60, 60, a.shape), 0, 255).astype(np.uint8)
        a[1] = 255
        b[2] = 255
        s = ctx.metrics(a, b, "ssim")
        for f in range(F):
            for c in range(C):
                assert s[f * C + c] == oracle.ssim(np.ascontiguousarray(a[f, :, :, c]),
                                                   np.ascontiguousarray(b[f, :, :, c])), (M, N, f, c)


def _config_cases():
    import json
    return json.load(open(os.path.join(G, "config_digests.json")))["cases"]


@pytest.mark.parametrize("name", sorted(_config_cases()))
def test_config_digests_rgb(ctx, name):
    """Every BASELINE config (4K adaptive b32 n8, the 12 sweep runs, CelebA,
    PETS) and the paper's other grid sides at 1080p, 3 planes each, against
    sha256 digests of the reference's own outputs (make_golden.py)."""
    c = _config_cases()[name]
    M, N, b, n = c["M"], c["N"], c["b"], c["n"]
    frames = oracle.synth_frames(5, 1, M, N, 3)
    masks = oracle.synth_masks(5, 1, M, N)
    assert hashlib.sha256(frames[0].tobytes()).hexdigest() == c["input_sha"]
    seeds = dp.plane_seeds(42, 1, 3, frame0=5)
    if c["adaptive"]:
        pls, img = ctx.pixelize_adaptive(frames, masks, dp.make_privacy_params(c["eps"], c["m"], b, n),
                                         dp.NOISE_KEYED, seeds)
        stats = [np.frombuffer(p, np.uint8) for p in pls]
    else:
        means, img = ctx.pixelize_uniform(frames, dp.make_privacy_params(c["eps"], c["m"], b),
                                          dp.NOISE_KEYED, seeds)
        stats = list(means)
    for ch, pl in enumerate(c["planes"]):
        assert stats[ch].size == pl["stats_len"], (name, ch)
        assert hashlib.sha256(stats[ch].tobytes()).hexdigest() == pl["stats_sha"], (name, ch)
        plane = np.ascontiguousarray(img[0, :, :, ch])
        assert hashlib.sha256(plane.tobytes()).hexdigest() == pl["image_sha"], (name, ch)


def test_one_read_sweep_matches_reference_digests(ctx):
    """K1s (dppx_pixelize_uniform_sweep_dev): ONE read of the 1917 x 1083 RGB
    frame for all 12 (b, eps) runs of config 3; every run's means and image
    equal the reference's own (config_digests.json sweep_b*_eps*)."""
    import torch
    cases = _config_cases()
    M, N, C = 1083, 1917, 3
    bl, el = [4, 8, 16, 32], [0.1, 0.5, 1.0]
    dev = torch.device("cuda:0")
    pitch = (N * C + 15) // 16 * 16
    d = dp._desc(M, N, C, 1, pitch=pitch, opitch=pitch)
    frames = oracle.synth_frames(5, 1, M, N, C)
    img = torch.zeros((1, M, pitch), dtype=torch.uint8, device=dev)
    img[:, :, :N * C] = torch.from_numpy(frames.reshape(1, M, N * C)).to(dev)
    nz, keep = dp.Context._noise(dp.NOISE_KEYED, dp.plane_seeds(42, 1, 3, frame0=5))
    means, outs = [], []
    for b in bl:
        G = dp.grid_dims(M, N, b).grid_count()
        for _ in el:
            means.append(torch.zeros((C, G), dtype=torch.uint8, device=dev))
            outs.append(torch.zeros((1, M, pitch), dtype=torch.uint8, device=dev))
    ctx.reset_stats()
    ctx.pixelize_uniform_sweep_dev(d, img, bl, el, 16, nz, means, outs)
    ctx.synchronize()
    assert ctx.stats()["launches"]["sweep"] == 1 and ctx.stats()["launches"]["stats_tma"] == 0
    k = 0
    for b in bl:
        for e in el:
            c = cases[f"sweep_b{b}_eps{e}"]
            mh = means[k].cpu().numpy()
            im = outs[k].cpu().numpy()[0, :, :N * C].reshape(M, N, C)
            for ch, pl in enumerate(c["planes"]):
                assert hashlib.sha256(mh[ch].tobytes()).hexdigest() == pl["stats_sha"], (b, e, ch)
                plane = np.ascontiguousarray(im[:, :, ch])
                assert hashlib.sha256(plane.tobytes()).hexdigest() == pl["image_sha"], (b, e, ch)
            k += 1
