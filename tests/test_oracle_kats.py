"""The oracle (oracle/dppx_oracle.c) against the known-answer tests of the
reference's own unit suites (proj/tests/test_*.cpp, restated here)."""
import math

import numpy as np
import pytest

import oracle


def test_grid_dims_kats():  # test_image.cpp:48-74
    g = oracle.grid_dims(768, 576, 16)
    assert (g.grid_rows, g.grid_cols, g.pad_rows, g.pad_cols) == (48, 36, 0, 0)
    g = oracle.grid_dims(10, 10, 3)
    assert (g.grid_rows, g.grid_cols, g.pad_rows, g.pad_cols) == (4, 4, 2, 2)
    g = oracle.grid_dims(1920, 1080, 30)
    assert (g.grid_rows, g.grid_cols, g.pad_rows, g.pad_cols) == (64, 36, 0, 0)
    for bad in [(4, 4, 0), (0, 4, 2), (4, 0, 2), (4, 6, 7)]:
        with pytest.raises(oracle.OracleError):
            oracle.grid_dims(*bad)
    oracle.grid_dims(4, 6, 6)
    # SURVEY §8a a2 shapes
    assert [tuple(getattr(oracle.grid_dims(1083, 1917, b), k) for k in
                  ("grid_rows", "grid_cols", "pad_rows", "pad_cols")) for b in (4, 8, 16, 32)] == [
        (271, 480, 1, 3), (136, 240, 5, 3), (68, 120, 5, 3), (34, 60, 5, 3)]


def test_mirror_padding_through_the_path():  # test_image.cpp:76-93
    img = np.array([[1, 2, 3], [4, 5, 6]], np.uint8)
    means, _ = oracle.pixelize_uniform(img, 2, 1.0)
    assert list(means[0]) == [3, 5]  # padded col 3 == col 2: {3,3,6,6} -> 4.5 -> 5
    img = np.arange(1, 10, dtype=np.uint8).reshape(3, 3)
    means, _ = oracle.pixelize_uniform(img, 2, 1.0)
    assert list(means[0]) == [3, 5, 8, 9]  # rows then columns reflected
    with pytest.raises(oracle.OracleError):  # test_image.cpp:102-106
        oracle.pixelize_uniform(np.full((3, 10), 5, np.uint8), 8, 1.0)


def test_grid_mean_and_quantize_kats():  # test_image.cpp:122-167, test_pixelize.cpp:53-90
    means, img = oracle.pixelize_uniform(np.array([[0, 0], [255, 255]], np.uint8), 2, 1.0)
    assert (img == 128).all()
    ramp = np.arange(16, dtype=np.uint8).reshape(4, 4)
    means, img = oracle.pixelize_uniform(ramp, 2, 1.0)
    assert list(means[0]) == [3, 5, 11, 13]
    assert img.tolist() == [[3, 3, 5, 5], [3, 3, 5, 5], [11, 11, 13, 13], [11, 11, 13, 13]]
    for b in (2, 3, 5):  # constant image is a fixed point
        c = np.full((11, 13), 77, np.uint8)
        assert (oracle.pixelize_uniform(c, b, 1.0)[1] == 77).all()
        assert (oracle.pixelize_reference(c, b, 1.0) == 77).all()


def test_privacy_params_kats():  # test_noise.cpp:29-88
    p = oracle.make_privacy_params(0.5, 16, 16, 4)
    assert (p.subgrid_side, p.delta, p.sigma, p.sigma_sub) == (4, 15.9375, 31.875, 31.875 * 16)
    assert oracle.make_privacy_params(1.0, 32, 32, 8).delta_sub == 510.0
    assert oracle.make_privacy_params(0.1, 1, 1).sigma == 2550.0
    for n in (1, 2, 3, 4, 6, 8):
        q = oracle.make_privacy_params(0.7, 5, 24, n)
        assert q.sigma_sub == q.sigma * (n * n)
    for bad in [(0.0, 1, 4, 1), (1.0, 0, 4, 1), (1.0, 1, 0, 1), (1.0, 1, 4, 3), (1.0, 1, 4, 0)]:
        with pytest.raises(oracle.OracleError):
            oracle.make_privacy_params(*bad)


def test_noise_kats():  # test_noise.cpp:90-128
    first = oracle.laplace_at(42, 0, 0, 0, 0, 1.0)
    assert first == oracle.laplace_at(42, 0, 0, 0, 0, 1.0)
    for k in [(1, 0, 0, 0), (0, 1, 0, 0), (0, 0, 1, 0), (0, 0, 0, 1)]:
        assert oracle.laplace_at(42, *k, 1.0) != first
    assert oracle.laplace_at(43, 0, 0, 0, 0, 1.0) != first
    lo, hi = oracle.uniform_from_bits(0), oracle.uniform_from_bits(2**64 - 1)
    assert -0.5 < lo and hi < 0.5
    assert math.isfinite(oracle.laplace_from_uniform(lo, 1.0))
    assert oracle.laplace_from_uniform(0.0, 123.0) == 0.0
    for k in range(32):
        key = (k, 3 * k, k % 5, k % 3)
        unit = oracle.laplace_at(7, *key, 1.0)
        assert oracle.laplace_at(7, *key, 2.0) == 2.0 * unit
        assert oracle.laplace_at(7, *key, 1024.0) == 1024.0 * unit


def test_noise_distribution_ks():  # test_noise.cpp:130-155, acceptance criterion 4
    n = 200_000
    xs = np.array([oracle.laplace_at(42, r, c, 0, 0, 1.0) for r in range(400) for c in range(500)])
    xs.sort()
    cdf = np.where(xs < 0, 0.5 * np.exp(xs), 1 - 0.5 * np.exp(-xs))
    i = np.arange(n)
    d = max(np.max(np.abs(cdf - i / n)), np.max(np.abs(cdf - (i + 1) / n)))
    assert d < 1.62762 / math.sqrt(n)
    assert abs(np.mean(np.abs(xs)) - 1.0) < 0.01
    assert abs(np.mean(xs)) < 5 / math.sqrt(n)


def test_adaptive_kats():  # test_adaptive.cpp:44-144
    half = np.array([[1, 1], [0, 0]], np.uint8)
    pl, _ = oracle.pixelize_adaptive(np.zeros((2, 2), np.uint8), half, 2, 1, 1.0, 1.0)
    mm, S, simple, cplx = oracle.parse_adaptive_payload(pl[0], 1, 1)
    assert mm[0] == np.float32(0.5) and S == 0  # tie -> complex
    ramp = np.arange(16, dtype=np.uint8).reshape(4, 4)
    pl, img = oracle.pixelize_adaptive(ramp, np.zeros((4, 4), np.uint8), 4, 2, 1.0, 4.0)
    mm, S, simple, cplx = oracle.parse_adaptive_payload(pl[0], 1, 2)
    assert S == 0 and list(cplx) == [3, 5, 11, 13]
    p = oracle.make_privacy_params(2.0, 3, 4, 2)
    pl, _ = oracle.pixelize_adaptive(np.full((4, 4), 100, np.uint8), np.zeros((4, 4), np.uint8),
                                     4, 2, p.sigma, p.sigma_sub, "keyed", [77])
    cplx = oracle.parse_adaptive_payload(pl[0], 1, 2)[3]
    for sr in range(2):
        for sc in range(2):
            v = min(max(100.0 + oracle.laplace_at(77, 0, 0, sr, sc, p.sigma_sub), 0.0), 255.0)
            assert cplx[sr * 2 + sc] == math.floor(v) + (1 if v - math.floor(v) >= 0.5 else 0)


def test_reassemble_kats():  # test_adaptive.cpp:185-234
    payload = (np.array([1.0, 0.0], "<f4").tobytes() + (1).to_bytes(4, "little")
               + bytes([9, 1, 2, 3, 4]))
    assert oracle.reassemble(payload, 2, 4, 2, 2).tolist() == [[9, 9, 1, 2], [9, 9, 3, 4]]
    with pytest.raises(oracle.OracleError):
        oracle.reassemble(payload[:-1], 2, 4, 2, 2)


def test_synthetic_generator_is_deterministic():
    a = oracle.synth_frames(5, 2, 40, 60, 3)
    b = oracle.synth_frames(5, 2, 40, 60, 3)
    assert np.array_equal(a, b) and a.std() > 20
    m = oracle.synth_masks(0, 1, 1080, 1920)[0]
    assert 0.2 < 1 - m.mean() < 0.3  # ~25 % foreground


def test_variance_classification_restatement():
    """EXTENSION check: the CPU restatement's variance test on hand-made cells."""
    img = np.zeros((8, 8), np.uint8)
    img[:4, 4:] = np.array([[0, 255] * 2] * 4)     # cell (0,1): var = 255^2/4
    mm = oracle.classify_variance(img, 4, 100.0)
    assert list(mm) == [1.0, 0.0, 1.0, 1.0]
    assert list(oracle.classify_variance(img, 4, 255.0 ** 2 / 4)) == [1.0, 0.0, 1.0, 1.0]
    assert list(oracle.classify_variance(img, 4, 255.0 ** 2 / 4 + 1e-9)) == [1.0] * 4
    assert list(oracle.classify_variance(img, 4, 0.0)) == [0.0] * 4  # var >= 0 always


def test_log1p_restatement_is_the_host_libm():
    """The restated glibc log1p (twin of the device's) equals the host libm bit for
    bit on the noise domain -2|u| and on random bit patterns (FMA hosts: glibc's
    ifunc picks the FMA variant the restatement follows)."""
    flags = open("/proc/cpuinfo").read().split()
    if not ("fma" in flags and "avx2" in flags):
        pytest.skip("host libm uses the non-FMA log1p variant")
    rng = np.random.default_rng(11)
    bits = rng.integers(0, 2**63, 2_000_000, dtype=np.uint64)
    u = (bits >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 - 0.5
    assert oracle.log1p_glibc_mismatches(-2.0 * np.abs(u))[0] == 0
    assert oracle.log1p_glibc_mismatches(rng.integers(0, 2**64, 10**6, dtype=np.uint64)
                                         .view(np.float64))[0] == 0
    edge = np.array([0.0, -0.0, -1.0, -1 + 2**-52, -2**-54, -2**-29, -0.2929, -0.29289,
                     0.41422, -0.5, 1e300, np.inf, -np.inf, np.nan])
    assert oracle.log1p_glibc_mismatches(edge)[0] == 0
