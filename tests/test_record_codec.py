"""The .dppx record codec (dppx_encode_record / dppx_decode_record, host code)
against the reference's record tests (proj/tests/test_record.cpp:83-263) and
the records the reference itself encoded (tests/golden/records.npz)."""
import os
import struct
import zlib

import numpy as np
import pytest

import oracle
import paper_2511_04261_b200 as dp

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def refresh_crc(b: bytearray):  # test_record.cpp:49-58
    b[-4:] = struct.pack("<I", zlib.crc32(bytes(b[:-4])))


def uniform_record(rng, M, N, b):
    img = rng.integers(0, 256, (M, N), dtype=np.uint8)
    p = oracle.make_privacy_params(0.5, 16, b)
    means, _ = oracle.pixelize_uniform(img, b, p.sigma, "keyed", [int(rng.integers(0, 2**62))],
                                       want_image=False)
    return dp.encode_record(M, N, b, 1, means[0].tobytes(), False)


def adaptive_record(rng, M, N, b, n):
    img = rng.integers(0, 256, (M, N), dtype=np.uint8)
    mask = rng.integers(0, 2, (M, N), dtype=np.uint8)
    p = oracle.make_privacy_params(0.5, 16, b, n)
    pl, _ = oracle.pixelize_adaptive(img, mask, b, n, p.sigma, p.sigma_sub, "keyed",
                                     [int(rng.integers(0, 2**62))], want_image=False)
    return dp.encode_record(M, N, b, n, pl[0], True)


def test_crc32_is_zlib():
    rng = np.random.default_rng(0)
    for n in (0, 1, 7, 8, 9, 1000, 4097):
        d = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert dp.crc32(d) == zlib.crc32(d)


def test_golden_records_byte_identical():
    z = np.load(os.path.join(G, "records.npz"))
    img = np.ascontiguousarray(oracle.synth_frames(0, 1, 576, 768, 1)[0, :, :, 0])
    p = oracle.make_privacy_params(0.5, 16, 16)
    means, _ = oracle.pixelize_uniform(img, 16, p.sigma, "keyed", [11])
    assert dp.encode_record(576, 768, 16, 1, means[0].tobytes(), False) == z["pets_uniform_b16"].tobytes()
    mask = oracle.synth_masks(0, 1, 576, 768)[0]
    p = oracle.make_privacy_params(0.5, 16, 16, 4)
    pl, _ = oracle.pixelize_adaptive(img, mask, 16, 4, p.sigma, p.sigma_sub, "keyed", [11])
    assert dp.encode_record(576, 768, 16, 4, pl[0], True) == z["pets_adaptive_b16n4"].tobytes()
    for k in ("pets_uniform_b16", "pets_adaptive_b16n4"):
        rec = dp.decode(z[k].tobytes())
        assert dp.encode(rec) == z[k].tobytes()


def test_size_laws():  # test_record.cpp:83-143
    assert len(dp.encode_record(16, 16, 16, 1, bytes([200]), False)) == 25
    rng = np.random.default_rng(41)
    assert len(uniform_record(rng, 768, 576, 16)) == 1752
    assert len(adaptive_record(rng, 4, 4, 4, 2)) <= 36
    prev = None
    for b in (1, 2, 4, 8, 16, 32, 64, 128):
        size = len(uniform_record(rng, 768, 576, b))
        if prev:
            assert size < prev
        prev = size


def test_decode_inverts_encode():  # test_record.cpp:145-160
    rng = np.random.default_rng(44)
    for rnd in range(20):
        M, N = int(rng.integers(2, 62)), int(rng.integers(2, 62))
        b = int(rng.integers(1, min(M, N, 12) + 1))
        if rnd % 2 == 0:
            rec = uniform_record(rng, M, N, b)
        else:
            rec = adaptive_record(rng, M, N, b, 2 if b % 2 == 0 else 1)
        assert dp.encode(dp.decode(rec)) == rec


def kind(bad):
    with pytest.raises(dp.RecordError) as e:
        dp.decode(bytes(bad))
    return e.value.kind


def test_failure_taxonomy():  # test_record.cpp:162-263
    rng = np.random.default_rng(45)
    rec = bytearray(uniform_record(rng, 32, 32, 8))
    bad = bytearray(rec); bad[0] = ord("X")
    assert kind(bad) == "not_a_record" and kind(b"") == "not_a_record"
    bad = bytearray(rec); bad[22] ^= 0x40
    assert kind(bad) == "corruption"
    bad = bytearray(rec); bad[-1] ^= 0x01
    assert kind(bad) == "corruption"
    assert kind(rec[:10]) == "corrupt_record"
    assert kind(rec[:-8]) == "corruption"
    rec = bytearray(uniform_record(rng, 16, 16, 4))
    for off, val, want in [(4, 2, "unsupported_version"), (6, 3, "corrupt_record"),
                           (7, 1, "corrupt_record"), (18, 2, "corrupt_record"),
                           (8, 32, "corrupt_record")]:
        bad = bytearray(rec); bad[off] = val; refresh_crc(bad)
        assert kind(bad) == want, off
    bad = bytearray(rec); bad[16] = 0; bad[17] = 0; refresh_crc(bad)
    assert kind(bad) == "corrupt_record"


def test_adaptive_count_must_match_mask_means():  # test_record.cpp:265-293
    rng = np.random.default_rng(49)
    img = rng.integers(0, 256, (16, 16), dtype=np.uint8)
    mask = np.ones((16, 16), np.uint8); mask[:, 8:] = 0
    p = oracle.make_privacy_params(0.5, 16, 4, 2)
    pl, _ = oracle.pixelize_adaptive(img, mask, 4, 2, p.sigma, p.sigma_sub, "keyed", [3])
    rec = bytearray(dp.encode_record(16, 16, 4, 2, pl[0], True))
    at = 20 + 4 * 16
    assert rec[at] == 8
    rec[at] = 7
    refresh_crc(rec)
    assert kind(rec) == "corrupt_record"
    with pytest.raises(ValueError):  # encode refuses the same inconsistency
        bad = bytearray(pl[0]); bad[4 * 16] = 7
        dp.encode_record(16, 16, 4, 2, bytes(bad), True)


def test_reference_decodes_our_records():
    if oracle.ref is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(5)
    for _ in range(10):
        M, N = int(rng.integers(8, 70)), int(rng.integers(8, 70))
        b = int(rng.choice([2, 4, 8]))
        img = rng.integers(0, 256, (M, N), dtype=np.uint8)
        mask = rng.integers(0, 2, (M, N), dtype=np.uint8)
        p = oracle.make_privacy_params(0.5, 16, b, 2)
        pl, im = oracle.pixelize_adaptive(img, mask, b, 2, p.sigma, p.sigma_sub, "keyed", [9])
        ours = dp.encode_record(M, N, b, 2, pl[0], True)
        assert ours == oracle.ref.encode_adaptive(img, mask, 0.5, 16, b, 2, 9)
