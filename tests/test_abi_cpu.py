"""CPU-side checks of the C ABI library: it loads without a GPU, exports every
symbol include/dppx_gpu.h declares, and its host helpers agree with the oracle.
No compute entry point is called here."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_2511_04261_b200 as dp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "dppx_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dppx_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(dp.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(dp.ABI), set(syms) ^ set(dp.ABI)


def test_dropin_library_exports_reference_api():
    import subprocess
    out = subprocess.run(["nm", "-D", "-C", "--defined-only", dp.DROPIN_PATH],
                         capture_output=True, text=True, check=True).stdout
    for fn in ["dppix::pixelize_parallel(", "dppix::pixelize_adaptive(", "dppix::broadcast_means(",
               "dppix::reassemble(", "dppix::classify_regions(", "dppix::make_privacy_params(",
               "dppix::grid_dims(", "dppix::laplace_at(", "dppix::keyed_bits(",
               "dppix::mirror_pad(", "dppix::grid_mean(", "dppix::mask_grid_mean(",
               "dppix::encode(", "dppix::decode(", "dppix::reconstruct(", "dppix::read_record(",
               "dppix::write_record("]:
        assert fn in out, fn


def test_kernels_are_sm100a_with_tma():
    import subprocess
    sass = subprocess.run(["cuobjdump", "-sass", dp.LIB_PATH], capture_output=True, text=True,
                          check=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", dp.LIB_PATH], capture_output=True,
                                       text=True).stdout
    assert "UBLKCP" in sass  # cp.async.bulk (TMA bulk copies)
    assert "SYNCS" in sass   # mbarrier ops
    assert "IDP.4A" in sass  # dp4a byte sums


def test_host_helpers_match_oracle():
    rng = np.random.default_rng(0)
    for _ in range(200):
        seed = int(rng.integers(0, 2**63))
        k = [int(x) for x in rng.integers(0, 2**32, 4)]
        assert dp.keyed_bits(seed, *k) == oracle.keyed_bits(seed, *k)
        assert dp.laplace_at(seed, *k, 3.5) == oracle.laplace_at(seed, *k, 3.5)
        assert dp.derive_plane_seed(seed, k[0], 2) == oracle.derive_plane_seed(seed, k[0], 2)
    for M, N, b in [(1080, 1920, 16), (1083, 1917, 4), (218, 178, 16), (1, 1, 1), (5, 3, 5)]:
        g, o = dp.grid_dims(M, N, b), oracle.grid_dims(M, N, b)
        assert (g.grid_rows, g.grid_cols, g.pad_rows, g.pad_cols) == (
            o.grid_rows, o.grid_cols, o.pad_rows, o.pad_cols)
    with pytest.raises(ValueError):
        dp.grid_dims(4, 4, 5)
    p = dp.make_privacy_params(0.5, 16, 16, 4)
    assert (p.sigma, p.sigma_sub, p.delta) == (31.875, 510.0, 15.9375)
    with pytest.raises(ValueError):
        dp.make_privacy_params(1.0, 1, 4, 3)
    assert dp.adaptive_payload_capacity(1080, 1920, 16, 4) == 4 * 8160 + 4 + 8160 * 16


def test_kernel_family_table_matches_header():
    """The ctypes dppx_kernel_stats mirror has as many families as the header."""
    import re
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "include", "dppx_gpu.h")).read()
    count = int(re.search(r"DPPX_K_COUNT\s*=\s*(\d+)", hdr).group(1))
    assert dp.K_COUNT == count == len(dp.KERNEL_FAMILIES)
