"""The C++ drop-in (include/dppix + libdppix_gpu.so) passes the reference's own
unit-test cases restated in tests/cpp/test_dropin.cpp."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_cpp_dropin_program(ctx):
    exe = os.path.join(HERE, "cpp", "test_dropin")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr


GATE = os.path.join(HERE, "cpp", "_ref_gate")


def _gate_exe(name):
    exe = os.path.join(GATE, name)
    if not os.path.exists(exe):
        pytest.skip(f"{name} not built (needs /root/reference at build time)")
    return exe


def test_reference_release_gate_on_dropin(ctx):
    """The reference's own release gate, acceptance_main.cpp compiled UNMODIFIED
    against include/dppix + libdppix_gpu.so (every L1/L0 call runs on the
    GPU): criteria 1-7, 9 and 10 must PASS. Criterion 8 times the drop-in's
    pixelize_parallel against its pixelize_reference (a CPU thread-scaling
    floor in the reference); it is reported, not required."""
    r = subprocess.run([_gate_exe("dppix_acceptance_gpu")], capture_output=True, text=True,
                       timeout=900)
    print(r.stdout, r.stderr)
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    passes = [ln for ln in lines if "PASS" in ln]
    fails = [ln for ln in lines if "FAIL" in ln and "[ 8]" not in ln]
    assert not fails, r.stdout
    assert len(passes) >= 9, r.stdout


def test_reference_unit_suites_on_dropin(ctx):
    """The reference's doctest unit suites (image, noise, pixelize, adaptive,
    record, metrics), unmodified, through the doctest shim, against the GPU
    drop-in: every test case passes."""
    r = subprocess.run([_gate_exe("dppix_unit_gpu")], capture_output=True, text=True, timeout=900)
    print(r.stdout, r.stderr[-5000:])
    assert r.returncode == 0, r.stderr[-5000:]
    assert "test cases: 84 | 84 passed | 0 failed" in r.stdout, r.stdout
