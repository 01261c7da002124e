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
