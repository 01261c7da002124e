"""The doctest shim (tests/cpp/doctest_shim/doctest.h) runs the reference's
unit suites unmodified against the reference CPU library itself: all 87 test
cases pass, so a failure of the same suites against the GPU drop-in
(tests/test_gpu_dropin.py) is the drop-in's, not the harness's."""
import os
import subprocess

import pytest

EXE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_ref_gate", "dppix_unit_ref")


@pytest.mark.skipif(not os.path.exists(EXE), reason="built only where /root/reference exists")
def test_shim_runs_reference_suites_on_reference():
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "test cases: 87 | 87 passed | 0 failed" in r.stdout, r.stdout
