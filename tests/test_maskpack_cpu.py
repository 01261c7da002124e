"""Host mask bit packing of the pinned pipeline (no GPU): tests/cpp/test_maskpack.cpp."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def test_maskpack_program():
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp"), "test_maskpack"], check=True)
    r = subprocess.run([os.path.join(HERE, "cpp", "test_maskpack")], capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0, r.stderr
    assert "all checks passed" in r.stdout
