"""PGM ingest of the C++ drop-in (host code, no GPU): tests/cpp/test_pgm.cpp."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def test_pgm_program():
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp"), "test_pgm"], check=True)
    r = subprocess.run([os.path.join(HERE, "cpp", "test_pgm")], capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
