"""The C++ drop-in (include/mgrx_b200.hpp) against the unmodified reference:
runs oracle/_ref/test_dropin (built by `make -C oracle dropin` where the
reference sources exist) on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "test_dropin")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="drop-in test binary not built (needs /root/reference)")
def test_cpp_dropin_matches_reference():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL OK" in r.stdout
