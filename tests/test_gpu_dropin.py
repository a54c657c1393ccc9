"""The reference's own C++ call sites against the picgpu:: drop-in (built by
oracle/Makefile from the unmodified reference headers + include/picgpu.hpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_parity")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/dropin_parity not built")
def test_cpp_dropin_parity():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "drop-in parity ok" in r.stdout
