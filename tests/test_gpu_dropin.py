"""The C++ drop-in (include/belief_b200.hpp) against the reference's own engine, both compiled
into one test binary (tests/cpp/, built by __graft_entry__.build() where /root/reference exists)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(__file__), "cpp", "_build", "dropin_test")


def test_cpp_dropin_matches_reference_engine():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_build/dropin_test not built (needs /root/reference at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "FAIL" not in out.stdout
