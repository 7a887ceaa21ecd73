"""CPU-side checks of the C-ABI boundary: the library loads without a GPU and exports every
entry point include/gabp_b200.h declares; error paths that need no device behave."""
import ctypes
import os
import re

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "gabp_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"\b(bg(?:abp|mg)_[a-z0-9_]+)\s*\(", text)
    return sorted(set(names))


def test_header_declares_the_reference_surface():
    names = declared_functions()
    for must in ["bgabp_create", "bgabp_sweep", "bgabp_solve", "bgabp_precompute_lambda", "bgabp_correction_sweeps",
                 "bgabp_error_correction_apply", "bgabp_solve_error_correction", "bgabp_node_precisions",
                 "bgabp_residual_inf_norm", "bgmg_create", "bgmg_vcycle", "bgmg_solve", "bgmg_restrict",
                 "bgmg_prolong"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1904_04093_b200 import gabp
    L = ctypes.CDLL(gabp.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(L, n)]
    assert not missing, missing


def test_library_is_built_for_sm100a():
    from paper_1904_04093_b200 import gabp
    assert gabp.lib().bgabp_version() == b"gabp_b200 sm_100a"
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", gabp.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_invalid_inputs_rejected_before_any_device_work():
    """Structural checks run on the host first (gabp.cpp:29-33): no GPU needed to reject."""
    import numpy as np

    from paper_1904_04093_b200 import GabpEngine, SparseMatrix
    A = SparseMatrix(2, np.array([0, 2, 3], np.int32), np.array([0, 1, 0], np.int32), np.array([1.0, 1.0, 1.0]))
    with pytest.raises(ValueError, match="structurally zero diagonal"):
        GabpEngine(A)
    B = SparseMatrix(2, np.array([0, 2, 4], np.int32), np.array([1, 0, 0, 1], np.int32), np.ones(4))
    with pytest.raises(ValueError, match="canonical"):
        GabpEngine(B)


def test_bench_reference_arm_loads_only_the_oracle():
    """The reference arm's input comes from the oracle's own generators: the product library
    must not be mapped into that process (the driver records the .so files each arm loads)."""
    import subprocess
    import sys
    code = ("import sys; sys.argv=['bench.py']; import bench; o, kind, A, b = bench.oracle_config2(); "
            "print(A.n, b.shape[0]); print(open('/proc/self/maps').read())")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    assert out.stdout.startswith("4194304 4194304")
    assert "libgabp_b200" not in out.stdout
