"""Parity helpers shared by the GPU tests.

The bar (BASELINE.json north_star, SURVEY.md §7 hard part 1): per-iteration messages, beliefs and
x agree to relative 1e-10 in fp64 for the synchronous schedules,

    |g - c| <= 1e-10 * max(|c|, 1e-6 * ||c||_inf)          (elementwise)

and the number of entries that are not bit-identical is reported.  The kernels issue the
reference's operations in the reference's order with explicit rounding and no FMA contraction, so
the expected count of non-bitwise entries is zero; the tests assert that too where noted.
"""
import numpy as np

REL = 1e-10


def close(gpu, cpu, rel=REL):
    gpu = np.asarray(gpu, dtype=np.float64)
    cpu = np.asarray(cpu, dtype=np.float64)
    assert gpu.shape == cpu.shape
    both_nan = np.isnan(gpu) & np.isnan(cpu)
    scale = np.maximum(np.abs(cpu), 1e-6 * (np.nanmax(np.abs(cpu)) if cpu.size else 0.0))
    ok = both_nan | (np.abs(gpu - cpu) <= rel * scale) | (gpu == cpu)
    return bool(np.all(ok)), int(np.sum(gpu.view(np.uint64) != cpu.view(np.uint64)))


def assert_close(gpu, cpu, what="", rel=REL, bitwise=False):
    ok, nbits = close(gpu, cpu, rel)
    assert ok, f"{what}: exceeds rel {rel} (non-bitwise entries: {nbits})"
    if bitwise:
        assert nbits == 0, f"{what}: {nbits} entries not bit-identical"
    return nbits
