"""Seeded input generators: C and Python twins agree; recipes hold (-m "not gpu")."""
import numpy as np
import pytest

import workloads


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5, 6, 7, 8])
def test_c_matches_python(cfg):
    a = workloads.generate(cfg, 1500, impl="py")
    b = workloads.generate(cfg, 1500, impl="c", threads=3)
    assert np.array_equal(a.data, b.data)
    assert np.array_equal(a.offsets, b.offsets)
    assert np.array_equal(a.exp_bits, b.exp_bits)
    assert np.array_equal(a.exp_status, b.exp_status)
    assert np.array_equal(a.known, b.known)


def test_thread_partition_invariant():
    a = workloads.generate(4, 50_000, impl="c", threads=1)
    b = workloads.generate(4, 50_000, impl="c", threads=7)
    assert np.array_equal(a.data, b.data) and np.array_equal(a.offsets, b.offsets)


def test_recipe_shapes():
    w = workloads.generate(2, 20_000, impl="c")
    lines = bytes(w.data).split(b"\n")
    assert lines[-1] == b"" and len(lines) == 20_001
    mean = w.data.size / w.n
    assert 18.5 < mean < 20.5                       # ~19 chars + '\n'
    w3 = workloads.generate(3, 20_000, impl="c")
    assert w3.data.size / w3.n < 16                 # short coordinate strings
    assert bytes(w3.data).count(b",") == 10_000
    w5 = workloads.generate(5, 4_000, impl="c")
    assert w5.data.size / w5.n > 150                # long adversarial strings
    assert w5.known.mean() > 0.6
