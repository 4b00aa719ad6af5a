"""Synthetic system generators."""
import numpy as np
import pytest

from paper_2405_01420_b200 import systems


@pytest.mark.parametrize("name,n", [("water3k", None), ("rnase24k", None), ("mem82k", None), ("stmv", 60000),
                                    ("water12m", 30000)])
def test_generator(name, n):
    s = systems.make(name, n)
    N = s.natoms
    if n is None:
        assert N == {"water3k": 3000, "rnase24k": 24024, "mem82k": 82000}[name]
    else:
        assert N == n
    assert s.x.dtype == np.float32 and s.x.shape == (N, 3)
    assert np.all(s.x >= 0) and np.all(s.x < s.box)
    assert abs(float(s.q.astype(np.float64).sum())) < 1e-3  # neutral
    assert np.isclose(N / np.prod(s.box.astype(np.float64)), 100.0, rtol=1e-3)  # presets.py:41
    # exclusions symmetric, no self, in range
    a = np.repeat(np.arange(N), np.diff(s.excl_offsets))
    b = s.excl_gids
    assert np.all(a != b) and np.all((b >= 0) & (b < N))
    pairs = set(zip(a.tolist(), b.tolist()))
    assert all((y, x) in pairs for x, y in pairs)
    assert s.c6c12.shape[0] == s.c6c12.shape[1] and np.all(s.type < s.c6c12.shape[0])
    assert s.rc <= s.rlist_inner <= s.rlist_outer
    assert np.all(s.box >= 2 * s.rlist_outer)


def test_deterministic():
    a = systems.make("rnase24k")
    b = systems.make("rnase24k")
    assert np.array_equal(a.x, b.x) and np.array_equal(a.q, b.q)


def test_full_size_counts():
    assert systems.make("stmv").natoms == 1066628
