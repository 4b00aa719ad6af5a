"""Property tests (hypothesis) of the oracle's list construction on random ragged inputs:
every pair within rc is present exactly once, exclusions only ever carry correction bits,
and the inner list is a subset of the outer list.  (The GPU lists are bit-identical to these,
tests/test_gpu_parity.py.)"""
import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import oracle as O
from paper_2405_01420_b200 import systems
from tests.helpers import flatten_pairs


def _system(n, L, seed, nexcl):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-0.5 * L, 1.5 * L, size=(n, 3)).astype(np.float32)  # some outside the box
    q = rng.uniform(-0.6, 0.6, n).astype(np.float32)
    t = rng.integers(0, 2, n).astype(np.int32)
    pairs = set()
    for _ in range(nexcl):
        a, b = rng.integers(0, n, 2)
        if a != b:
            pairs.add((int(min(a, b)), int(max(a, b))))
    lists = [[] for _ in range(n)]
    for a, b in pairs:
        lists[a].append(b)
        lists[b].append(a)
    eo = np.zeros(n + 1, np.int32)
    eo[1:] = np.cumsum([len(v) for v in lists])
    eg = np.array([g for v in lists for g in sorted(v)], np.int32)
    base = systems.make("water3k", 300)
    return systems.System("prop", x, q, t, base.c6c12, eo, eg, np.full(3, L, np.float32), "ewald", 0.9, 1.0,
                          0.92), pairs


@settings(max_examples=25, deadline=None)
@given(n=st.integers(1, 400), L=st.floats(2.05, 3.5), seed=st.integers(0, 10**6), nexcl=st.integers(0, 40))
def test_list_covers_each_pair_once(n, L, seed, nexcl):
    s, excl = _system(n, L, seed, nexcl)
    on = O.OracleNonbonded(s)
    on.search(s.x)
    g = on.grid.export()
    outer = flatten_pairs(on.list.export(0))
    inner = flatten_pairs(on.list.export(1))
    # A sparse tiny box can list several periodic images of one pair (or an atom and its own
    # image) because one cluster spans much of the box; with box >= 2 rlist at most one image is
    # inside rc, and only that one is ever computed.  Count images inside rc.
    seen = {}
    for ci, cj, sh, im, cm in outer:
        svec = np.array([(sh % 3 - 1), ((sh // 3) % 3 - 1), (sh // 9 - 1)], np.float64) * L
        for i in range(4):
            for j in range(8):
                bit = 1 << (i * 8 + j)
                if (im | cm) & bit:
                    ai, bj = 4 * ci + i, 8 * cj + j
                    a, b = int(g["gid"][ai]), int(g["gid"][bj])
                    key = (min(a, b), max(a, b))
                    if a != b:
                        assert bool(cm & bit) == (key in excl)
                    r = np.linalg.norm(g["xq"][ai, :3].astype(np.float64) + svec - g["xq"][bj, :3])
                    if r < 0.9:
                        assert a != b
                        seen[key] = seen.get(key, 0) + 1
    assert all(v == 1 for v in seen.values())
    # every pair inside rc (minimum image) is listed
    xw = np.mod(s.x.astype(np.float64), L)
    d = xw[:, None] - xw[None]
    d -= L * np.round(d / L)
    r2 = (d**2).sum(-1)
    ia, ib = np.nonzero(np.triu(r2 < (0.9 * (1 - 1e-6)) ** 2, 1))
    for a, b in zip(ia.tolist(), ib.tolist()):
        assert (a, b) in seen
    # inner (pruned) tiles are a subset of outer tiles
    outer_set = {(r[0], r[1], r[2]) for r in outer}
    assert all((r[0], r[1], r[2]) in outer_set for r in inner)
