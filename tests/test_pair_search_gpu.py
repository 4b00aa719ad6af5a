"""nbx_grid_search_pair (the DD search step's two grids and two lists on two streams) builds
exactly the lists of the sequential nbx_grid_build(0/1) + nbx_search(LOCAL/NONLOCAL) calls,
outer and inner, bit for bit -- including when the coordinates are produced on the main
stream just before the call (the side stream must not start before them)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lists(eng):
    from paper_2405_01420_b200 import nbx
    out = {}
    for lst in (0, 1):
        s = nbx.ListSizes()
        nbx.check(nbx.lib().nbx_list_sizes_get(eng.ctx.h, lst, C.byref(s)))
        for which in (0, 1):
            sci = np.empty(s.n_sci, nbx.SCI_DTYPE)
            cj = np.empty(s.n_cj_outer if which == 0 else s.n_cj_inner, nbx.CJ_DTYPE)
            pool = np.empty(s.n_pool, nbx.POOL_DTYPE)
            nbx.check(nbx.lib().nbx_list_export(eng.ctx.h, lst, which, nbx._ptr(sci), nbx._ptr(cj), nbx._ptr(pool)))
            out[(lst, which)] = (sci, cj, pool)
    return out


@pytest.mark.parametrize("config", ["rnase24k", "stmv"])
def test_pair_search_matches_sequential(gpu, config):
    import torch

    from paper_2405_01420_b200 import dd, systems
    s = systems.make(config, 120000 if config == "stmv" else None)
    L = np.asarray(s.box, np.float64)
    rl = s.rlist_outer
    xw = np.mod(s.x.astype(np.float64), L)
    # a 2x1x1 decomposition seen from rank 0: home = lower half in x, halo = the slab of width
    # rlist_outer above it (the +x neighbour's atoms, the half-shell import)
    home = np.nonzero(xw[:, 0] < 0.5 * L[0])[0].astype(np.int32)
    halo = np.nonzero((xw[:, 0] >= 0.5 * L[0]) & (xw[:, 0] < 0.5 * L[0] + rl))[0].astype(np.int32)
    D = 0.5 * L[0]
    lo_l, size_l = np.array([0, 0, 0], np.float32), np.array([D, L[1], L[2]], np.float32)
    lo_n, size_n = np.array([-rl, 0, 0], np.float32), np.array([D + 2 * rl, L[1], L[2]], np.float32)
    xh = torch.from_numpy(xw[home].astype(np.float32)).cuda()
    xn = torch.from_numpy(xw[halo].astype(np.float32)).cuda()
    gh, gn = torch.from_numpy(home).cuda(), torch.from_numpy(halo).cuda()

    ref = dd.NbxEngine(s, 0, [0, 1, 1])
    ref.grid_build(0, xh, gh, lo_l, size_l)
    ref.grid_build(1, xn, gn, lo_n, size_n)
    ref.search(0)
    ref.search(1)
    want = _lists(ref)
    assert want[(1, 0)][1].shape[0] > 0  # the nonlocal list is not empty

    eng = dd.NbxEngine(s, 0, [0, 1, 1])
    side = torch.cuda.Stream()
    for rep in range(2):  # the second search takes the single-pass path
        torch.cuda.synchronize()
        torch.cuda._sleep(20_000_000)  # keep the main stream busy ...
        xh2, xn2 = xh * 1.0, xn * 1.0  # ... while it produces the inputs
        eng.grid_search_pair(xh2, gh, lo_l, size_l, xn2, gn, lo_n, size_n, side)
        torch.cuda.synchronize()
        got = _lists(eng)
        for key, (a, b, c) in want.items():
            ga, gb, gc = got[key]
            assert np.array_equal(a, ga) and np.array_equal(b, gb) and np.array_equal(c, gc), (rep, key)
