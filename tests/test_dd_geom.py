"""CPU check of the device-side repartition's geometry (DomainDecomposition.dd_geom, the
nbx_dd_geom that csrc/peer.cu's k_rp_pull_home / k_rp_pull_halo consume).

The kernels' selection rules are replayed in numpy float32 (the same IEEE operations): every
atom gets exactly one new home, and every pair within rlist_outer (minimum image) is then
covered exactly once -- by the owner's local list, or by exactly one rank's half-shell import
of the partner's periodic image (reference halo shape: /root/reference/pkg/src/mdgpusim/
pipeline.py:273-278, 363-380).  world 2, 4, 8 -> (2,1,1), (2,2,1), (2,2,2)."""
import numpy as np
import pytest

from paper_2405_01420_b200 import dd as DD
from paper_2405_01420_b200 import systems


def _rank_view(s, rank, world):
    d = object.__new__(DD.DomainDecomposition)
    d.rank, d.world = rank, world
    d.dims = DD.balanced_dims(world)
    d.coord = DD.rank_coords(rank, d.dims)
    d.box = np.asarray(s.box, np.float64)
    d.D = d.box / np.array(d.dims)
    d.rl = float(s.rlist_outer)
    d._geom = None
    return d


def _wrap(x, L):
    # k_rp_pull_home's rp_wrap: x - floor(x / L) L in float32
    return (x - np.floor(x / L).astype(np.float32) * L).astype(np.float32)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_device_repartition_geometry_covers_pairs_once(world):
    s = systems.water_box(3000, seed=21, coulomb="ewald", rc=1.0, rlist_outer=1.1, rlist_inner=1.02)
    rng = np.random.default_rng(5)
    x = (s.x + rng.uniform(-0.3, 0.3, size=s.x.shape)).astype(np.float32)  # moved, some outside the box
    n = len(x)
    views = [_rank_view(s, r, world) for r in range(world)]
    geoms = [v.dd_geom() for v in views]
    g0 = geoms[0]
    box = np.array(g0.box[:], np.float32)
    dlen = np.array(g0.dlen[:], np.float32)
    dims = np.array(g0.dims[:])
    split = (dims > 1).astype(int)  # undivided dimensions stay periodic in the searches
    xw = np.stack([_wrap(x[:, d], box[d]) for d in range(3)], 1)
    c = np.stack([np.clip(np.floor(xw[:, d] / dlen[d]).astype(int), 0, dims[d] - 1) for d in range(3)], 1)
    owner = c[:, 0] + dims[0] * (c[:, 1] + dims[1] * c[:, 2])
    # home pull: rank r takes the atoms of its src ranks whose owner is r -> exactly one home each
    homes = [np.nonzero(owner == r)[0] for r in range(world)]
    assert np.array_equal(np.sort(np.concatenate(homes)), np.arange(n))
    for r, g in enumerate(geoms):
        # dims <= 2 per dimension: every rank is within +-1 of every other -> all are sources
        assert sorted(g.src_rank[:g.n_src]) == list(range(world))
        # half-shell offsets: 1 / 4 / 13 for 1 / 2 / 3 split dimensions
        assert g.n_off == {2: 1, 4: 4, 8: 13}[world]
    # halo pull: imported (atom, image shift) per rank, in the importer's frame
    imports = []
    for r, g in enumerate(geoms):
        lo, hi, rl = np.array(g.lo[:], np.float32), np.array(g.hi[:], np.float32), np.float32(g.rl)
        imp = {}
        for k in range(g.n_off):
            src = homes[g.off_rank[k]]
            sh = np.array(g.off_shift[k][:], np.float32)
            xs = (xw[src] + sh).astype(np.float32)
            ok = np.ones(len(src), bool)
            for d in range(3):
                o = g.off_dir[k][d]
                if o > 0:
                    ok &= xs[:, d] < np.float32(hi[d] + rl)
                if o < 0:
                    ok &= xs[:, d] >= np.float32(lo[d] - rl)
            for a, p in zip(src[ok], xs[ok]):
                key = (int(a), tuple(np.round((p - xw[a]) / box).astype(int) * split))
                assert key not in imp, "an atom image imported twice"
                imp[key] = p
        imports.append(imp)
    # every pair within rlist_outer (minimum image, box >= 2 rl) is covered exactly once
    rl2 = float(s.rlist_outer) ** 2
    boxd = box.astype(np.float64)
    xd = xw.astype(np.float64)
    for a in range(0, n, 97):  # a sample of i atoms against all j (keeps the test fast)
        dv = xd - xd[a]
        img = -np.round(dv / boxd)  # image of b nearest to a: b + img * box
        dv += img * boxd
        partners = np.nonzero(((dv * dv).sum(1) < rl2 * 0.98) & (np.arange(n) != a))[0]
        for b in partners:
            ra, rb = owner[a], owner[b]
            covered = 0
            if ra == rb:
                covered += 1  # local list (periodic in undivided dims)
            # (images in undivided dimensions come from the nonlocal search's periodic shifts)
            else:
                # a's rank imports b's image nearest to a, or b's rank imports a's image nearest to b
                if (int(b), tuple(img[b].astype(int) * split)) in imports[ra]:
                    covered += 1
                if (int(a), tuple((-img[b]).astype(int) * split)) in imports[rb]:
                    covered += 1
            assert covered == 1, (a, b, ra, rb, covered)
