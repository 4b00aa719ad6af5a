"""CPU tests of the oracle: pinned against float64 brute force, analytic identities and the
committed golden fixtures (tests/golden/, made by tools/make_golden.py)."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from oracle.brute import brute_force
from paper_2405_01420_b200 import systems
from tests.helpers import flatten_pairs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_derived_constants():
    # beta from erfc(beta rc) = 1e-5 (SURVEY.md section 7 quotes 3.4705 / 3.1234 / 2.6028)
    for rc, beta in ((0.9, 3.4705), (1.0, 3.1234), (1.2, 2.6028)):
        c = O.derive_consts(O.make_params("ewald", rc, rc + 0.1, rc + 0.02))
        assert abs(c["beta"] - beta) < 2e-4
    c = O.derive_consts(O.make_params("rf", 0.9, 1.0, 0.92, epsilon_rf=0.0))
    assert np.isclose(c["k_rf"], 1 / (2 * 0.9**3), rtol=1e-7)
    assert np.isclose(c["c_rf"], 1 / 0.9 + c["k_rf"] * 0.81, rtol=1e-7)
    assert np.isclose(c["epsfac"], 138.935458, rtol=1e-7)
    c2 = O.derive_consts(O.make_params("rf", 1.0, 1.1, 1.02, epsilon_r=1.0, epsilon_rf=78.0))
    assert np.isclose(c2["k_rf"], (78 - 1) / (2 * 78 + 1), rtol=1e-6)


def test_ewald_rational_accuracy():
    from tools.fit_ewald import G_exact, H_exact
    z = np.linspace(0, 12.5, 4001)
    g = np.array([O.ewald_G(v) for v in z])
    h = np.array([O.ewald_H(v) for v in z])
    assert np.max(np.abs(g - G_exact(z)) / G_exact(z)) < 6e-7
    assert np.max(np.abs(h - H_exact(z)) / H_exact(z)) < 3.5e-7  # (6,5) fit, fp32 evaluation


@pytest.mark.parametrize("name,n,coul_tol", [("water3k", None, 2e-6), ("rnase24k", 4000, 5e-5),
                                             ("mem82k", 5000, 5e-5)])
def test_oracle_vs_brute_force(name, n, coul_tol):
    s = systems.make(name, n)
    on = O.OracleNonbonded(s)
    on.search(s.x)
    f, e, vir, _ = on.forces()
    c = O.derive_consts(on.params)
    fb, eb, vb = brute_force(s.x, s.q, s.type, s.c6c12, s.excl_offsets, s.excl_gids, s.box, c,
                             s.coulomb, s.rc)
    rel = np.sqrt(((f - fb) ** 2).sum() / (fb**2).sum())
    assert rel < 5e-6
    assert abs(e[0] - eb[0]) / abs(eb[0]) < 1e-5
    # fp32 Ewald real space: erfc/r = 1/r - erf/r cancels near rc
    assert abs(e[1] - eb[1]) / abs(eb[1]) < coul_tol
    assert np.abs(vir - vb).max() / np.abs(vb).max() < 5e-6


def test_newton_third_law():
    s = systems.make("rnase24k", 4000)
    on = O.OracleNonbonded(s)
    on.search(s.x)
    f, _, _, _ = on.forces()
    assert np.abs(f.astype(np.float64).sum(0)).max() < 1e-5 * np.abs(f).sum()


def _grid_atom_pairs(on, lst):
    """Expand a list into the set of (gid_a, gid_b, shift) atom pairs it presents."""
    g = on.grid.export()
    rows = flatten_pairs(lst)
    out = set()
    for ci, cj, s, im, cm in rows:
        m = im | cm
        for i in range(4):
            for j in range(8):
                if m >> (i * 8 + j) & 1:
                    a, b = g["gid"][4 * ci + i], g["gid"][8 * cj + j]
                    out.add((min(a, b), max(a, b)))
    return out, rows


def test_half_list_covers_every_pair_once():
    """Every pair within rc appears in the inner list exactly once (half list, 14 shifts)."""
    s = systems.make("water3k")
    on = O.OracleNonbonded(s)
    on.search(s.x)
    lst = on.list.export(1)
    g = on.grid.export()
    rows = flatten_pairs(lst)
    assert rows[:, 2].min() >= 13  # half shell
    seen = {}
    for ci, cj, sh, im, cm in rows:
        m = im | cm
        for i in range(4):
            for j in range(8):
                if m >> (i * 8 + j) & 1:
                    a, b = int(g["gid"][4 * ci + i]), int(g["gid"][8 * cj + j])
                    key = (min(a, b), max(a, b))
                    seen[key] = seen.get(key, 0) + 1
    assert max(seen.values()) == 1
    x = s.x.astype(np.float64)
    d = x[:, None] - x[None]
    d -= s.box * np.round(d / s.box)
    r2 = (d**2).sum(-1)
    ia, ib = np.nonzero(np.triu(r2 < s.rc**2, 1))
    for a, b in zip(ia.tolist(), ib.tolist()):
        assert (a, b) in seen, f"pair {a},{b} within rc missing from list"


def test_exclusion_masks():
    """Excluded pairs carry correction bits, never interaction bits."""
    s = systems.make("rnase24k", 4000)
    on = O.OracleNonbonded(s)
    on.search(s.x)
    g = on.grid.export()
    rows = flatten_pairs(on.list.export(0))
    excl = set()
    for a in range(s.natoms):
        for b in s.excl_gids[s.excl_offsets[a]:s.excl_offsets[a + 1]]:
            excl.add((a, int(b)))
    n_corr = 0
    for ci, cj, sh, im, cm in rows:
        for i in range(4):
            for j in range(8):
                bit = 1 << (i * 8 + j)
                a, b = int(g["gid"][4 * ci + i]), int(g["gid"][8 * cj + j])
                if im & bit:
                    assert (a, b) not in excl
                if cm & bit:
                    assert (a, b) in excl
                    n_corr += 1
    assert n_corr > 0


def test_virial_matches_box_scaling_derivative():
    """tr(Xi) = -1/2 sum r.F = 1/2 dE/dlambda for uniform scaling x -> (1+l)x (fixed beta)."""
    s = systems.make("water3k")
    on = O.OracleNonbonded(s)
    on.search(s.x)
    _, _, vir, _ = on.forces()
    c = O.derive_consts(on.params)
    h = 1e-5
    es = []
    for lam in (-h, h):
        xs = s.x.astype(np.float64) * (1 + lam)
        _, eb, _ = brute_force(xs, s.q, s.type, s.c6c12, s.excl_offsets, s.excl_gids,
                               s.box.astype(np.float64) * (1 + lam), c, s.coulomb, s.rc)
        es.append(sum(eb))
    dE = (es[1] - es[0]) / (2 * h)
    assert abs(np.trace(vir) - 0.5 * dE) / abs(0.5 * dE) < 1e-3


def test_prune_rolling_equals_full():
    s = systems.make("mem82k", 5000)
    on = O.OracleNonbonded(s)
    on.search(s.x)
    rng = np.random.default_rng(1)
    x1 = (s.x + rng.uniform(-0.03, 0.03, s.x.shape)).astype(np.float32)
    on.put_x(x1)
    on.prune()
    full = on.list.export(1)
    on2 = O.OracleNonbonded(s)
    on2.search(s.x)
    on2.put_x(x1)
    for p in range(4):
        on2.prune(p, 4)
    roll = on2.list.export(1)
    for k in ("sci", "cj", "pool"):
        assert np.array_equal(full[k], roll[k])


def test_golden_fixtures():
    """Oracle vs the committed float64 brute-force fixtures (tools/make_golden.py)."""
    files = sorted(f for f in os.listdir(GOLDEN) if f.startswith("brute_") and f.endswith(".npz"))
    assert files, "golden fixtures missing"
    for fn in files:
        d = np.load(os.path.join(GOLDEN, fn))
        s = systems.System(fn, d["x"], d["q"], d["type"], d["c6c12"], d["excl_offsets"], d["excl_gids"],
                           d["box"], str(d["coulomb"]), float(d["rc"]), float(d["rlist_outer"]),
                           float(d["rlist_inner"]))
        on = O.OracleNonbonded(s)
        on.search(s.x)
        f, e, vir, _ = on.forces()
        rel = np.sqrt(((f - d["f"]) ** 2).sum() / (d["f"] ** 2).sum())
        assert rel < 5e-6, fn
        assert np.abs(vir - d["virial"]).max() / np.abs(d["virial"]).max() < 5e-6, fn
        assert abs(e[0] - d["energies"][0]) / abs(d["energies"][0]) < 1e-5, fn
        assert abs(e[1] - d["energies"][1]) / abs(d["energies"][1]) < float(d["coul_tol"]), fn
        # oracle list sizes are part of the fixture: the list algorithm is pinned too
        sz = on.list.sizes()
        assert [sz["n_sci"], sz["n_cj_outer"], sz["n_cj_inner"], sz["n_pool"]] == list(d["list_sizes"]), fn
        assert int(d["list_crc"]) == _list_crc(on.list.export(1)), fn


def _list_crc(lst):
    import zlib
    return zlib.crc32(lst["sci"].tobytes() + lst["cj"].tobytes() + lst["pool"].tobytes())


def test_force_switch_vs_brute_force():
    """Row f3: force-switch LJ (GROMACS vdw-modifier = force-switch) against float64."""
    s = systems.make("stmv_fsw", 6000)
    on = O.OracleNonbonded(s)
    on.search(s.x)
    f, e, vir, _ = on.forces()
    c = O.derive_consts(on.params)
    fb, eb, vb = brute_force(s.x, s.q, s.type, s.c6c12, s.excl_offsets, s.excl_gids, s.box, c, s.coulomb, s.rc,
                             lj_modifier="force-switch", rvdw_switch=s.rvdw_switch)
    assert np.sqrt(((f - fb) ** 2).sum() / (fb**2).sum()) < 5e-6
    assert abs(e[0] - eb[0]) / abs(eb[0]) < 1e-5
    assert np.abs(vir - vb).max() / np.abs(vb).max() < 5e-6
    # the switched force vanishes continuously at rc: a pair just inside rc has ~0 LJ force
    cf = O.derive_consts(O.make_params(**s.params()))
    assert cf["fsw_r1"] == np.float32(1.0)


def test_tabulated_ewald_vs_brute_force():
    """Row f3: tabulated Ewald real space (the paper's kernel flavour) against float64 with
    exact erfc, with force-switch LJ (the paper's STMV flavour)."""
    s = systems.make("stmv_tab", 6000)
    on = O.OracleNonbonded(s)
    on.search(s.x)
    f, e, vir, _ = on.forces()
    c = O.derive_consts(on.params)
    assert c["tab_n"] > 0
    fb, eb, vb = brute_force(s.x, s.q, s.type, s.c6c12, s.excl_offsets, s.excl_gids, s.box, c, "ewald", s.rc,
                             lj_modifier="force-switch", rvdw_switch=s.rvdw_switch)
    assert np.sqrt(((f - fb) ** 2).sum() / (fb**2).sum()) < 5e-6
    assert abs(e[0] - eb[0]) / abs(eb[0]) < 1e-5
    assert abs(e[1] - eb[1]) / abs(eb[1]) < 1e-5
    assert np.abs(vir - vb).max() / np.abs(vb).max() < 5e-6
    # and close to the analytical-rational flavour on the same list
    s2 = systems.make("stmv_fsw", 6000)
    on2 = O.OracleNonbonded(s2)
    on2.search(s2.x)
    f2, e2, _, _ = on2.forces()
    assert np.sqrt(((f - f2) ** 2).sum() / (f2**2).sum()) < 5e-6


@pytest.mark.parametrize("config", ["rnase24k_lb", "rnase24k_geom"])
def test_combination_rule_vs_brute_force(config):
    """Row f3: combination-rule LJ (the paper's Grappa kernel flavour).  The
    oracle's per-pair parameters come from per-type parameters, the brute force uses the
    (LB- or geometric-mixed) float64 table: forces, energies and virial agree."""
    s = systems.make(config, 3000)
    on = O.OracleNonbonded(s)
    on.search(s.x)
    f, e, vir, _ = on.forces()
    c = O.derive_consts(on.params)
    fb, eb, vb = brute_force(s.x, s.q, s.type, s.c6c12, s.excl_offsets, s.excl_gids, s.box, c, s.coulomb, s.rc)
    assert np.sqrt(((f - fb) ** 2).sum() / (fb**2).sum()) < 5e-6
    assert abs(e[0] - eb[0]) / abs(eb[0]) < 1e-5
    assert np.abs(vir - vb).max() / np.abs(vb).max() < 5e-6
    # the per-pair parameters reproduce the table (float rounding only)
    import ctypes as C
    nt = s.c6c12.shape[0]
    pt = np.zeros(2 * nt, dtype=np.float32)
    tab = np.ascontiguousarray(s.c6c12, dtype=np.float32)
    mod = {"comb-geom": 2, "comb-lb": 3}[s.lj_modifier]
    O.lib().ora_lj_comb_params(mod, nt, tab.ctypes.data_as(C.POINTER(C.c_float)), pt.ctypes.data_as(C.POINTER(C.c_float)))
    p = pt.reshape(nt, 2).astype(np.float64)
    if mod == 2:
        c6, c12 = np.outer(p[:, 0], p[:, 0]), np.outer(p[:, 1], p[:, 1])
    else:
        sg = p[:, 0][:, None] + p[:, 0][None, :]
        c6 = np.outer(p[:, 1], p[:, 1]) * sg**6
        c12 = 2.0 * c6 * sg**6
    np.testing.assert_allclose(c6, 6.0 * s.c6c12[..., 0], rtol=2e-6, atol=1e-12)
    np.testing.assert_allclose(c12, 12.0 * s.c6c12[..., 1], rtol=2e-6, atol=1e-18)


def test_grappa_flavour_vs_brute_force():
    """Row f3: the Grappa kernel flavour -- tabulated Ewald + LB combination-rule LJ."""
    s = systems.make("grappa1.5m", 3000)
    on = O.OracleNonbonded(s)
    on.search(s.x)
    f, e, vir, _ = on.forces()
    c = O.derive_consts(on.params)
    fb, eb, vb = brute_force(s.x, s.q, s.type, s.c6c12, s.excl_offsets, s.excl_gids, s.box, c, "ewald", s.rc)
    assert np.sqrt(((f - fb) ** 2).sum() / (fb**2).sum()) < 5e-6
    assert abs(e[0] - eb[0]) / abs(eb[0]) < 1e-5
    assert np.abs(vir - vb).max() / np.abs(vb).max() < 5e-6
