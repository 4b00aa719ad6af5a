"""GPU parity: libnbx.so (through its C-ABI via paper_2405_01420_b200.nbx) against the CPU
oracle (oracle/nbx_oracle.c) on identical inputs.

Bars (BASELINE.json north_star): grid layout, outer and inner pair lists and masks bit-exact;
forces rel RMS <= 1e-5 and max <= 1e-4; energies and virial relative error <= 1e-6.
"""
import functools

import numpy as np
import pytest

from oracle import oracle as O
from paper_2405_01420_b200 import systems
from tests.helpers import (assert_energies, assert_forces, assert_lists_equal, assert_virial,
                           flatten_pairs)

pytestmark = pytest.mark.gpu

SMALL = ["water3k", "rnase24k", "mem82k"]


@functools.lru_cache(maxsize=None)
def get_system(name, natoms=None):
    return systems.make(name, natoms)


def gpu_nb(system):
    from paper_2405_01420_b200 import nbx
    return nbx.Nonbonded(system, device=0)


def to_dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()


def run_pair(system, x=None):
    import torch
    x = system.x if x is None else x
    nb = gpu_nb(system)
    xd = to_dev(x)
    nb.search(xd)
    on = O.OracleNonbonded(system)
    on.search(x)
    torch.cuda.synchronize()
    return nb, on, xd


@pytest.mark.parametrize("name", SMALL)
def test_grid_bit_exact(gpu, name):
    s = get_system(name)
    nb, on, _ = run_pair(s)
    g = nb.grid_export()
    o = on.grid.export()
    assert nb.grid_info()["nslots"] == on.grid.nslots
    np.testing.assert_array_equal(g["order"], o["order"])
    np.testing.assert_array_equal(g["type"], o["type"])
    assert np.array_equal(g["xq"].view(np.uint32), o["xq"].view(np.uint32))


@pytest.mark.parametrize("name", SMALL)
def test_lists_bit_exact(gpu, name):
    s = get_system(name)
    nb, on, _ = run_pair(s)
    for which in (0, 1):
        assert_lists_equal(nb.pairlist(which), on.list.export(which), f"{name} list{which}")
    sz = nb.list_sizes()
    assert sz == on.list.sizes()
    assert sz["n_cj_inner"] <= sz["n_cj_outer"]


@pytest.mark.parametrize("name", SMALL)
def test_forces_energies_virial(gpu, name):
    import torch
    s = get_system(name)
    nb, on, xd = run_pair(s)
    f, (e, vir) = nb.forces(xd, energy=True, virial=True)
    torch.cuda.synchronize()
    fo, eo, viro, _ = on.forces()
    assert_forces(f.cpu().numpy(), fo)
    assert_energies(e, eo)
    assert_virial(vir, viro)
    # F-only variant gives the same forces
    f2 = nb.forces(xd)
    assert_forces(f2.cpu().numpy(), fo)


@pytest.mark.parametrize("name", SMALL)
def test_prune_after_motion(gpu, name):
    """Displace atoms (as between steps), prune: inner list bit-exact, forces in tolerance."""
    import torch
    s = get_system(name)
    nb, on, xd = run_pair(s)
    rng = np.random.default_rng(7)
    x1 = (s.x + rng.uniform(-0.03, 0.03, size=s.x.shape)).astype(np.float32)
    x1d = to_dev(x1)
    nb.put_x(x1d)
    nb.prune()
    on.put_x(x1)
    on.prune()
    assert_lists_equal(nb.pairlist(1), on.list.export(1), f"{name} pruned")
    f, (e, vir) = nb.forces(x1d, energy=True, virial=True)
    torch.cuda.synchronize()
    fo, eo, viro, _ = on.forces()
    assert_forces(f.cpu().numpy(), fo)
    assert_energies(e, eo)
    assert_virial(vir, viro)


@pytest.mark.parametrize("name", ["rnase24k", "water3k"])
def test_prune_kernels_identical(gpu, name, monkeypatch):
    """All prune kernels (NBX_PRUNE_KERNEL=0: lane per cj entry, 1: lane per i atom, 2: packed
    active tiles, per entry and -- NBX_PRUNE_SPLIT=1 -- split into 32-entry chunks plus a
    gather, the short-list form) give the oracle's inner list bit-exactly after motion, whole
    and rolling."""
    s = get_system(name)
    rng = np.random.default_rng(11)
    x1 = (s.x + rng.uniform(-0.04, 0.04, size=s.x.shape)).astype(np.float32)
    lists = []
    variants = (("0", "0"), ("1", "0"), ("2", "0"), ("2", "1"))
    for kern, split in variants:
        monkeypatch.setenv("NBX_PRUNE_KERNEL", kern)
        monkeypatch.setenv("NBX_PRUNE_SPLIT", split)
        nb, on, xd = run_pair(s)
        nb.put_x(to_dev(x1))
        for p in range(2):
            nb.prune(part=p, nparts=2)
        lists.append(nb.pairlist(1))
    on.put_x(x1)
    on.prune()
    for (kern, split), lg in zip(variants, lists):
        assert_lists_equal(lg, on.list.export(1), f"{name} prune kernel {kern} split {split}")


def test_rolling_prune_parts(gpu):
    """Rolling prune over 3 parts == one full prune (GROMACS-style rolling dynamic prune)."""
    s = get_system("rnase24k")
    nb, on, xd = run_pair(s)
    rng = np.random.default_rng(3)
    x1 = (s.x + rng.uniform(-0.03, 0.03, size=s.x.shape)).astype(np.float32)
    nb.put_x(to_dev(x1))
    for p in range(3):
        nb.prune(part=p, nparts=3)
    on.put_x(x1)
    on.prune()
    assert_lists_equal(nb.pairlist(1), on.list.export(1), "rolling")


def test_step_cadence(gpu):
    """Nonbonded.step applies the reference cadence (pipeline.py:222-235): search at 0,
    prune at 10, 20; forces every step match the oracle following the same schedule."""
    import torch
    s = get_system("water3k")
    nb = gpu_nb(s)
    on = O.OracleNonbonded(s)
    rng = np.random.default_rng(11)
    x = s.x.copy()
    f = torch.empty((s.natoms, 3), dtype=torch.float32, device="cuda")
    for step in range(0, 23):
        xd = to_dev(x)
        nb.step(xd, f, step)
        if step % s.nstlist == 0:
            on.search(x)
        else:
            on.put_x(x)
            if step % s.prune_every == 0:
                on.prune()
        if step in (0, 10, 21):
            torch.cuda.synchronize()
            assert_lists_equal(nb.pairlist(1), on.list.export(1), f"step{step}")
            fo, _, _, _ = on.forces(flags=0)
            assert_forces(f.cpu().numpy(), fo)
        x = (x + rng.uniform(-0.002, 0.002, size=x.shape)).astype(np.float32)


def test_oracle_force_on_gpu_list(gpu):
    """Force parity isolated from list parity: oracle forces on the GPU-built list."""
    import torch
    s = get_system("mem82k")
    nb, on, xd = run_pair(s)
    lst = nb.pairlist(1)
    g = nb.grid_export()
    fi, _, e2, _ = O.force_on_list(lst, g, g, on.c6c12, on.params, on.box, flags=1)
    fc = nb.forces(xd)
    torch.cuda.synchronize()
    fo = np.zeros((s.natoms, 3), np.float64)
    real = g["order"] >= 0
    fo[g["order"][real]] = fi[real]
    assert_forces(fc.cpu().numpy(), fo)


def test_two_particle_known_answer(gpu):
    """Two atoms (LJ + Ewald), across the periodic boundary: GPU vs float64 brute force."""
    import torch
    from oracle.brute import brute_force
    base = get_system("water3k")
    L = 3.0
    for coul in ("ewald", "rf"):
        for r in (0.3, 0.5, 0.85):
            x = np.array([[0.05, 1.0, 1.0], [0.05 - r, 1.0, 1.0]], np.float32) % L
            s = systems.System("pair", x, np.array([0.5, -0.7], np.float32), np.array([0, 0], np.int32),
                               base.c6c12, np.zeros(3, np.int32), np.zeros(0, np.int32),
                               np.full(3, L, np.float32), coul, 0.9, 1.0, 0.92)
            nb = gpu_nb(s)
            xd = to_dev(x)
            nb.search(xd)
            f, (e, vir) = nb.forces(xd, energy=True, virial=True)
            torch.cuda.synchronize()
            c = O.derive_consts(O.make_params(**s.params()))
            fb, eb, vb = brute_force(x, s.q, s.type, s.c6c12, s.excl_offsets, s.excl_gids, s.box, c, coul, 0.9)
            np.testing.assert_allclose(f.cpu().numpy(), fb, rtol=2e-5, atol=1e-3)
            np.testing.assert_allclose(e, eb, rtol=2e-5, atol=1e-4)
            np.testing.assert_allclose(vir, vb, rtol=2e-5, atol=1e-4)


def test_edge_geometry(gpu):
    """Ragged and degenerate inputs: atoms on/outside box faces, -0.0, several box images away,
    a count that is not a multiple of 32, all atoms in one column."""
    import torch
    base = get_system("water3k")
    rng = np.random.default_rng(5)
    L = 3.2
    n = 517
    g = (np.arange(8) + 0.5) * (L / 8)
    lat = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    x = (lat[rng.permutation(512)[:n - 5]] + rng.uniform(-0.05, 0.05, (n - 5, 3)))
    x = np.concatenate([np.zeros((5, 3)), x]).astype(np.float32)
    x[0] = [0.0, 0.0, 0.0]
    x[1] = [L, L, 1.3]
    x[2] = [-0.0, np.float32(L) - np.float32(1e-7), 1.7]
    x[3] = [-2 * L + 0.1, 3 * L + 0.2, 0.5]
    x[4] = [np.nextafter(np.float32(L), np.float32(0)), 0.6, -1e-8]
    x[5:40, 0:2] = 0.01  # a dense column
    x[5:40, 2] = np.linspace(0.0, L, 35, endpoint=False)
    q = rng.uniform(-0.5, 0.5, n).astype(np.float32)
    t = rng.integers(0, 2, n).astype(np.int32)
    eo = np.zeros(n + 1, np.int32)
    s = systems.System("edge", x, q, t, base.c6c12, eo, np.zeros(0, np.int32), np.full(3, L, np.float32),
                       "ewald", 0.9, 1.0, 0.92)
    nb, on, xd = run_pair(s)
    g = nb.grid_export()
    o = on.grid.export()
    np.testing.assert_array_equal(g["order"], o["order"])
    assert np.array_equal(g["xq"].view(np.uint32), o["xq"].view(np.uint32))
    for which in (0, 1):
        assert_lists_equal(nb.pairlist(which), on.list.export(which), f"edge list{which}")
    f, (e, vir) = nb.forces(xd, energy=True, virial=True)
    torch.cuda.synchronize()
    fo, eo_, viro, _ = on.forces()
    assert_forces(f.cpu().numpy(), fo)


def test_tiny_and_empty(gpu):
    import torch
    base = get_system("water3k")
    L = 3.0
    for n in (0, 1, 2, 33):
        x = (np.arange(3 * n, dtype=np.float32).reshape(n, 3) * 0.137) % L
        s = systems.System("tiny", x, np.full(n, 0.1, np.float32), np.zeros(n, np.int32), base.c6c12,
                           np.zeros(n + 1, np.int32), np.zeros(0, np.int32), np.full(3, L, np.float32),
                           "rf", 0.9, 1.0, 0.92)
        nb = gpu_nb(s)
        xd = to_dev(x.reshape(n, 3))
        nb.search(xd)
        f = nb.forces(xd)
        torch.cuda.synchronize()
        on = O.OracleNonbonded(s)
        on.search(x)
        fo, _, _, _ = on.forces()
        if n:
            assert_forces(f.cpu().numpy(), fo)
        assert_lists_equal(nb.pairlist(1), on.list.export(1), f"tiny{n}")


def test_bad_arguments_fail_loudly(gpu):
    from paper_2405_01420_b200 import nbx
    s = get_system("water3k")
    with pytest.raises(nbx.NbxError):
        nbx.Context(nbx.make_params(rc=1.0, rlist_outer=0.9, rlist_inner=0.95))
    nb = gpu_nb(s)
    with pytest.raises(nbx.NbxError):
        nb.prune()  # before search
    with pytest.raises(nbx.NbxError):
        nbx.check(nbx.lib().nbx_prune(nb.ctx.h, 0, 3, 2, None))


@pytest.mark.parametrize("name", ["stmv"])
def test_full_size_stmv(gpu, name):
    """The 1M-atom roofline config at full size: lists bit-exact, forces/energies in tolerance."""
    import torch
    s = get_system(name)
    nb, on, xd = run_pair(s)
    assert_lists_equal(nb.pairlist(1), on.list.export(1), f"{name} inner")
    f, (e, vir) = nb.forces(xd, energy=True, virial=True)
    torch.cuda.synchronize()
    fo, eo, viro, _ = on.forces()
    assert_forces(f.cpu().numpy(), fo)
    assert_energies(e, eo)
    assert_virial(vir, viro)
    # size-independent property: Newton's third law (sum of forces ~ 0)
    fsum = f.double().sum(0).abs().max().item()
    assert fsum <= 1e-6 * f.double().abs().sum().item()


def test_full_size_water12m_properties(gpu):
    """12M-atom box: GPU list == oracle list (bit-exact), forces vs oracle on the same list,
    Newton III and energy consistency between F and VF kernels."""
    import torch
    s = get_system("water12m")
    nb, on, xd = run_pair(s)
    assert_lists_equal(nb.pairlist(1), on.list.export(1), "12m inner")
    f, (e, vir) = nb.forces(xd, energy=True, virial=True)
    torch.cuda.synchronize()
    fo, eo, viro, _ = on.forces()
    assert_forces(f.cpu().numpy(), fo)
    assert_energies(e, eo)
    assert_virial(vir, viro)


def test_repeated_search_single_pass_and_overflow(gpu):
    """Second and later searches on a context use the single-pass search sized by the previous
    one; a denser configuration overflows those capacities and falls back to count + fill.
    Both must stay bit-exact with the oracle."""
    import torch
    s = get_system("rnase24k")
    nb = gpu_nb(s)
    rng = np.random.default_rng(9)
    xs = [s.x, (s.x + rng.uniform(-0.05, 0.05, s.x.shape)).astype(np.float32)]
    dense = s.x.copy()
    half = s.natoms // 2
    dense[:half] = (s.x[:half] * 0.55).astype(np.float32)  # squeeze half the atoms: denser lists
    xs.append(dense)
    for x in xs:
        nb.search(to_dev(x))
        torch.cuda.synchronize()
        on = O.OracleNonbonded(s)
        on.search(x)
        for which in (0, 1):
            assert_lists_equal(nb.pairlist(which), on.list.export(which), f"repeat list{which}")


def test_graph_steps_match_eager(gpu):
    """CUDA-graph replayed steps (Nonbonded.step(graphs=True), nbx_step_graph) give the eager
    forces, across several searches (graphs refreshed in place) and prune steps."""
    import dataclasses
    import torch
    s = dataclasses.replace(get_system("rnase24k"), nstlist=20, prune_every=5)
    nb_e, nb_g = gpu_nb(s), gpu_nb(s)
    rng = np.random.default_rng(2)
    x = to_dev(s.x)
    fe = torch.empty_like(x)
    fg = torch.empty_like(x)
    l0 = nb_g.launch_count()
    for step in range(0, 67):
        nb_e.step(x, fe, step)
        nb_g.step(x, fg, step, graphs=True)
        torch.cuda.synchronize()
        assert torch.equal(fe, fg) or float((fe - fg).abs().max()) < 1e-3 * float(fe.abs().max()), step
        x.add_(torch.from_numpy(rng.uniform(-0.002, 0.002, s.x.shape).astype(np.float32)).cuda())
    assert nb_g.launch_count() - l0 >= 67 * 3  # graph replays count their kernel nodes


def test_graph_cache_bounded(gpu):
    """A caller passing a fresh force tensor every step: the per-context graph cache evicts
    its oldest graph (16 kept) and every replay still gives the eager forces."""
    import torch
    s = get_system("water3k")
    nb = gpu_nb(s)
    x = to_dev(s.x)
    fe = torch.empty_like(x)
    nb.step(x, fe, 0)
    fe2 = torch.empty_like(x)
    nb.step(x, fe2, 1)
    for step in range(1, 40):
        fg = torch.empty_like(x)
        nb.step(x, fg, step if step % 10 else step + 1, graphs=True)
        torch.cuda.synchronize()
        assert float((fg - fe2).abs().max()) < 1e-3 * float(fe2.abs().max()), step


@pytest.mark.parametrize("natoms", [60000, None])
@pytest.mark.parametrize("config", ["stmv_fsw", "stmv_tab"])
def test_force_switch_flavour(gpu, natoms, config):
    """Row f3: force-switch LJ kernels (F and VF) vs the oracle, with the analytical or the
    tabulated Ewald correction (stmv_tab: the paper's STMV kernel flavour); None = full STMV."""
    import torch
    s = get_system(config, natoms)
    nb, on, xd = run_pair(s)
    f, (e, vir) = nb.forces(xd, energy=True, virial=True)
    f2 = nb.forces(xd)
    torch.cuda.synchronize()
    fo, eo, viro, _ = on.forces()
    assert_forces(f.cpu().numpy(), fo)
    assert_forces(f2.cpu().numpy(), fo)
    assert_energies(e, eo)
    assert_virial(vir, viro)


@pytest.mark.parametrize("config,natoms", [("rnase24k_lb", None), ("rnase24k_geom", None), ("grappa1.5m", 60000),
                                           ("grappa1.5m", None)])
def test_combination_rule_flavour(gpu, config, natoms):
    """Row f3: combination-rule LJ kernels (F and VF; grappa1.5m = the paper's Grappa flavour,
    tabulated Ewald + LB rule, at full size) vs the oracle: lists bit-exact, forces, energies
    and virial within the north_star tolerances."""
    import torch
    s = get_system(config, natoms)
    nb, on, xd = run_pair(s)
    assert_lists_equal(nb.pairlist(1), on.list.export(1), config)
    f, (e, vir) = nb.forces(xd, energy=True, virial=True)
    f2 = nb.forces(xd)
    torch.cuda.synchronize()
    fo, eo, viro, _ = on.forces()
    assert_forces(f.cpu().numpy(), fo)
    assert_forces(f2.cpu().numpy(), fo)
    assert_energies(e, eo)
    assert_virial(vir, viro)


def test_combination_rule_table_check(gpu):
    """A table that does not follow the selected rule is rejected (NBX_EINVAL), not silently
    replaced: the generator's LB-mixed protein table is not geometric."""
    from paper_2405_01420_b200 import nbx
    s = systems.make("rnase24k", 3000)
    s.lj_modifier = "comb-geom"
    with pytest.raises(nbx.NbxError, match="combination rule"):
        nbx.Nonbonded(s, device=0)
    s.lj_modifier = "comb-lb"
    nbx.Nonbonded(s, device=0)  # LB-mixed: accepted


@pytest.mark.parametrize("name", SMALL + ["stmv"])
def test_entry_order_longest_first(gpu, name, monkeypatch):
    """Row f2 (post-prune list sort by length; the reference's HIP prune_sort
    task, /root/reference/pkg/src/mdgpusim/pipeline.py:236-240): with the longest-first
    processing order the force kernel visits the same inner list in another order, so forces,
    energies and virial still match the oracle (the list itself is unchanged, bit-exact), after
    a search and after a moved-atom prune + graph step."""
    import torch
    monkeypatch.setenv("NBX_ENTRY_ORDER", "1")  # read by nbx_create
    s = get_system(name, 200000 if name == "stmv" else None)
    nb, on, xd = run_pair(s)
    assert_lists_equal(nb.pairlist(1), on.list.export(1), f"{name} sorted-order inner")
    f, (e, vir) = nb.forces(xd, energy=True, virial=True)
    torch.cuda.synchronize()
    fo, eo, viro, _ = on.forces()
    assert_forces(f.cpu().numpy(), fo)
    assert_energies(e, eo)
    assert_virial(vir, viro)
    rng = np.random.default_rng(5)
    x1 = (s.x + rng.uniform(-0.02, 0.02, size=s.x.shape)).astype(np.float32)
    x1d = to_dev(x1)
    fg = torch.empty_like(x1d)
    nb.graph_step(x1d, fg, prune=True)  # X op + prune (+ sort) + force + F op as one graph
    torch.cuda.synchronize()
    on.put_x(x1)
    on.prune()
    assert_lists_equal(nb.pairlist(1), on.list.export(1), f"{name} sorted-order pruned")
    fo1, _, _, _ = on.forces()
    assert_forces(fg.cpu().numpy(), fo1)
