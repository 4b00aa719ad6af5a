"""Row f4 on the GPU: the sm_100a PME (spread / cuFFT / solve / gather, pme.cu) against the
float64 oracle restatement (oracle/pme.py) on identical inputs and grids, through the C-ABI;
and the leap-frog update.  The bar for PME is looser than the nonbonded one because the
charge grid is accumulated and transformed in fp32: forces rel RMS <= 2e-5, energy and
virial rel <= 1e-5 (the fp32 grid/FFT limit; the oracle's own grid error at these settings
is ~1e-4, tests/test_pme_oracle.py)."""
import numpy as np
import pytest

from oracle import pme as P
from paper_2405_01420_b200 import systems

pytestmark = pytest.mark.gpu

FTOL, ETOL = 2e-5, 1e-5


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


@pytest.mark.parametrize("config,natoms", [("rnase24k", None), ("water12m", 30000), ("stmv", 200000)])
def test_pme_matches_oracle(gpu, config, natoms):
    import torch
    from paper_2405_01420_b200 import pme
    s = systems.make(config, natoms)
    pm = pme.Pme.for_system(s)
    x, q = _dev(s.x), _dev(s.q)
    f, (e, vir) = pm.compute(x, q, energy=True, virial=True)
    f2 = pm.compute(x, q)  # force-only call gives the same forces
    torch.cuda.synchronize()
    Eo, fo, vo = P.pme(s.x, s.q, s.box, pm_beta(s), 138.935458, pm.nk, 4)
    fg = f.cpu().numpy().astype(np.float64)
    rel = np.sqrt(((fg - fo) ** 2).sum() / (fo**2).sum())
    assert rel <= FTOL, rel
    assert np.sqrt(((f2.cpu().numpy() - fo) ** 2).sum() / (fo**2).sum()) <= FTOL
    assert abs(e - Eo) / abs(Eo) <= ETOL, (e, Eo)
    assert np.abs(vir - vo).max() / np.abs(vo).max() <= ETOL
    assert pm.launch_count() >= 6


def pm_beta(s):
    from paper_2405_01420_b200 import nbx
    return float(nbx.derive_consts(nbx.make_params(**s.params()))["beta"])


def test_pme_accumulates_and_moves(gpu):
    """out= accumulates; coordinates outside the box (several images away) give the same
    forces as wrapped ones."""
    import torch
    from paper_2405_01420_b200 import pme
    s = systems.make("rnase24k", 3000)
    pm = pme.Pme.for_system(s)
    x, q = _dev(s.x), _dev(s.q)
    f1 = pm.compute(x, q)
    f = torch.ones_like(x)
    pm.compute(x, q, out=f)
    torch.testing.assert_close(f, f1 + 1.0, rtol=1e-5, atol=1e-3)  # fp32 atomics: order-dependent
    shift = np.array([2, -3, 1], dtype=np.float32) * s.box
    f3 = pm.compute(_dev(s.x + shift), q)
    torch.cuda.synchronize()
    rel = float((f3 - f1).norm() / f1.norm())
    assert rel < 1e-4, rel


def test_pme_rejects_bad_parameters(gpu):
    from paper_2405_01420_b200 import nbx, pme
    with pytest.raises(nbx.NbxError):
        pme.Pme([3.0, 3.0, 3.0], 3.0, nk=(25, 24, 24))
    with pytest.raises(nbx.NbxError):
        pme.Pme([3.0, 3.0, 3.0], 3.0, order=5)
    with pytest.raises(ValueError):
        pme.Pme.for_system(systems.make("water3k"))  # reaction field: no PME


def test_leapfrog(gpu):
    import torch
    from paper_2405_01420_b200 import pme
    rng = np.random.default_rng(3)
    n = 1000
    x, v, f = (rng.standard_normal((n, 3)).astype(np.float32) for _ in range(3))
    im = rng.uniform(0.05, 1.0, n).astype(np.float32)
    xd, vd, fd, imd = _dev(x), _dev(v), _dev(f), _dev(im)
    pme.leapfrog(xd, vd, fd, imd, 0.002)
    torch.cuda.synchronize()
    vn = v + f * im[:, None] * np.float32(0.002)
    np.testing.assert_allclose(vd.cpu().numpy(), vn, rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(xd.cpu().numpy(), x + vn * np.float32(0.002), rtol=1e-6, atol=1e-6)


def test_pme_profile_stages(gpu):
    """nbx_pme_profile: one evaluation with per-stage times under the reference's kernel kinds
    (pipeline.py:241-257); forces as from compute."""
    import torch
    from paper_2405_01420_b200 import pme
    s = systems.make("rnase24k")
    pm = pme.Pme.for_system(s)
    x, q = _dev(s.x), _dev(s.q)
    f = torch.zeros_like(x)
    ms = pm.profile(x, q, out=f)
    assert set(ms) == set(pme.Pme.STAGES) and all(v >= 0.0 for v in ms.values())
    f2 = pm.compute(x, q)
    torch.cuda.synchronize()
    assert float((f - f2).norm() / f2.norm()) < 1e-5


@pytest.mark.parametrize("config", ["rnase24k", "water12m"])
def test_pme_on_nonbonded_grid(gpu, config):
    """nbx_pme_compute_grid: PME on the nonbonded grid's cluster-ordered atoms with the forces
    added to its cluster force buffer -- Nonbonded.step(pme=...) returns NB + PME forces equal
    to the NB step plus the user-order PME (fp32 atomics: rel 1e-5)."""
    import torch
    from paper_2405_01420_b200 import nbx, pme
    s = systems.make(config, 30000 if config == "water12m" else None)
    nb = nbx.Nonbonded(s)
    pm = pme.Pme.for_system(s)
    x, q = _dev(s.x), _dev(s.q)
    f1 = torch.empty_like(x)
    f2 = torch.empty_like(x)
    for k in range(3):
        nb.step(x, f1, k, pme=pm)
    nb.step(x, f2, 3)
    f2p = pm.compute(x, q, out=f2.clone())
    f1b = torch.empty_like(x)
    nb.step(x, f1b, 4, pme=pm)
    e_grid = None
    nb.step(x, f1b, 5, energy=True, pme=pm)
    e_grid, _ = pm.energy()
    _, (e_user, _) = pm.compute(x, q, energy=True)
    torch.cuda.synchronize()
    rel = float((f1b - f2p).norm() / f2p.norm())
    assert rel < 1e-5, rel
    assert abs(e_grid - e_user) <= 1e-5 * abs(e_user)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_pme_random_noncubic_boxes(gpu, seed):
    """Random rectangular boxes (edges 2.6-6 nm, uneven grid sizes), uniform random atoms
    (some outside the box), random charges: GPU == oracle on the same grid."""
    from paper_2405_01420_b200 import pme
    rng = np.random.default_rng(100 + seed)
    box = rng.uniform(2.6, 6.0, 3).astype(np.float32)
    n = int(rng.integers(500, 5000))
    x = (rng.uniform(-0.5, 1.5, (n, 3)) * box).astype(np.float32)
    q = rng.uniform(-1, 1, n).astype(np.float32)
    beta = float(rng.uniform(2.5, 3.5))
    pm = pme.Pme(box, beta)
    f, (e, vir) = pm.compute(_dev(x), _dev(q), energy=True, virial=True)
    Eo, fo, vo = P.pme(x, q, box, beta, 138.935458, pm.nk, 4)
    fg = f.cpu().numpy().astype(np.float64)
    assert np.sqrt(((fg - fo) ** 2).sum() / (fo**2).sum()) <= FTOL
    assert abs(e - Eo) / abs(Eo) <= ETOL
    assert np.abs(vir - vo).max() / np.abs(vo).max() <= ETOL


def test_gpu_pme_against_golden_direct_sum(gpu):
    """The sm_100a PME (order 4) on a fine grid against the exact reciprocal Ewald sum of
    tests/golden/ewald_recip_600.npz: the physics anchor, not just the restatement."""
    import os
    from paper_2405_01420_b200 import pme
    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "ewald_recip_600.npz"))
    box = d["box"].astype(np.float32)
    pm = pme.Pme(box, float(d["beta"]), float(d["epsfac"]), nk=P.grid_dims(box, 0.04, 4))
    f, (e, vir) = pm.compute(_dev(d["x"]), _dev(d["q"]), energy=True, virial=True)
    fg = f.cpu().numpy().astype(np.float64)
    assert abs(e - float(d["energy"])) / abs(float(d["energy"])) < 1e-4
    assert np.sqrt(((fg - d["f"]) ** 2).sum() / (d["f"] ** 2).sum()) < 5e-4
    assert np.abs(vir - d["virial"]).max() / np.abs(d["virial"]).max() < 5e-4


def test_pme_edge_cases(gpu):
    """No atoms; all-zero charges; a bad grid index on the nonbonded-grid entry point."""
    import torch
    from paper_2405_01420_b200 import nbx, pme
    pm = pme.Pme([3.0, 3.2, 3.4], 3.1)
    x0 = torch.zeros((0, 3), device="cuda")
    q0 = torch.zeros((0,), device="cuda")
    f0, (e0, v0) = pm.compute(x0, q0, energy=True, virial=True)
    assert f0.shape == (0, 3) and e0 == 0.0 and np.all(v0 == 0.0)
    rng = np.random.default_rng(5)
    x = _dev(rng.uniform(0, 3, (100, 3)))
    fz, (ez, _) = pm.compute(x, torch.zeros(100, device="cuda"), energy=True)
    torch.cuda.synchronize()
    assert float(fz.abs().max()) == 0.0 and ez == 0.0
    s = systems.make("rnase24k", 3000)
    nb = nbx.Nonbonded(s)
    nb.search(_dev(s.x))
    with pytest.raises(nbx.NbxError):
        nbx.check(nbx.lib().nbx_pme_compute_grid(pm.h, nb.ctx.h, 5, 0, None))


def test_md_step_graph_matches_eager(gpu):
    """nbx_step_graph_pme: a whole non-search MD step (X op, prune, force, PME, F op, leap-frog)
    replayed as one graph gives the eager md_step's x and v, across searches (graph refreshed),
    prune steps and a PME box reset (graph re-captured).  PME spreads with fp32 atomics, so the
    two runs agree to rel 1e-5 in v, not bitwise."""
    import dataclasses
    import torch
    from paper_2405_01420_b200 import nbx, pme
    s = dataclasses.replace(systems.make("rnase24k"), nstlist=20, prune_every=5)
    runs = []
    for graphs in (False, True):
        nb = nbx.Nonbonded(s)
        pm = pme.Pme.for_system(s)
        x = _dev(s.x)
        v = torch.zeros_like(x)
        f = torch.empty_like(x)
        im = torch.full((s.natoms,), 0.1, dtype=torch.float32, device="cuda")
        l0 = nb.launch_count()
        for k in range(47):
            if k == 33:
                pm.set_box(s.box)
            nb.md_step(x, f, v, im, 1e-4, k, pm, graphs=graphs)
        torch.cuda.synchronize()
        runs.append((x, v, nb.launch_count() - l0))
    (xe, ve, _), (xg, vg, lg) = runs
    assert float((vg - ve).norm() / ve.norm()) < 1e-5
    assert float((xg - xe).abs().max()) < 1e-5
    assert float(ve.norm()) > 0
    assert lg >= 47 * 3  # graph replays count their kernel nodes
