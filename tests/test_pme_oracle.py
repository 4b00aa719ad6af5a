"""Row f4 oracle (CPU): the PME restatement (oracle/pme.py) against the exact reciprocal
Ewald sum, the virial against the box-scaling derivative, and the full Ewald energy (the
nonbonded oracle's real space + exclusion and self terms + PME) against float64 direct sums."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from oracle import pme as P
from paper_2405_01420_b200 import systems

EPS = 138.935458


def _random_box(n=200, seed=0):
    rng = np.random.default_rng(seed)
    L = np.array([2.5, 2.7, 2.6])
    x = rng.uniform(0, 1, (n, 3)) * L
    q = rng.uniform(-1, 1, n)
    q -= q.mean()
    return x, q, L


@pytest.mark.parametrize("spacing,order,etol,ftol", [(0.12, 4, 1e-3, 3e-3), (0.08, 4, 2e-4, 1e-3),
                                                     (0.06, 6, 1e-6, 5e-6)])
def test_pme_converges_to_direct_sum(spacing, order, etol, ftol):
    x, q, L = _random_box()
    beta = 3.1234
    Ed, fd, vd = P.ewald_recip_direct(x, q, L, beta, EPS)
    E, f, v = P.pme(x, q, L, beta, EPS, P.grid_dims(L, spacing, order), order)
    assert abs(E - Ed) / abs(Ed) < etol
    assert np.sqrt(((f - fd) ** 2).sum() / (fd**2).sum()) < ftol
    assert np.abs(v - vd).max() / np.abs(vd).max() < 5 * etol


def test_pme_virial_is_box_derivative():
    """Xi_aa = 1/2 dE/d(eps_a) under x -> (1 + eps_a) x, L -> (1 + eps_a) L (fixed grid)."""
    x, q, L = _random_box(seed=1)
    beta, nk = 3.1234, P.grid_dims(L, 0.1)
    _, _, v = P.pme(x, q, L, beta, EPS, nk)
    h = 1e-5
    for a in range(3):
        s = np.ones(3)
        s[a] = 1 + h
        Ep, _, _ = P.pme(x * s, q, L * s, beta, EPS, nk)
        s[a] = 1 - h
        Em, _, _ = P.pme(x * s, q, L * s, beta, EPS, nk)
        assert abs(0.5 * (Ep - Em) / (2 * h) - v[a, a]) < 1e-6 * np.abs(v).max()


def test_bspline_partition_of_unity():
    w = np.linspace(0, 0.999, 50)
    x = np.stack([w, w, w], 1) * 0 + np.array([[0.3, 1.7, 2.2]])
    th, dth, _ = P.splines(np.repeat(x, 1, 0), np.array([2.5, 2.5, 2.5]), (20, 20, 20))
    np.testing.assert_allclose(th.sum(-1), 1.0, rtol=1e-12)
    np.testing.assert_allclose(dth.sum(-1), 0.0, atol=1e-12)


def test_grid_dims_are_fft_friendly():
    for L in (3.1, 6.2, 22.0, 49.3):
        (k,) = P.grid_dims([L], 0.12)[:1]
        assert k % 2 == 0 and k >= L / 0.12
        r = k
        for p in (2, 3, 5, 7):
            while r % p == 0:
                r //= p
        assert r == 1


def _direct_real(x, q, L, beta, rc, excl_pairs):
    """float64 real-space Ewald (minimum image, r < rc) plus exclusion correction and self."""
    n = len(q)
    E = 0.0
    ex = set(map(tuple, excl_pairs))
    for i in range(n):
        d = x[i + 1:] - x[i]
        d -= L * np.round(d / L)
        r = np.sqrt((d**2).sum(1))
        js = np.arange(i + 1, n)
        for j, rr in zip(js, r):
            qq = q[i] * q[j]
            if (i, j) in ex:
                E -= EPS * qq * math.erf(beta * rr) / rr
            elif rr < rc:
                E += EPS * qq * (math.erfc(beta * rr) / rr - math.erfc(beta * rc) / rc)
    E -= EPS * beta / math.sqrt(math.pi) * (q**2).sum()
    return E


def test_full_ewald_energy():
    """Nonbonded oracle E_coul (real space, exclusion correction, self term) + PME = the float64
    Ewald energy of the same molecules, within the real-space tolerance and grid error."""
    s = systems.make("rnase24k", 1500)
    on = O.OracleNonbonded(s)
    on.search(s.x)
    _, e, _, _ = on.forces()
    c = O.derive_consts(on.params)
    beta = float(c["beta"])
    Erec, _, _ = P.pme(s.x, s.q, s.box, beta, float(c["epsfac"]), P.grid_dims(s.box, 0.06, 6), 6)
    excl = []
    for i in range(s.natoms):
        for j in s.excl_gids[s.excl_offsets[i]:s.excl_offsets[i + 1]]:
            if j > i:
                excl.append((i, int(j)))
    Ereal = _direct_real(s.x.astype(np.float64), s.q.astype(np.float64), s.box.astype(np.float64), beta,
                         float(s.rc), excl)
    Erec_d, _, _ = P.ewald_recip_direct(s.x, s.q, s.box, beta, float(c["epsfac"]))
    E_ref = Ereal + Erec_d
    assert abs(Erec - Erec_d) / abs(Erec_d) < 5e-6  # order 6, spacing 0.06 nm: grid error
    # the fp32 real-space pair energies cancel (E_coul within 5e-5 of
    # exact), so the bar is relative to the size of the two halves, not to their sum
    assert abs((e[1] + Erec) - E_ref) < 5e-5 * (abs(Ereal) + abs(Erec_d))


def test_pme_oracle_matches_golden_direct_sum():
    """tests/golden/ewald_recip_600.npz (tools/make_golden.py): the exact reciprocal-space sum
    of a random neutral box; the oracle PME at order 6 / 0.05 nm reproduces it."""
    import os
    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "ewald_recip_600.npz"))
    x, q, box, beta, eps = d["x"], d["q"], d["box"], float(d["beta"]), float(d["epsfac"])
    E, f, v = P.pme(x, q, box, beta, eps, P.grid_dims(box, 0.05, 6), 6)
    assert abs(E - float(d["energy"])) / abs(float(d["energy"])) < 2e-6
    assert np.sqrt(((f - d["f"]) ** 2).sum() / (d["f"] ** 2).sum()) < 1e-5
    assert np.abs(v - d["virial"]).max() / np.abs(d["virial"]).max() < 1e-5
