"""Published known answers for the nonbonded physics.  TEST INFRASTRUCTURE ONLY.

The reference computes no forces, so nothing under
/root/reference pins the Ewald / reaction-field / Lennard-Jones conventions of DESIGN.md
section 3.  This module builds the classic crystal and molecule cases whose answers are in the
literature, so the oracle and libnbx are checked against numbers neither of them produced:

  * Madelung constants (nearest-neighbour convention), e.g. Kittel, "Introduction to Solid
    State Physics", ch. 3; Glasser & Zucker, "Lattice sums", Theor. Chem. Adv. Persp. 5 (1980):
      rock salt (NaCl)        M = 1.747564594633182
      caesium chloride (CsCl) M = 1.762674773070
    E_coulomb = -(N/2) * M * f q^2 / d  (N ions, d nearest-neighbour distance, f = 138.935458
    kJ mol^-1 nm e^-2): the Ewald real-space sum + reciprocal sum + self term must add to this.
  * Lennard-Jones lattice sums of the fcc lattice (Lennard-Jones & Ingham 1925; Kittel ch. 3;
    Ashcroft & Mermin ch. 20): A12 = sum_j (r_nn / r_j)^12 = 12.13188,
    A6 = sum_j (r_nn / r_j)^6 = 14.45392.  `lj_lattice_sums` enumerates the lattice in float64
    (pinned to these constants by the tests), and also returns the cut-off sums the
    potential-shift kernel computes, so E_lj of an fcc crystal has a closed form.
  * Reaction field (GROMACS convention, with the exclusion correction and
    the self term): for neutral molecules whose intermolecular pairs all lie inside rc,
        E_coul = f sum_{i in A, j in B, A != B} q_i q_j / r_ij  -  f k_rf |sum_i q_i x_i|^2,
    because sum_{i<j} q_i q_j r_ij^2 = -|mu|^2 for a neutral set and the c_rf terms cancel.
    For one isolated molecule this is -f k_rf mu^2: with eps_rf = inf (k_rf = 1 / (2 rc^3))
    the Onsager (1936) reaction-field energy of a point dipole in a spherical cavity of radius
    rc, -mu^2 / (2 rc^3) in Gaussian units.
"""
from __future__ import annotations

import math

import numpy as np

EPSFAC = 138.935458  # kJ mol^-1 nm e^-2 (GROMACS ONE_4PI_EPS0)
MADELUNG_NACL = 1.747564594633182
MADELUNG_CSCL = 1.762674773070
FCC_A12 = 12.13188
FCC_A6 = 14.45392


def _system(name, x, q, typ, c6c12, box, coulomb, rc, rlist_outer, rlist_inner, ewald_rtol=1e-8,
            excl_lists=None):
    from paper_2405_01420_b200.systems import System
    n = len(q)
    if excl_lists is None:
        offs = np.zeros(n + 1, np.int32)
        gids = np.zeros(0, np.int32)
    else:
        offs = np.zeros(n + 1, np.int32)
        offs[1:] = np.cumsum([len(e) for e in excl_lists])
        gids = np.array([g for e in excl_lists for g in e], np.int32)
    return System(name=name, x=np.asarray(x, np.float32), q=np.asarray(q, np.float32),
                  type=np.asarray(typ, np.int32), c6c12=np.asarray(c6c12, np.float32),
                  excl_offsets=offs, excl_gids=gids, box=np.asarray(box, np.float32), coulomb=coulomb,
                  rc=rc, rlist_outer=rlist_outer, rlist_inner=rlist_inner, ewald_rtol=ewald_rtol)


def _cells(n):
    return np.array([[i, j, k] for i in range(n) for j in range(n) for k in range(n)], np.float64)


def rock_salt(n=5, a0=0.564, rc=1.2, ewald_rtol=1e-8):
    """NaCl: n^3 conventional cells (8 n^3 ions, q = +-1), nearest-neighbour d = a0 / 2."""
    b = np.array([[0, 0, 0], [0, .5, .5], [.5, 0, .5], [.5, .5, 0]])
    na = (_cells(n)[:, None, :] + b[None]).reshape(-1, 3) * a0
    cl = na + np.array([0.5 * a0, 0.0, 0.0])
    x = np.concatenate([na, cl]) % (n * a0)
    q = np.concatenate([np.ones(len(na)), -np.ones(len(cl))])
    s = _system("nacl", x, q, np.zeros(len(q)), np.zeros((1, 1, 2)), np.full(3, n * a0), "ewald", rc,
                rc + 0.1, rc + 0.02, ewald_rtol)
    return s, 0.5 * a0, MADELUNG_NACL


def caesium_chloride(n=7, a0=0.4123, rc=1.2, ewald_rtol=1e-8):
    """CsCl: n^3 simple-cubic cells with a second ion at the body centre; d = a0 sqrt(3) / 2."""
    c = _cells(n) * a0
    x = np.concatenate([c, c + 0.5 * a0])
    q = np.concatenate([np.ones(len(c)), -np.ones(len(c))])
    s = _system("cscl", x, q, np.zeros(len(q)), np.zeros((1, 1, 2)), np.full(3, n * a0), "ewald", rc,
                rc + 0.1, rc + 0.02, ewald_rtol)
    return s, 0.5 * math.sqrt(3.0) * a0, MADELUNG_CSCL


def madelung_from_energy(e_coul, natoms, d, q=1.0):
    """M from the total Coulomb energy of an N-ion binary crystal: E = -(N/2) M f q^2 / d."""
    return -e_coul * d / (0.5 * natoms * EPSFAC * q * q)


def fcc_crystal(n=5, sigma=0.34, eps=0.99, rc=1.2, coulomb="rf"):
    """Neutral LJ fcc crystal at the pair-potential minimum spacing r_nn = 2^(1/6) sigma."""
    rnn = 2.0 ** (1.0 / 6.0) * sigma
    a0 = rnn * math.sqrt(2.0)
    b = np.array([[0, 0, 0], [0, .5, .5], [.5, 0, .5], [.5, .5, 0]])
    x = (_cells(n)[:, None, :] + b[None]).reshape(-1, 3) * a0
    c6, c12 = 4 * eps * sigma**6, 4 * eps * sigma**12
    s = _system("fcc", x, np.zeros(len(x)), np.zeros(len(x)), np.array([[[c6, c12]]]), np.full(3, n * a0),
                coulomb, rc, rc + 0.1, rc + 0.02)
    return s, rnn, c6, c12


def lj_lattice_sums(rcut_nn=None, rmax_nn=40.0):
    """fcc lattice sums in units of r_nn, float64 enumeration.

    Returns (A12, A6, count) over 0 < r <= rcut_nn (all three) when rcut_nn is given, else the
    infinite sums (A12, A6) with the analytic continuum tail beyond rmax_nn
    (4 pi rho / ((p - 3) R^(p-3)), rho = sqrt(2) sites per r_nn^3)."""
    R = rmax_nn if rcut_nn is None else rcut_nn
    m = int(math.ceil(R * math.sqrt(2.0))) + 1  # conventional cells (a0 = sqrt(2) r_nn)
    g = np.arange(-m, m + 1, dtype=np.float64)
    b = np.array([[0, 0, 0], [0, .5, .5], [.5, 0, .5], [.5, .5, 0]])
    A12 = A6 = 0.0
    cnt = 0
    for i in g:  # one slab of cells at a time (memory)
        c = np.stack(np.meshgrid([i], g, g, indexing="ij"), -1).reshape(-1, 3)
        p = (c[:, None, :] + b[None]).reshape(-1, 3) * math.sqrt(2.0)
        r2 = (p * p).sum(1)
        sel = (r2 > 0) & (r2 <= R * R * (1 + 1e-12))
        r2 = r2[sel]
        A12 += float((r2 ** -6).sum())
        A6 += float((r2 ** -3).sum())
        cnt += int(sel.sum())
    if rcut_nn is not None:
        return A12, A6, cnt
    rho = math.sqrt(2.0)
    return A12 + 4 * math.pi * rho / (9 * R**9), A6 + 4 * math.pi * rho / (3 * R**3)


def fcc_lj_energy(natoms, rnn, c6, c12, rc):
    """E_lj of an fcc crystal with the potential-shift cut-off at rc:
    (N/2) sum_{r_j < rc} [c12 (r^-12 - rc^-12) - c6 (r^-6 - rc^-6)], from the lattice sums."""
    A12, A6, cnt = lj_lattice_sums(rcut_nn=rc / rnn * (1 - 1e-9))
    per = c12 * (A12 / rnn**12 - cnt / rc**12) - c6 * (A6 / rnn**6 - cnt / rc**6)
    return 0.5 * natoms * per


def spce_molecule(o, h1, h2):
    return np.array([o, h1, h2], np.float64), np.array([-0.8476, 0.4238, 0.4238])


def two_waters(sep=0.31, box=3.2, rc=0.9):
    """Two rigid SPC/E waters (a hydrogen-bonded-like dimer) in an otherwise empty box."""
    from paper_2405_01420_b200.systems import SPCE_EPS, SPCE_SIG
    ang, b = np.deg2rad(109.47) / 2, 0.1
    c = np.full(3, box / 2)
    xa, qa = spce_molecule(c, c + b * np.array([np.sin(ang), 0, np.cos(ang)]),
                           c + b * np.array([-np.sin(ang), 0, np.cos(ang)]))
    o2 = c + np.array([0.0, 0.0, -sep])
    xb, qb = spce_molecule(o2, o2 + b * np.array([0, np.sin(ang), -np.cos(ang)]),
                           o2 + b * np.array([0, -np.sin(ang), -np.cos(ang)]))
    x = np.concatenate([xa, xb])
    q = np.concatenate([qa, qb])
    typ = np.array([0, 1, 1, 0, 1, 1])
    c6o, c12o = 4 * SPCE_EPS * SPCE_SIG**6, 4 * SPCE_EPS * SPCE_SIG**12
    c6c12 = np.zeros((2, 2, 2))
    c6c12[0, 0] = (c6o, c12o)
    excl = [[1, 2], [0, 2], [0, 1], [4, 5], [3, 5], [3, 4]]
    s = _system("two_waters", x, q, typ, c6c12, np.full(3, box), "rf", rc, rc + 0.1, rc + 0.02, excl_lists=excl)
    return s, [(0, 3), (3, 6)]


def rf_energy_closed_form(x, q, molecules, rc, epsfac=EPSFAC):
    """E_coul of neutral molecules under GROMACS reaction field with eps_rf = inf, all
    intermolecular pairs inside rc:  f sum_inter q_i q_j / r_ij - f k_rf |mu_total|^2."""
    x = np.asarray(x, np.float64)
    q = np.asarray(q, np.float64)
    krf = 1.0 / (2.0 * rc**3)
    e = 0.0
    for a, (a0, a1) in enumerate(molecules):
        for b, (b0, b1) in enumerate(molecules):
            if b <= a:
                continue
            d = x[a0:a1, None, :] - x[None, b0:b1, :]
            r = np.sqrt((d * d).sum(-1))
            assert r.max() < rc, "closed form needs every intermolecular pair inside rc"
            e += float((q[a0:a1, None] * q[None, b0:b1] / r).sum())
    mu = (q[:, None] * x).sum(0)
    return epsfac * e - epsfac * krf * float(mu @ mu)


def ewald_shift_energy(x, q, box, rc, sh_ewald, epsfac=EPSFAC):
    """The potential-shift part of the real-space Ewald energy, -f sh_ewald sum_{i<j, r<rc}
    q_i q_j (minimum image, float64): the kernels' convention V = f q q (erfc(beta r)/r -
    erfc(beta rc)/rc) minus the plain Ewald real-space sum."""
    x = np.asarray(x, np.float64)
    q = np.asarray(q, np.float64)
    box = np.asarray(box, np.float64)
    s = 0.0
    for a in range(len(q)):
        d = x[a + 1:] - x[a]
        d -= box * np.round(d / box)
        r2 = (d * d).sum(1)
        s += float(q[a] * q[a + 1:][r2 < rc * rc].sum())
    return -epsfac * sh_ewald * s


def ewald_tail_energy(x, q, box, rc, beta, epsfac=EPSFAC, rmax_tol=1e-17):
    """The real-space Ewald terms the cut-off drops, f sum_{i<j, images, r >= rc} q_i q_j
    erfc(beta r) / r (float64, all periodic images out to erfc(beta r) < rmax_tol)."""
    from scipy.special import erfc
    x = np.asarray(x, np.float64)
    q = np.asarray(q, np.float64)
    L = np.asarray(box, np.float64)
    rmax = rc
    while math.erfc(beta * rmax) > rmax_tol:
        rmax += 0.05
    nimg = [int(math.ceil(rmax / l)) for l in L]
    shifts = np.array([[a, b, c] for a in range(-nimg[0], nimg[0] + 1) for b in range(-nimg[1], nimg[1] + 1)
                       for c in range(-nimg[2], nimg[2] + 1)], np.float64) * L
    e = 0.0
    for a in range(len(q)):
        d = x[a] - x[None, :, :] + shifts[:, None, :]  # [S, N, 3]: x_a - (x_b - shift)
        r = np.sqrt((d * d).sum(-1))
        sel = (r >= rc) & (r < rmax)
        # every ordered (a, b, image) once; halve for unordered pairs (a == b images included:
        # an ion interacts with its own periodic images, each pair of images counted twice)
        e += 0.5 * float((q[a] * np.broadcast_to(q[None, :], r.shape)[sel] * erfc(beta * r[sel]) / r[sel]).sum())
    return epsfac * e
