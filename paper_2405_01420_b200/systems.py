"""Synthetic benchmark systems, deterministic per seed.

The reference sizes its benchmark systems by atom count, cut-off and density only
(`SystemPreset`, /root/reference/pkg/src/mdgpusim/presets.py:28-49, data/systems.cfg:79-106);
it carries no coordinates or force-field parameters.  These generators build coordinates,
charges, LJ types and exclusions of the named sizes at rho = 100 atoms/nm^3
(presets.py:41 density_per_nm3):

  water      SPC/E molecules on a jittered cubic lattice with random orientations
  protein    a sphere of bonded chain "residues" (1.3x water density, 8 LJ types,
             net-neutral 5-atom residues, 1-2/1-3 exclusions) solvated in SPC/E water
  membrane   a slab of neutral LJ tail beads (0.8x water density, 10-bead chains with
             1-2/1-3 exclusions) between two water layers

All arrays are numpy; the generators run in seconds even at 12 M atoms.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

RHO = 100.0  # atoms / nm^3 (presets.py:41)

# SPC/E (ext): q_O = -0.8476, q_H = +0.4238, sigma_O = 0.316557 nm, eps_O = 0.650194 kJ/mol
SPCE_QO, SPCE_QH = -0.8476, 0.4238
SPCE_SIG, SPCE_EPS = 0.316557, 0.650194
SPCE_BOND, SPCE_ANGLE = 0.1, np.deg2rad(109.47)


@dataclass
class System:
    name: str
    x: np.ndarray  # float32 [N,3]
    q: np.ndarray  # float32 [N]
    type: np.ndarray  # int32 [N]
    c6c12: np.ndarray  # float32 [T,T,2] plain (c6, c12)
    excl_offsets: np.ndarray  # int32 [N+1]
    excl_gids: np.ndarray  # int32 [nexcl]
    box: np.ndarray  # float32 [3]
    coulomb: str  # "rf" | "ewald" | "ewald-tab"
    rc: float
    rlist_outer: float
    rlist_inner: float
    epsilon_r: float = 1.0
    epsilon_rf: float = 0.0  # 0 = infinity
    ewald_rtol: float = 1e-5
    lj_modifier: str = "pot-shift"  # or "force-switch" (CHARMM/STMV flavour)
    rvdw_switch: float = 0.0
    nstlist: int = 100  # presets.py:44
    prune_every: int = 10  # presets.py:45
    dt_fs: float = 2.0  # presets.py:42
    seed: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def natoms(self) -> int:
        return int(self.x.shape[0])

    @property
    def ntypes(self) -> int:
        return int(self.c6c12.shape[0])

    def params(self) -> dict:
        return dict(coulomb=self.coulomb, rc=self.rc, rlist_outer=self.rlist_outer,
                    rlist_inner=self.rlist_inner, epsilon_r=self.epsilon_r,
                    epsilon_rf=self.epsilon_rf, ewald_rtol=self.ewald_rtol,
                    lj_modifier=self.lj_modifier, rvdw_switch=self.rvdw_switch)

    def expected_pairs(self) -> float:
        """In-cut-off unordered pairs at uniform density."""
        return self.natoms * RHO * (4.0 / 3.0) * np.pi * self.rc**3 / 2.0


# ----------------------------------------------------------------------------- helpers


def _lj_table(sigmas, epsilons) -> np.ndarray:
    """Lorentz-Berthelot mixed (c6, c12) table; zero rows for eps == 0 types."""
    s = np.asarray(sigmas, dtype=np.float64)
    e = np.asarray(epsilons, dtype=np.float64)
    sij = 0.5 * (s[:, None] + s[None, :])
    eij = np.sqrt(e[:, None] * e[None, :])
    c6 = 4.0 * eij * sij**6
    c12 = 4.0 * eij * sij**12
    return np.stack([c6, c12], axis=-1).astype(np.float32)


def _random_rotations(rng, n):
    qv = rng.normal(size=(n, 4))
    qv /= np.linalg.norm(qv, axis=1, keepdims=True)
    w, x, y, z = qv.T
    R = np.empty((n, 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z)
    R[:, 0, 1] = 2 * (x * y - z * w)
    R[:, 0, 2] = 2 * (x * z + y * w)
    R[:, 1, 0] = 2 * (x * y + z * w)
    R[:, 1, 1] = 1 - 2 * (x * x + z * z)
    R[:, 1, 2] = 2 * (y * z - x * w)
    R[:, 2, 0] = 2 * (x * z - y * w)
    R[:, 2, 1] = 2 * (y * z + x * w)
    R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def _water_molecules(rng, sites):
    """SPC/E molecules with O at `sites` (+-0.02 nm jitter), random orientation."""
    n = sites.shape[0]
    O = sites + rng.uniform(-0.02, 0.02, size=(n, 3))
    half = SPCE_ANGLE / 2
    h1 = np.array([np.sin(half), 0.0, np.cos(half)]) * SPCE_BOND
    h2 = np.array([-np.sin(half), 0.0, np.cos(half)]) * SPCE_BOND
    R = _random_rotations(rng, n)
    H1 = O + R @ h1
    H2 = O + R @ h2
    x = np.stack([O, H1, H2], axis=1).reshape(-1, 3)
    return x


def _lattice(L, nsites_min, rng=None):
    m = int(np.ceil(nsites_min ** (1.0 / 3.0)))
    a = L / m
    g = (np.arange(m) + 0.5) * a
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    return np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1), a


def _chain_exclusions(n, chain_len, start_gid):
    """1-2 and 1-3 exclusions inside consecutive chains of `chain_len` atoms."""
    lists = []
    for k in range(n):
        pos = k % chain_len
        lo = max(0, pos - 2)
        hi = min(chain_len - 1, pos + 2, n - 1 - (k - pos))
        lists.append([start_gid + k - pos + p for p in range(lo, hi + 1) if p != pos])
    return lists


def _water_exclusions(nw, start_gid):
    base = start_gid + 3 * np.arange(nw)
    o, h1, h2 = base, base + 1, base + 2
    return np.stack([np.stack([h1, h2], 1), np.stack([o, h2], 1), np.stack([o, h1], 1)], 1).reshape(-1, 2)


def _csr(n, per_atom_lists_or_fixed):
    if isinstance(per_atom_lists_or_fixed, np.ndarray):
        arr = per_atom_lists_or_fixed.astype(np.int32)
        k = arr.shape[1]
        offs = (np.arange(n + 1) * k).astype(np.int32)
        return offs, np.sort(arr, axis=1).ravel().astype(np.int32)
    offs = np.zeros(n + 1, dtype=np.int64)
    offs[1:] = np.cumsum([len(v) for v in per_atom_lists_or_fixed])
    flat = np.array([g for v in per_atom_lists_or_fixed for g in sorted(v)], dtype=np.int32)
    return offs.astype(np.int32), flat


def _concat_csr(parts):
    offs = [np.zeros(1, dtype=np.int64)]
    flat = []
    base = 0
    for o, f in parts:
        offs.append(o[1:].astype(np.int64) + base)
        base += int(o[-1])
        flat.append(f)
    return np.concatenate(offs).astype(np.int32), np.concatenate(flat).astype(np.int32)


# ----------------------------------------------------------------------------- systems


def water_box(n_waters: int, seed: int, coulomb="ewald", rc=1.0, rlist_outer=None,
              rlist_inner=None, name=None, epsilon_rf=0.0) -> System:
    rng = np.random.default_rng(seed)
    N = 3 * n_waters
    L = (N / RHO) ** (1.0 / 3.0)
    sites, a = _lattice(L, n_waters)
    if sites.shape[0] > n_waters:
        sites = sites[np.sort(rng.permutation(sites.shape[0])[:n_waters])]
    x = _water_molecules(rng, sites)
    x = np.mod(x, L).astype(np.float32)
    q = np.tile(np.array([SPCE_QO, SPCE_QH, SPCE_QH], dtype=np.float32), n_waters)
    t = np.tile(np.array([0, 1, 1], dtype=np.int32), n_waters)
    c6c12 = _lj_table([SPCE_SIG, 0.0], [SPCE_EPS, 0.0])
    eo, eg = _csr(N, _water_exclusions(n_waters, 0))
    return System(name or f"water{N}", x, q, t, c6c12, eo, eg,
                  np.full(3, L, dtype=np.float32), coulomb, rc,
                  rlist_outer or rc + 0.1, rlist_inner or rc + 0.02,
                  epsilon_rf=epsilon_rf, seed=seed)


# sigma range chosen so that nearest protein-lattice neighbours (0.197 nm at 1.3x density)
# are not in hard overlap (SURVEY.md proposed 0.25-0.38 nm)
PROT_SIG = [0.16, 0.175, 0.19, 0.205, 0.22, 0.235, 0.25, 0.265]
PROT_EPS = [0.1, 0.2, 0.35, 0.45, 0.55, 0.65, 0.8, 0.9]


def _split_counts(N, frac, mult):
    n = int(round(N * frac / mult)) * mult
    while (N - n) % 3 != 0:
        n += mult
    return n


def protein_box(natoms: int, seed: int, rc=1.0, rlist_outer=None, rlist_inner=None,
                frac=0.1, name=None) -> System:
    """Solvated protein-like blob: chains of 5-atom residues in a sphere (1.3x density)."""
    rng = np.random.default_rng(seed)
    N = natoms
    L = (N / RHO) ** (1.0 / 3.0)
    nprot = _split_counts(N, frac, 5)
    nw = (N - nprot) // 3
    rho_p = 1.3 * RHO
    R = (3 * nprot / (4 * np.pi * rho_p)) ** (1.0 / 3.0)
    c = np.full(3, L / 2)
    # protein sites: dense lattice inside the sphere, serpentine order -> chains
    a = rho_p ** (-1.0 / 3.0)
    m = int(np.ceil(2 * R / a)) + 2
    g = (np.arange(m) - (m - 1) / 2) * a
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    # serpentine: reverse every other row / plane so consecutive sites are neighbours
    Y = np.where((np.arange(m)[:, None, None] % 2) == 1, Y[:, ::-1, :], Y)
    Z = np.where(((np.arange(m)[:, None, None] * m + np.arange(m)[None, :, None]) % 2) == 1, Z[:, :, ::-1], Z)
    P = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1)
    r = np.linalg.norm(P, axis=1)
    order = np.argsort(r, kind="stable")[:nprot]
    P = P[np.sort(order)]  # keep serpentine order among the innermost nprot sites
    Rp = np.linalg.norm(P, axis=1).max()
    xp = c + P + rng.uniform(-0.015, 0.015, size=P.shape)
    tp = rng.integers(0, 8, size=nprot).astype(np.int32) + 2
    qp = rng.uniform(-0.8, 0.8, size=(nprot // 5, 5))
    qp = (qp - qp.mean(axis=1, keepdims=True)).ravel().astype(np.float32)
    # water outside the sphere
    sites, _ = _lattice(L, int(1.15 * nw / (1.0 - (4 / 3 * np.pi * (Rp + 0.25) ** 3) / L**3)) + 64)
    keep = np.linalg.norm(sites - c, axis=1) > Rp + 0.25
    sites = sites[keep]
    if sites.shape[0] < nw:
        raise RuntimeError("not enough water sites")
    sites = sites[np.sort(rng.permutation(sites.shape[0])[:nw])]
    xw = _water_molecules(rng, sites)
    x = np.mod(np.concatenate([xp, xw]), L).astype(np.float32)
    q = np.concatenate([qp, np.tile(np.array([SPCE_QO, SPCE_QH, SPCE_QH], np.float32), nw)])
    t = np.concatenate([tp, np.tile(np.array([0, 1, 1], np.int32), nw)])
    c6c12 = _lj_table([SPCE_SIG, 0.0] + PROT_SIG, [SPCE_EPS, 0.0] + PROT_EPS)
    ep = _csr(nprot, _chain_exclusions(nprot, 50, 0))
    ew = _csr(3 * nw, _water_exclusions(nw, 0) + nprot)
    eo, eg = _concat_csr([ep, ew])
    return System(name or f"protein{N}", x, q, t, c6c12, eo, eg,
                  np.full(3, L, dtype=np.float32), "ewald", rc,
                  rlist_outer or rc + 0.1, rlist_inner or rc + 0.02, seed=seed,
                  meta=dict(nprot=nprot, nwater=nw))


def membrane_box(natoms: int, seed: int, rc=1.0, rlist_outer=None, rlist_inner=None,
                 name=None) -> System:
    """Slab of neutral LJ tail beads (0.8x water density, z-middle third) between water."""
    rng = np.random.default_rng(seed)
    N = natoms
    L = (N / RHO) ** (1.0 / 3.0)
    rho_b = 0.8 * RHO
    t_slab = L / 3.0
    nb = _split_counts(N, rho_b * L * L * t_slab / N, 10)
    nw = (N - nb) // 3
    a = rho_b ** (-1.0 / 3.0)
    mxy = int(np.ceil(L / a))
    mz = int(np.ceil(nb / mxy**2))
    ax = L / mxy
    az = t_slab / mz
    gx = (np.arange(mxy) + 0.5) * ax
    gz = L / 3.0 + (np.arange(mz) + 0.5) * az
    # chains run along z (tail-like), serpentine within each (x,y) column
    X, Y, Z = np.meshgrid(gx, gx, gz, indexing="ij")
    P = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1)[:nb]
    xb = P + rng.uniform(-0.02, 0.02, size=P.shape)
    # water in the two outer thirds
    zlo, zhi = L / 3.0 - 0.15, 2 * L / 3.0 + 0.15
    sites, _ = _lattice(L, int(1.15 * nw * L / (L - (zhi - zlo))) + 64)
    keep = (sites[:, 2] < zlo) | (sites[:, 2] > zhi)
    sites = sites[keep]
    if sites.shape[0] < nw:
        raise RuntimeError("not enough water sites")
    sites = sites[np.sort(rng.permutation(sites.shape[0])[:nw])]
    xw = _water_molecules(rng, sites)
    x = np.mod(np.concatenate([xb, xw]), L).astype(np.float32)
    q = np.concatenate([np.zeros(nb, np.float32), np.tile(np.array([SPCE_QO, SPCE_QH, SPCE_QH], np.float32), nw)])
    t = np.concatenate([np.full(nb, 2, np.int32), np.tile(np.array([0, 1, 1], np.int32), nw)])
    c6c12 = _lj_table([SPCE_SIG, 0.0, 0.3905], [SPCE_EPS, 0.0, 0.4937])
    eb = _csr(nb, _chain_exclusions(nb, 10, 0))
    ew = _csr(3 * nw, _water_exclusions(nw, 0) + nb)
    eo, eg = _concat_csr([eb, ew])
    return System(name or f"membrane{N}", x, q, t, c6c12, eo, eg,
                  np.full(3, L, dtype=np.float32), "ewald", rc,
                  rlist_outer or rc + 0.1, rlist_inner or rc + 0.02, seed=seed,
                  meta=dict(nbeads=nb, nwater=nw))


# BASELINE.json "configs"
CONFIGS = {
    "water3k": dict(desc="SPC/E water box 3k atoms (1k waters), reaction-field, rc=0.9 nm"),
    "rnase24k": dict(desc="RNase-sized 24,024-atom solvated protein-like box, Ewald, rc=1.0 nm"),
    "mem82k": dict(desc="benchMEM-sized 82k-atom membrane-like box, Ewald, prune every 10"),
    "stmv": dict(desc="STMV-sized 1,066,628-atom water/protein box, Ewald, rc=1.2 nm"),
    "stmv_fsw": dict(desc="STMV box with force-switch LJ (rvdw_switch 1.0 nm, rc 1.2 nm)"),
    "stmv_tab": dict(desc="STMV box, the paper's STMV kernel flavour: tabulated Ewald + force-switch LJ"),
    "water12m": dict(desc="12M-atom water box, Ewald, rc=1.0 nm"),
    "rnase24k_lb": dict(desc="RNase-sized protein-like box, Ewald, Lorentz-Berthelot combination-rule LJ"),
    "rnase24k_geom": dict(desc="RNase-sized protein-like box (geometric LJ table), Ewald, geometric combination-rule LJ"),
    "grappa1.5m": dict(desc="Grappa-flavour kernel (PAPER.md:235): tabulated Ewald + Lorentz-Berthelot combination-rule LJ, "
                            "uniform-density 1.5M-atom water box, rc=1.0 nm"),
}


def geometric_table(c6c12: np.ndarray) -> np.ndarray:
    """(c6, c12) table with geometric mixing of its diagonal: c_ij = sqrt(c_ii c_jj)."""
    d = np.diagonal(c6c12.astype(np.float64), axis1=0, axis2=1).T  # [T, 2]
    t = np.sqrt(d[:, None, :] * d[None, :, :])
    return t.astype(np.float32)


def make(name: str, natoms: int | None = None) -> System:
    """Build a named benchmark system; `natoms` overrides the size (tests)."""
    if name == "water3k":
        n = natoms or 3000
        return water_box(n // 3, seed=1, coulomb="rf", rc=0.9, rlist_outer=1.0,
                         rlist_inner=0.92, name="water3k")
    if name == "rnase24k":
        return protein_box(natoms or 24024, seed=2, rc=1.0, name="rnase24k")
    if name == "mem82k":
        return membrane_box(natoms or 82000, seed=3, rc=1.0, name="mem82k")
    if name == "stmv":
        return protein_box(natoms or 1066628, seed=4, rc=1.2, frac=0.15, name="stmv")
    if name == "stmv_fsw":
        # the paper's STMV flavour: force-switch LJ (rvdw_switch 1.0, rc 1.2)
        s = protein_box(natoms or 1066628, seed=4, rc=1.2, frac=0.15, name="stmv_fsw")
        s.lj_modifier, s.rvdw_switch = "force-switch", 1.0
        return s
    if name == "stmv_tab":
        # the paper's STMV kernel flavour exactly: tabulated Ewald + force-switch LJ
        s = protein_box(natoms or 1066628, seed=4, rc=1.2, frac=0.15, name="stmv_tab")
        s.lj_modifier, s.rvdw_switch = "force-switch", 1.0
        s.coulomb = "ewald-tab"
        return s
    if name == "water12m":
        n = natoms or 12_000_000
        return water_box(n // 3, seed=5, coulomb="ewald", rc=1.0, name="water12m")
    if name == "rnase24k_lb":
        # the generator's table is Lorentz-Berthelot mixed (_lj_table): the LB rule reproduces it
        s = protein_box(natoms or 24024, seed=2, rc=1.0, name="rnase24k_lb")
        s.lj_modifier = "comb-lb"
        return s
    if name == "rnase24k_geom":
        s = protein_box(natoms or 24024, seed=2, rc=1.0, name="rnase24k_geom")
        s.c6c12 = geometric_table(s.c6c12)
        s.lj_modifier = "comb-geom"
        return s
    if name == "grappa1.5m":
        n = natoms or 1_500_000
        s = water_box(n // 3, seed=6, coulomb="ewald", rc=1.0, name="grappa1.5m")
        s.coulomb, s.lj_modifier = "ewald-tab", "comb-lb"
        return s
    raise KeyError(f"unknown system {name!r}; known: {sorted(CONFIGS)}")
