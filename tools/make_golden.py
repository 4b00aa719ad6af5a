"""Generate tests/golden/ fixtures.

brute_*.npz   small synthetic systems with float64 brute-force forces/energies/virial
              (oracle/brute.py, exact erfc) plus the oracle's list sizes and list CRC.
ewald_recip_600.npz  exact reciprocal Ewald sum of a random neutral box (PME anchor, row f4).
costs_golden.json  the reference simulator's own cost-law outputs (imported from
              /root/reference/pkg/src, run in THIS container only) for the adapter tests.
"""
import json
import os
import sys
import zlib

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from oracle.brute import brute_force  # noqa: E402
from paper_2405_01420_b200 import systems  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def brute_fixture(tag, s, coul_tol):
    on = O.OracleNonbonded(s)
    on.search(s.x)
    c = O.derive_consts(on.params)
    fb, eb, vb = brute_force(s.x, s.q, s.type, s.c6c12, s.excl_offsets, s.excl_gids, s.box, c, s.coulomb, s.rc)
    sz = on.list.sizes()
    lst = on.list.export(1)
    crc = zlib.crc32(lst["sci"].tobytes() + lst["cj"].tobytes() + lst["pool"].tobytes())
    np.savez_compressed(os.path.join(OUT, f"brute_{tag}.npz"), x=s.x, q=s.q, type=s.type, c6c12=s.c6c12,
                        excl_offsets=s.excl_offsets, excl_gids=s.excl_gids, box=s.box, coulomb=s.coulomb,
                        rc=s.rc, rlist_outer=s.rlist_outer, rlist_inner=s.rlist_inner, f=fb,
                        energies=np.array(eb), virial=vb, coul_tol=coul_tol,
                        list_sizes=np.array([sz["n_sci"], sz["n_cj_outer"], sz["n_cj_inner"], sz["n_pool"]]),
                        list_crc=crc)
    print(tag, s.natoms, sz)


def ewald_recip_fixture():
    """Row f4: exact reciprocal-space Ewald sum (float64, explicit k vectors) of a random
    neutral 600-atom box, the anchor for the PME oracle and the GPU PME."""
    from oracle import pme as P
    rng = np.random.default_rng(2024)
    box = np.array([2.8, 3.1, 2.9])
    n = 600
    x = rng.uniform(0, 1, (n, 3)) * box
    q = rng.uniform(-1, 1, n)
    q -= q.mean()
    beta, eps = 3.1234, 138.935458
    E, f, v = P.ewald_recip_direct(x, q, box, beta, eps, tol=1e-14)
    np.savez_compressed(os.path.join(OUT, "ewald_recip_600.npz"), x=x, q=q, box=box, beta=beta, epsfac=eps,
                        energy=E, f=f, virial=v)
    print("ewald_recip_600", E)


def costs_golden():
    sys.path.insert(0, "/root/reference/pkg/src")
    from mdgpusim import costs, presets  # noqa
    t = costs.default_cost_table()
    out = {"anchors": [list(a) for a in costs.NBNXM_ANCHORS], "ratio": costs.NBNXM_BACKEND_RATIO, "points": []}
    for name, atoms in (("water3k", 3000), ("rnase24k", 24024), ("mem82k", 82000), ("stmv", 1066628),
                        ("water12m", 12000000)):
        for kind in ("NBNXM_LOCAL", "PRUNE_ONLY", "PAIR_SEARCH", "REDUCE_FORCES", "HALO_PACK_UNPACK"):
            for be in ("sycl", "hip"):
                k = getattr(costs.KernelKind, kind)
                out["points"].append([name, atoms, kind, be, t.duration_ns(k, atoms, be)])
    fit = costs.fit_affine([(1500, 19200.0), (6144000, 20000000.0)])
    out["fit_anchor"] = [fit.floor_ns, fit.slope_ns_per_atom]
    with open(os.path.join(OUT, "costs_golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("costs_golden.json", len(out["points"]))


if __name__ == "__main__" and "--ewald-only" in sys.argv:
    ewald_recip_fixture()
    sys.exit(0)

if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    brute_fixture("water_rf_1500", systems.water_box(500, seed=11, coulomb="rf", rc=0.9, rlist_outer=1.0,
                                                     rlist_inner=0.92), 2e-6)
    brute_fixture("protein_ewald_3000", systems.protein_box(3000, seed=12, rc=1.0), 5e-5)
    brute_fixture("membrane_ewald_3000", systems.membrane_box(3000, seed=13, rc=1.0), 5e-5)
    ewald_recip_fixture()
    if os.path.isdir("/root/reference/pkg/src"):
        costs_golden()
