"""Domain decomposition host logic on CPU: world_size 2 and 4 `gloo` ranks, oracle engine.

DD(N) forces/energies/virial == single-domain oracle; every interacting pair is computed on
exactly one rank (pair multisets identical after mapping to global ids)."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_01420_b200 import dd as DD
from paper_2405_01420_b200 import systems


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_balanced_dims_matches_reference():
    # pipeline.balanced_dims, pinned by the reference's tests/test_pipeline.py:69-76
    assert DD.balanced_dims(1) == (1, 1, 1)
    assert DD.balanced_dims(2) == (2, 1, 1)
    assert DD.balanced_dims(4) == (2, 2, 1)
    assert DD.balanced_dims(8) == (2, 2, 2)
    assert DD.balanced_dims(6) == (3, 2, 1)


def _system():
    # 3.0k waters: L = 4.48 nm >= 2 * 2 * rlist_outer for 2x2 splits
    return systems.water_box(3000, seed=21, coulomb="ewald", rc=1.0, rlist_outer=1.1, rlist_inner=1.02)


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from tests.dd_oracle_engine import OracleEngine
    s = _system()
    d = DD.DomainDecomposition(s, rank, world, lambda sy, pbc: OracleEngine(sy, pbc))
    x = torch.from_numpy(s.x)
    d.repartition(x)
    f, (e, vir) = d.step(None, step=1, energy=True, virial=True, prune=False)
    # pairs this rank computes (global ids), from the inner lists' interaction bits within rc
    eng = d.engine
    pairs = []
    for lst in (0, 1):
        gi = eng.grids[0].export()
        gj = eng.grids[lst].export()
        l = eng.lists[lst].export(1)
        for e_ in l["sci"]:
            for q in range(e_["cj_start"], e_["cj_end"]):
                meta = int(l["cj"][q]["meta"])
                im, p = meta & 0xFF, meta >> 8
                sh = int(e_["shift"])
                v = np.array([(sh % 3 - 1), ((sh // 3) % 3 - 1), (sh // 9 - 1)]) * s.box
                for k in range(8):
                    if not (im >> k & 1):
                        continue
                    m = int(l["pool"][p][k][0]) if p else 0xFFFFFFFF
                    ci, cj = 8 * int(e_["sci"]) + k, int(l["cj"][q]["cj"])
                    for i in range(4):
                        for j in range(8):
                            if m >> (i * 8 + j) & 1:
                                a, b = 4 * ci + i, 8 * cj + j
                                r = gi["xq"][a, :3] + v - gj["xq"][b, :3]
                                if (r * r).sum() < s.rc**2:
                                    ga, gb = int(gi["gid"][a]), int(gj["gid"][b])
                                    pairs.append((min(ga, gb), max(ga, gb)))
    np.savez(os.path.join(outdir, f"r{rank}.npz"), gid=d.home_gid.numpy(), f=f.numpy(), e=e, vir=vir,
             pairs=np.array(pairs, np.int64).reshape(-1, 2), n_home=d.n_home, n_ext=d.n_ext)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_dd_matches_single_domain(world):
    from oracle import oracle as O
    s = _system()
    with tempfile.TemporaryDirectory() as tmp:
        mp.start_processes(_worker, args=(world, _free_port(), tmp), nprocs=world, start_method="spawn")
        parts = [np.load(os.path.join(tmp, f"r{r}.npz")) for r in range(world)]
    gids = np.concatenate([p["gid"] for p in parts])
    assert np.array_equal(np.sort(gids), np.arange(s.natoms)), "every atom has exactly one home rank"
    f = np.zeros((s.natoms, 3))
    f[gids] = np.concatenate([p["f"] for p in parts])
    on = O.OracleNonbonded(s)
    on.search(s.x)
    fo, eo, viro, _ = on.forces()
    rel = np.sqrt(((f - fo) ** 2).sum() / (fo**2).sum())
    assert rel < 1e-5, rel
    e = parts[0]["e"]
    assert np.all(np.abs(e - eo) <= 1e-6 * np.abs(eo)), (e, eo)
    assert np.abs(parts[0]["vir"] - viro).max() <= 1e-6 * np.abs(viro).max()
    # pair multiset: each interacting pair exactly once across ranks
    allp = np.concatenate([p["pairs"] for p in parts])
    keys = allp[:, 0] * s.natoms + allp[:, 1]
    assert len(np.unique(keys)) == len(keys), "a pair was computed on two ranks"
    from scipy.spatial import cKDTree
    x = np.mod(s.x.astype(np.float64), s.box.astype(np.float64))
    tree = cKDTree(x, boxsize=s.box.astype(np.float64) * (1 + 1e-12))
    pr = tree.query_pairs(s.rc * (1 - 1e-6), output_type="ndarray")
    a, b = pr.min(1), pr.max(1)
    excl = set()
    for i in range(s.natoms):
        for j in s.excl_gids[s.excl_offsets[i]:s.excl_offsets[i + 1]]:
            excl.add((i, int(j)))
    ref = np.array([(i, j) for i, j in zip(a.tolist(), b.tolist()) if (i, j) not in excl], np.int64)
    # every pair clearly inside rc is computed (pairs within 1e-6 of rc may round either way)
    assert np.all(np.isin(ref[:, 0] * s.natoms + ref[:, 1], keys))
