"""CPU test double of dd.NbxEngine backed by the oracle (TEST INFRASTRUCTURE ONLY): lets the
domain-decomposition host logic run on CPU ranks with gloo (tests/test_dd.py)."""
import ctypes as C

import numpy as np
import torch

from oracle import oracle as O


class OracleEngine:
    def __init__(self, system, pbc):
        self.sys = system
        self.params = O.make_params(**system.params())
        self.consts = O.derive_consts(self.params)
        self.arrays = (np.ascontiguousarray(system.q, np.float32), np.ascontiguousarray(system.type, np.int32),
                       np.ascontiguousarray(system.excl_offsets, np.int32),
                       np.ascontiguousarray(system.excl_gids, np.int32))
        self.c6c12 = np.ascontiguousarray(system.c6c12, np.float32)
        self.box = np.asarray(system.box, np.float32)
        self.pbc = np.asarray(pbc, np.int32)
        self.density = system.natoms / float(np.prod(self.box.astype(np.float64)))
        self.grids = [None, None]
        self.lists = [None, None]
        self.f = [None, None]
        self.e2 = np.zeros(2)
        self.fsh = np.zeros((27, 3))

    def grid_build(self, g, x, gid, lo, size):
        self.grids[g] = O.OracleGrid(x.numpy(), gid.numpy(), self.arrays, self.box, self.pbc, lo, size,
                                     self.density)
        self.f[g] = np.zeros((self.grids[g].nslots, 3))

    def search(self, lst):
        self.lists[lst] = O.OracleList(self.grids[0], self.grids[lst], lst, self.params, self.box, self.pbc)

    def put_x(self, g, x, stream=None):
        if x.shape[0]:
            self.grids[g].put_x(x.numpy())

    def prune(self, lst, stream=None):
        self.lists[lst].prune()

    def force(self, lst, flags, stream=None):
        gi = self.grids[0].export()
        gj = self.grids[lst].export()
        fi, fj, e2, fsh = O.force_on_list(self.lists[lst].export(1), gi, gj, self.c6c12, self.params, self.box,
                                          flags=3, same=(lst == 0), nthreads=1)
        self.f[0] += fi
        if lst == 1:
            self.f[1] += fj
        self.e2 += e2
        self.fsh += fsh

    def clear_energies(self, stream=None):
        self.e2[:] = 0
        self.fsh[:] = 0

    def energies(self, stream=None):
        vir = np.zeros(9)
        w = np.zeros((3, 3))
        for g in (0, 1):
            if self.grids[g] is None:
                continue
            ex = self.grids[g].export()
            real = ex["order"] >= 0
            w += ex["xq"][real, :3].astype(np.float64).T @ self.f[g][real]
        for s in range(27):
            v = np.array([(s % 3 - 1) * self.box[0], ((s // 3) % 3 - 1) * self.box[1], (s // 9 - 1) * self.box[2]],
                         np.float32).astype(np.float64)
            w += np.outer(v, self.fsh[s])
        vir[:] = (-0.5 * w).ravel()
        eself = O.lib().ora_self_energy(C.byref(self.params), self.grids[0].sumq2())
        return np.array([self.e2[0], self.e2[1] + eself]), vir

    def get_f(self, g, f, accumulate=False, stream=None):
        if not f.shape[0]:
            return
        out = np.zeros((f.shape[0], 3), np.float32)
        O.lib().ora_grid_get_f(self.grids[g].h, O._p(self.f[g]), O._p(out), 0)
        if accumulate:
            f += torch.from_numpy(out)
        else:
            f.copy_(torch.from_numpy(out))
        self.f[g][:] = 0

    def count_pairs(self, lst):
        gi = self.grids[0].export()
        gj = self.grids[lst].export()
        l = self.lists[lst].export(1)
        n = O.lib().ora_count_pairs(len(l["sci"]), O._p(l["sci"]), O._p(l["cj"]), O._p(l["pool"]), O._p(gi["xq"]),
                                    O._p(gj["xq"]), C.byref(self.params), O._p(self.box))
        return n, 0

    def halo_pack(self, x, idx, shift, out, stream=None):
        if idx.numel():
            out.copy_(x[idx.long()] + torch.from_numpy(np.asarray(shift, np.float32)))

    def halo_unpack_add(self, f, idx, buf, stream=None):
        if idx.numel():
            f.index_add_(0, idx.long(), buf)

    def launch_count(self):
        return 0
