"""ctypes binding of the CPU oracle (liboracle.so).  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module, as the checker or the timed CPU baseline; the product (libnbx.so and
paper_2405_01420_b200/) never does.  See nbx_oracle.h for the parity status.

The class mirrors the product API (paper_2405_01420_b200.nbx.Nonbonded) on numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "nbx_oracle.c")

CFLAGS = ["-O3", "-std=c11", "-D_GNU_SOURCE", "-ffp-contract=off", "-mfma", "-mavx2",
          "-fopenmp", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile oracle/nbx_oracle.c -> oracle/liboracle.so (gcc; called by build())."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "nbx_oracle.h"))):
        subprocess.check_call(["gcc", *CFLAGS, "-o", LIB, SRC, "-lm"])
    return LIB


class Params(C.Structure):
    _fields_ = [("coulomb_type", C.c_int32), ("rc", C.c_float), ("rlist_outer", C.c_float),
                ("rlist_inner", C.c_float), ("epsilon_r", C.c_float), ("epsilon_rf", C.c_float),
                ("ewald_rtol", C.c_float), ("lj_modifier", C.c_int32), ("rvdw_switch", C.c_float)]


class Consts(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("epsfac", "k_rf", "c_rf", "beta", "sh_ewald", "sh_lj6",
                                         "sh_lj12", "rc2", "rlo2", "rli2", "fsw_r1", "fsw_a6", "fsw_b6",
                                         "fsw_a12", "fsw_b12", "fsw_p6", "fsw_q6", "fsw_p12", "fsw_q12",
                                         "fsw_c6", "fsw_c12", "tab_scale")] + [("tab_n", C.c_int32)]


class ListSizes(C.Structure):
    _fields_ = [("n_sci", C.c_int64), ("n_cj_outer", C.c_int64), ("n_cj_inner", C.c_int64),
                ("n_pool", C.c_int64)]


SCI_DTYPE = np.dtype([("sci", "<i4"), ("shift", "<i4"), ("cj_start", "<i4"), ("cj_end", "<i4")])
CJ_DTYPE = np.dtype([("cj", "<i4"), ("meta", "<u4")])
POOL_DTYPE = np.dtype(("<u4", (8, 2)))

_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        vp = C.c_void_p
        L.ora_derive_consts.argtypes = [C.POINTER(Params), C.POINTER(Consts)]
        L.ora_ewald_table.argtypes = [C.POINTER(Consts), C.c_void_p, C.c_void_p]
        L.ora_lj_comb_params.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_float)]
        L.ora_grid_build.restype = vp
        L.ora_grid_build.argtypes = [C.c_int, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_double]
        L.ora_grid_free.argtypes = [vp]
        for f in ("ora_grid_nslots", "ora_grid_ncx", "ora_grid_ncy"):
            getattr(L, f).argtypes = [vp]
            getattr(L, f).restype = C.c_int
        L.ora_grid_sumq2.argtypes = [vp]
        L.ora_grid_sumq2.restype = C.c_double
        L.ora_grid_export.argtypes = [vp, vp, vp, vp, vp]
        L.ora_grid_put_x.argtypes = [vp, vp]
        L.ora_search.restype = vp
        L.ora_search.argtypes = [vp, vp, C.c_int, C.POINTER(Params), vp, vp]
        L.ora_list_free.argtypes = [vp]
        L.ora_list_sizes.argtypes = [vp, C.POINTER(ListSizes)]
        L.ora_list_export.argtypes = [vp, C.c_int, vp, vp, vp]
        L.ora_prune.argtypes = [vp, vp, vp, C.POINTER(Params), vp, C.c_int, C.c_int]
        L.ora_force.argtypes = [C.c_int, vp, vp, vp, vp, vp, vp, vp, C.c_int, vp, C.POINTER(Params),
                                vp, C.c_uint, vp, vp, vp, vp, C.c_int]
        L.ora_count_pairs.argtypes = [C.c_int, vp, vp, vp, vp, vp, C.POINTER(Params), vp]
        L.ora_count_pairs.restype = C.c_longlong
        L.ora_self_energy.argtypes = [C.POINTER(Params), C.c_double]
        L.ora_self_energy.restype = C.c_double
        L.ora_grid_get_f.argtypes = [vp, vp, vp, C.c_int]
        L.ora_virial.argtypes = [vp, vp, vp, vp, vp]
        L.ora_ewald_G.argtypes = [C.c_float]
        L.ora_ewald_G.restype = C.c_float
        L.ora_ewald_H.argtypes = [C.c_float]
        L.ora_ewald_H.restype = C.c_float
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def make_params(coulomb="ewald", rc=1.0, rlist_outer=1.1, rlist_inner=1.02, epsilon_r=1.0,
                epsilon_rf=0.0, ewald_rtol=1e-5, lj_modifier="pot-shift", rvdw_switch=0.0) -> Params:
    return Params({"rf": 0, "ewald": 1, "ewald-tab": 2}[coulomb], rc, rlist_outer, rlist_inner, epsilon_r,
                  epsilon_rf, ewald_rtol, {"pot-shift": 0, "force-switch": 1, "comb-geom": 2, "comb-lb": 3}[lj_modifier], rvdw_switch)


def ewald_table(params: Params):
    """EWALD_TAB (value, next - value) tables: (ftab[tab_n, 2], vtab[tab_n, 2])."""
    c = Consts()
    lib().ora_derive_consts(C.byref(params), C.byref(c))
    ft = np.zeros((c.tab_n, 2), np.float32)
    vt = np.zeros((c.tab_n, 2), np.float32)
    if lib().ora_ewald_table(C.byref(c), _p(ft), _p(vt)):
        raise ValueError("no Ewald table for these parameters")
    return ft, vt


def derive_consts(params: Params) -> dict:
    c = Consts()
    lib().ora_derive_consts(C.byref(params), C.byref(c))
    return {n: getattr(c, n) for n, _ in Consts._fields_}


def grid_dims(size, density):
    """Python restatement of ora_grid_dims (for tests)."""
    s = (32.0 / density) ** (1.0 / 3.0)
    n = [max(1, int(np.floor(float(np.float32(v)) / s + 0.5))) for v in size[:2]]
    return n


class OracleGrid:
    def __init__(self, x, gid, system_arrays, box, pbc, lo, size, density):
        q, t, eo, eg = system_arrays
        self._keep = [q, t, eo, eg]
        x = np.ascontiguousarray(x, dtype=np.float32)
        gid = None if gid is None else np.ascontiguousarray(gid, dtype=np.int32)
        self.box = np.ascontiguousarray(box, dtype=np.float32)
        self.pbc = np.ascontiguousarray(pbc, dtype=np.int32)
        lo = np.ascontiguousarray(lo, dtype=np.float32)
        size = np.ascontiguousarray(size, dtype=np.float32)
        self.n = x.shape[0]
        self.h = lib().ora_grid_build(self.n, _p(x), _p(gid), _p(q), _p(t), _p(eo), _p(eg),
                                      _p(self.box), _p(self.pbc), _p(lo), _p(size), density)
        self.nslots = lib().ora_grid_nslots(self.h)
        self.ncx = lib().ora_grid_ncx(self.h)
        self.ncy = lib().ora_grid_ncy(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ora_grid_free(self.h)
            self.h = None

    def export(self):
        ns = self.nslots
        order = np.empty(ns, np.int32)
        xq = np.empty((ns, 4), np.float32)
        typ = np.empty(ns, np.int32)
        gid = np.empty(ns, np.int32)
        lib().ora_grid_export(self.h, _p(order), _p(xq), _p(typ), _p(gid))
        return dict(order=order, xq=xq, type=typ, gid=gid)

    def put_x(self, x):
        x = np.ascontiguousarray(x, dtype=np.float32)
        lib().ora_grid_put_x(self.h, _p(x))

    def sumq2(self):
        return lib().ora_grid_sumq2(self.h)


class OracleList:
    def __init__(self, gi: OracleGrid, gj: OracleGrid, mode: int, params: Params, box, pbc):
        self.gi, self.gj, self.mode, self.params = gi, gj, mode, params
        self.box = np.ascontiguousarray(box, dtype=np.float32)
        self.pbc = np.ascontiguousarray(pbc, dtype=np.int32)
        self.h = lib().ora_search(gi.h, gj.h, mode, C.byref(params), _p(self.box), _p(self.pbc))

    def __del__(self):
        if getattr(self, "h", None):
            lib().ora_list_free(self.h)
            self.h = None

    def sizes(self):
        s = ListSizes()
        lib().ora_list_sizes(self.h, C.byref(s))
        return dict(n_sci=s.n_sci, n_cj_outer=s.n_cj_outer, n_cj_inner=s.n_cj_inner, n_pool=s.n_pool)

    def export(self, which: int):
        s = self.sizes()
        sci = np.empty(s["n_sci"], SCI_DTYPE)
        cj = np.empty(s["n_cj_outer"] if which == 0 else s["n_cj_inner"], CJ_DTYPE)
        pool = np.empty(s["n_pool"], POOL_DTYPE)
        lib().ora_list_export(self.h, which, _p(sci), _p(cj), _p(pool))
        return dict(sci=sci, cj=cj, pool=pool)

    def prune(self, part=0, nparts=1):
        lib().ora_prune(self.h, self.gi.h, self.gj.h, C.byref(self.params), _p(self.box), part, nparts)


def force_on_list(lst: dict, gi: dict, gj: dict, c6c12, params: Params, box, flags=3,
                  same=True, nthreads=0):
    """Evaluate forces over explicit list arrays (e.g. exported from the GPU)."""
    ntypes = c6c12.shape[0]
    c6c12 = np.ascontiguousarray(c6c12, dtype=np.float32)
    box = np.ascontiguousarray(box, dtype=np.float32)
    fi = np.zeros((gi["xq"].shape[0], 3), np.float64)
    fj = fi if same else np.zeros((gj["xq"].shape[0], 3), np.float64)
    e2 = np.zeros(2, np.float64)
    fsh = np.zeros((27, 3), np.float64)
    sci = np.ascontiguousarray(lst["sci"])
    cj = np.ascontiguousarray(lst["cj"])
    pool = np.ascontiguousarray(lst["pool"])
    lib().ora_force(len(sci), _p(sci), _p(cj), _p(pool), _p(gi["xq"]), _p(gi["type"]), _p(gj["xq"]),
                    _p(gj["type"]), ntypes, _p(c6c12), C.byref(params), _p(box), flags, _p(fi), _p(fj),
                    _p(e2), _p(fsh), nthreads)
    return fi, fj, e2, fsh


class OracleNonbonded:
    """Single-domain oracle pipeline, mirroring paper_2405_01420_b200.nbx.Nonbonded."""

    def __init__(self, system):
        self.sys = system
        self.params = make_params(**system.params())
        self.arrays = (np.ascontiguousarray(system.q, np.float32), np.ascontiguousarray(system.type, np.int32),
                       np.ascontiguousarray(system.excl_offsets, np.int32),
                       np.ascontiguousarray(system.excl_gids, np.int32))
        self.c6c12 = np.ascontiguousarray(system.c6c12, np.float32)
        self.box = np.asarray(system.box, np.float32)
        self.pbc = np.ones(3, np.int32)
        self.density = system.natoms / float(np.prod(self.box.astype(np.float64)))
        self.grid = None
        self.list = None

    def search(self, x):
        self.grid = OracleGrid(x, None, self.arrays, self.box, self.pbc, np.zeros(3, np.float32),
                               self.box, self.density)
        self.list = OracleList(self.grid, self.grid, 0, self.params, self.box, self.pbc)

    def put_x(self, x):
        self.grid.put_x(x)

    def prune(self, part=0, nparts=1):
        self.list.prune(part, nparts)

    def count_pairs(self):
        g = self.grid.export()
        lst = self.list.export(1)
        return lib().ora_count_pairs(len(lst["sci"]), _p(lst["sci"]), _p(lst["cj"]), _p(lst["pool"]),
                                     _p(g["xq"]), _p(g["xq"]), C.byref(self.params), _p(self.box))

    def forces(self, flags=3, lst=None, nthreads=0):
        g = self.grid.export()
        if lst is None:
            lst = self.list.export(1)
        fi, _, e2, fsh = force_on_list(lst, g, g, self.c6c12, self.params, self.box, flags,
                                       same=True, nthreads=nthreads)
        f = np.zeros((self.sys.natoms, 3), np.float32)
        lib().ora_grid_get_f(self.grid.h, _p(fi), _p(f), 0)
        vir = np.zeros(9, np.float64)
        lib().ora_virial(self.grid.h, _p(fi), _p(fsh), _p(self.box), _p(vir))
        eself = lib().ora_self_energy(C.byref(self.params), self.grid.sumq2())
        energies = np.array([e2[0], e2[1] + eself])
        return f, energies, vir.reshape(3, 3), fsh


def ewald_G(z):
    return lib().ora_ewald_G(float(z))


def ewald_H(z):
    return lib().ora_ewald_H(float(z))
