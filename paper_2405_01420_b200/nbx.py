"""Python host API over libnbx.so (ctypes; torch only for device memory and streams).

The reference has no physics API for this path; its only interface is
`CostTable.duration_ns(kind, atoms, backend, scale)` (/root/reference/pkg/src/mdgpusim/
costs.py:137-140), driven per MD step by `pipeline._single_rank_app` (pipeline.py:217-261).
`Nonbonded` is the real computation behind those simulated kernels and keeps the same step
cadence: search when step % nstlist == 0, prune when not searching and
step % prune_every == 0, force every step (pipeline.py:223-224, pinned by
tests/test_pipeline.py:103-115 of the reference).

There is no CPU fallback: importing this module without libnbx.so, or constructing a
`Nonbonded` without an sm_100 GPU, raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NBX_LIB") or os.path.join(HERE, "libnbx.so")  # NBX_LIB: variant builds (tools/)

NBX_COULOMB_RF, NBX_COULOMB_EWALD, NBX_COULOMB_EWALD_TAB = 0, 1, 2
LIST_LOCAL, LIST_NONLOCAL = 0, 1
FORCE_ENERGY, FORCE_VIRIAL = 1, 2

STATUS = {0: "NBX_OK", 1: "NBX_EINVAL", 2: "NBX_ECUDA", 3: "NBX_ENOMEM", 4: "NBX_ELIST_OVERFLOW",
          5: "NBX_ENCCL"}


class NbxError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


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


class DDGeom(C.Structure):
    """nbx_dd_geom (include/nbx.h): the device-side repartition's domain geometry."""
    _fields_ = [("box", C.c_float * 3), ("dlen", C.c_float * 3), ("lo", C.c_float * 3), ("hi", C.c_float * 3),
                ("rl", C.c_float), ("dims", C.c_int32 * 3), ("coord", C.c_int32 * 3), ("n_src", C.c_int32),
                ("src_rank", C.c_int32 * 27), ("n_off", C.c_int32), ("off_rank", C.c_int32 * 13),
                ("off_dir", (C.c_int32 * 3) * 13), ("off_shift", (C.c_float * 3) * 13)]


class GridInfo(C.Structure):
    _fields_ = [("n", C.c_int32), ("nslots", C.c_int32), ("ncx", C.c_int32), ("ncy", C.c_int32)]


SCI_DTYPE = np.dtype([("sci", "<i4"), ("shift", "<i4"), ("cj_start", "<i4"), ("cj_end", "<i4")])
CJ_DTYPE = np.dtype([("cj", "<i4"), ("meta", "<u4")])
POOL_DTYPE = np.dtype(("<u4", (8, 2)))

# every symbol include/nbx.h declares (checked by tests/test_capi.py)
EXPORTS = ["nbx_last_error", "nbx_version", "nbx_derive_consts", "nbx_ewald_table", "nbx_create", "nbx_destroy",
           "nbx_set_topology", "nbx_set_box", "nbx_grid_build", "nbx_search", "nbx_grid_search_pair", "nbx_put_x",
           "nbx_prune", "nbx_force", "nbx_get_f", "nbx_step_graph", "nbx_energies", "nbx_clear_energies",
           "nbx_grid_info_get", "nbx_grid_export", "nbx_list_sizes_get", "nbx_list_export",
           "nbx_count_pairs", "nbx_fma_peak", "nbx_launch_count", "nbx_alloc_count", "nbx_halo_pack_x", "nbx_halo_unpack_add_f",
           "nbx_peer_init", "nbx_peer_open", "nbx_peer_set_halo", "nbx_peer_put_x", "nbx_peer_halo_x",
           "nbx_peer_force_nonlocal", "nbx_peer_get_f", "nbx_peer_status", "nbx_peer_repartition",
           "nbx_pme_create", "nbx_pme_destroy", "nbx_pme_set_box", "nbx_pme_compute", "nbx_pme_energy",
           "nbx_pme_launch_count", "nbx_pme_profile", "nbx_pme_compute_grid", "nbx_leapfrog",
           "nbx_step_graph_pme"]

_lib = None


def lib():
    """Load libnbx.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2405_01420_b200.build` "
                              "(the product path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i32, u32 = C.c_void_p, C.c_int32, C.c_uint32
        L.nbx_last_error.restype = C.c_char_p
        L.nbx_version.restype = C.c_char_p
        L.nbx_derive_consts.argtypes = [C.POINTER(Params), C.POINTER(Consts)]
        L.nbx_ewald_table.argtypes = [C.POINTER(Consts), vp, vp]
        L.nbx_create.argtypes = [C.c_int, C.POINTER(Params), C.POINTER(vp)]
        L.nbx_destroy.argtypes = [vp]
        L.nbx_set_topology.argtypes = [vp, i32, vp, vp, i32, vp, vp, vp]
        L.nbx_set_box.argtypes = [vp, vp, vp]
        L.nbx_grid_build.argtypes = [vp, C.c_int, i32, vp, vp, vp, vp, vp]
        L.nbx_search.argtypes = [vp, C.c_int, vp]
        L.nbx_grid_search_pair.argtypes = [vp, i32, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp]
        L.nbx_put_x.argtypes = [vp, C.c_int, vp, vp]
        L.nbx_prune.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp]
        L.nbx_force.argtypes = [vp, C.c_int, u32, vp]
        L.nbx_get_f.argtypes = [vp, C.c_int, vp, C.c_int, vp]
        L.nbx_step_graph.argtypes = [vp, vp, vp, u32, vp]
        L.nbx_energies.argtypes = [vp, vp, vp, vp]
        L.nbx_clear_energies.argtypes = [vp, vp]
        L.nbx_grid_info_get.argtypes = [vp, C.c_int, C.POINTER(GridInfo)]
        L.nbx_grid_export.argtypes = [vp, C.c_int, vp, vp, vp]
        L.nbx_list_sizes_get.argtypes = [vp, C.c_int, C.POINTER(ListSizes)]
        L.nbx_list_export.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp]
        L.nbx_count_pairs.argtypes = [vp, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64), vp]
        L.nbx_fma_peak.argtypes = [vp, C.POINTER(C.c_double), vp]
        L.nbx_launch_count.argtypes = [vp]
        L.nbx_launch_count.restype = C.c_int64
        L.nbx_alloc_count.argtypes = []
        L.nbx_alloc_count.restype = C.c_int64
        L.nbx_halo_pack_x.argtypes = [vp, vp, i32, vp, vp, vp]
        L.nbx_halo_unpack_add_f.argtypes = [vp, vp, i32, vp, vp]
        L.nbx_peer_init.argtypes = [vp, i32, i32, i32, vp]
        L.nbx_peer_open.argtypes = [vp, vp]
        L.nbx_peer_set_halo.argtypes = [vp, i32, vp, vp, vp, vp]
        L.nbx_peer_put_x.argtypes = [vp, vp, u32, vp]
        L.nbx_peer_halo_x.argtypes = [vp, u32, vp]
        L.nbx_peer_force_nonlocal.argtypes = [vp, u32, u32, vp]
        L.nbx_peer_get_f.argtypes = [vp, vp, u32, u32, vp]
        L.nbx_peer_status.argtypes = [vp, vp]
        L.nbx_peer_repartition.argtypes = [vp, C.POINTER(DDGeom), vp, vp, i32, u32, i32, vp, vp, vp, vp, vp,
                                           C.POINTER(i32), C.POINTER(i32), vp]
        L.nbx_pme_create.argtypes = [C.c_int, vp, C.POINTER(vp)]
        L.nbx_pme_destroy.argtypes = [vp]
        L.nbx_pme_set_box.argtypes = [vp, vp]
        L.nbx_pme_compute.argtypes = [vp, i32, vp, vp, vp, u32, vp]
        L.nbx_pme_energy.argtypes = [vp, vp, vp, vp]
        L.nbx_pme_launch_count.argtypes = [vp]
        L.nbx_pme_launch_count.restype = C.c_int64
        L.nbx_pme_profile.argtypes = [vp, i32, vp, vp, vp, vp, vp]
        L.nbx_pme_compute_grid.argtypes = [vp, vp, C.c_int, u32, vp]
        L.nbx_step_graph_pme.argtypes = [vp, vp, vp, vp, vp, vp, C.c_float, u32, vp]
        L.nbx_leapfrog.argtypes = [i32, vp, vp, vp, vp, C.c_float, vp]
        _lib = L
    return _lib


def check(code):
    if code != 0:
        raise NbxError(code, lib().nbx_last_error().decode())


LJ_MODIFIERS = {"pot-shift": 0, "force-switch": 1, "comb-geom": 2, "comb-lb": 3}


def make_params(coulomb="ewald", rc=1.0, rlist_outer=1.1, rlist_inner=1.02, epsilon_r=1.0,
                epsilon_rf=0.0, ewald_rtol=1e-5, lj_modifier="pot-shift", rvdw_switch=0.0) -> Params:
    ct = {"rf": NBX_COULOMB_RF, "ewald": NBX_COULOMB_EWALD, "ewald-tab": NBX_COULOMB_EWALD_TAB}[coulomb]
    return Params(ct, rc, rlist_outer, rlist_inner, epsilon_r, epsilon_rf, ewald_rtol,
                  LJ_MODIFIERS[lj_modifier], rvdw_switch)


def derive_consts(params: Params) -> dict:
    c = Consts()
    check(lib().nbx_derive_consts(C.byref(params), C.byref(c)))
    return {n: getattr(c, n) for n, _ in Consts._fields_}


def _np(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _dev_ptr(t):
    return C.c_void_p(t.data_ptr())


def _stream(torch, stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


class Context:
    """Thin owner of an nbx_ctx (one device)."""

    def __init__(self, params: Params, device: int = 0):
        self.params = params
        self.device = device
        h = C.c_void_p()
        check(lib().nbx_create(device, C.byref(params), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().nbx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Nonbonded:
    """Single-domain NBNXM nonbonded engine on one B200.

    `system` is a paper_2405_01420_b200.systems.System (or any object with the same fields).
    Coordinates/forces are torch float32 CUDA tensors [N,3] in the caller's atom order.
    """

    def __init__(self, system, device: int = 0):
        import torch

        self.torch = torch
        self.sys = system
        self.device = device
        self.params = make_params(**system.params())
        self.consts = derive_consts(self.params)
        self.ctx = Context(self.params, device)
        self.n = system.natoms
        self.nstlist = system.nstlist
        self.prune_every = system.prune_every
        q, t = _np(system.q, np.float32), _np(system.type, np.int32)
        c6c12 = _np(system.c6c12, np.float32)
        eo, eg = _np(system.excl_offsets, np.int32), _np(system.excl_gids, np.int32)
        check(lib().nbx_set_topology(self.ctx.h, self.n, _ptr(q), _ptr(t), int(c6c12.shape[0]),
                                     _ptr(c6c12), _ptr(eo), _ptr(eg)))
        self.box = _np(system.box, np.float32)
        self.pbc = np.ones(3, np.int32)
        check(lib().nbx_set_box(self.ctx.h, _ptr(self.box), _ptr(self.pbc)))
        self._lo = np.zeros(3, np.float32)

    # -- the four simulated kernels, for real ----------------------------------------------
    def search(self, x, stream=None):
        """Grid + pair search at rlist_outer + prune to rlist_inner (KernelKind.PAIR_SEARCH)."""
        torch = self.torch
        x = x.contiguous()
        st = _stream(torch, stream)
        check(lib().nbx_grid_build(self.ctx.h, 0, self.n, _dev_ptr(x), None, _ptr(self._lo),
                                   _ptr(self.box), st))
        check(lib().nbx_search(self.ctx.h, LIST_LOCAL, st))

    def put_x(self, x, stream=None):
        check(lib().nbx_put_x(self.ctx.h, 0, _dev_ptr(x), _stream(self.torch, stream)))

    def prune(self, part=0, nparts=1, stream=None):
        """Rolling dynamic prune of the outer list (KernelKind.PRUNE_ONLY)."""
        check(lib().nbx_prune(self.ctx.h, LIST_LOCAL, part, nparts, _stream(self.torch, stream)))

    def compute(self, energy=False, virial=False, stream=None):
        """Force kernel on the inner list (KernelKind.NBNXM_LOCAL)."""
        flags = (FORCE_ENERGY if energy else 0) | (FORCE_VIRIAL if virial else 0)
        if flags:
            check(lib().nbx_clear_energies(self.ctx.h, _stream(self.torch, stream)))
        check(lib().nbx_force(self.ctx.h, LIST_LOCAL, flags, _stream(self.torch, stream)))

    def get_f(self, f, accumulate=False, stream=None):
        """F buffer op (KernelKind.REDUCE_FORCES)."""
        check(lib().nbx_get_f(self.ctx.h, 0, _dev_ptr(f), 1 if accumulate else 0,
                              _stream(self.torch, stream)))

    def energies(self, stream=None):
        e = np.zeros(2, np.float64)
        v = np.zeros(9, np.float64)
        check(lib().nbx_energies(self.ctx.h, _ptr(e), _ptr(v), _stream(self.torch, stream)))
        return e, v.reshape(3, 3)

    # -- convenience ---------------------------------------------------------------------
    def forces(self, x, energy=False, virial=False, out=None, stream=None):
        """x -> forces (and energies/virial) with the current inner list."""
        torch = self.torch
        self.put_x(x, stream)
        self.compute(energy=energy, virial=virial, stream=stream)
        res = None
        if energy or virial:
            res = self.energies(stream)
        if out is None:
            out = torch.empty((self.n, 3), dtype=torch.float32, device=x.device)
        self.get_f(out, stream=stream)
        return (out, res) if res is not None else out

    def graph_step(self, x, f, prune=False, stream=None):
        """X op (+ prune) + force + F op of a non-search step as one CUDA-graph launch.

        The graph is captured natively in libnbx.so (nbx_step_graph) per (x, f, prune) and
        refreshed in place after every search, so launch overhead is paid once per step
        (matters for the small boxes, ~4 launches per step) and no capture ever runs on the
        caller's stream."""
        check(lib().nbx_step_graph(self.ctx.h, _dev_ptr(x), _dev_ptr(f), 1 if prune else 0,
                                   _stream(self.torch, stream)))

    def step(self, x, f, step, energy=False, virial=False, stream=None, graphs=False, pme=None):
        """One NB-path MD step with the reference cadence (pipeline.py:222-235).
        graphs=True replays non-search, non-energy steps as a captured CUDA graph.
        pme (paper_2405_01420_b200.pme.Pme): add the reciprocal-space forces on the grid's
        cluster-ordered atoms before the F buffer op (f = nonbonded + PME)."""
        search = step % self.nstlist == 0
        prune = (not search) and self.prune_every and step % self.prune_every == 0
        if graphs and pme is None and not search and not (energy or virial):
            self.graph_step(x, f, prune=bool(prune), stream=stream)
            return None
        if search:
            self.search(x, stream)  # builds the cluster xyzq buffer from x as well
        else:
            self.put_x(x, stream)
            if prune:
                self.prune(stream=stream)
        self.compute(energy=energy, virial=virial, stream=stream)
        res = self.energies(stream) if (energy or virial) else None
        if pme is not None:
            pme.compute_grid(self, energy=energy, virial=virial, stream=stream)
        self.get_f(f, stream=stream)
        return res

    def md_step(self, x, f, v, inv_mass, dt, step, pme, energy=False, virial=False, stream=None, graphs=True):
        """One GPU-resident MD step of a PME system: step() with pme (NB cadence + PME on the
        grid's cluster order) followed by the leap-frog update of x and v in place
        (pipeline.py:222-257, KernelKind.LEAP_FROG).  graphs=True replays non-search,
        non-energy steps as ONE captured graph (nbx_step_graph_pme: X op, prune, force, PME
        memset/spread/R2C/solve/C2R/gather, F op, update) -- launch overhead is what bounds
        the small boxes."""
        search = step % self.nstlist == 0
        prune = (not search) and self.prune_every and step % self.prune_every == 0
        if graphs and not search and not (energy or virial):
            check(lib().nbx_step_graph_pme(self.ctx.h, pme.h, _dev_ptr(x), _dev_ptr(f), _dev_ptr(v),
                                           _dev_ptr(inv_mass), C.c_float(dt), 1 if prune else 0,
                                           _stream(self.torch, stream)))
            return None
        res = self.step(x, f, step, energy=energy, virial=virial, stream=stream, pme=pme)
        st = _stream(self.torch, stream)
        check(lib().nbx_leapfrog(int(x.shape[0]), _dev_ptr(x), _dev_ptr(v), _dev_ptr(f), _dev_ptr(inv_mass),
                                 C.c_float(dt), st))
        return res

    # -- introspection -------------------------------------------------------------------
    def grid_info(self):
        gi = GridInfo()
        check(lib().nbx_grid_info_get(self.ctx.h, 0, C.byref(gi)))
        return dict(n=gi.n, nslots=gi.nslots, ncx=gi.ncx, ncy=gi.ncy)

    def grid_export(self):
        ns = self.grid_info()["nslots"]
        order = np.empty(ns, np.int32)
        xq = np.empty((ns, 4), np.float32)
        typ = np.empty(ns, np.int32)
        check(lib().nbx_grid_export(self.ctx.h, 0, _ptr(order), _ptr(xq), _ptr(typ)))
        return dict(order=order, xq=xq, type=typ)

    def list_sizes(self, which_list=LIST_LOCAL):
        s = ListSizes()
        check(lib().nbx_list_sizes_get(self.ctx.h, which_list, C.byref(s)))
        return dict(n_sci=s.n_sci, n_cj_outer=s.n_cj_outer, n_cj_inner=s.n_cj_inner, n_pool=s.n_pool)

    def pairlist(self, which=1, which_list=LIST_LOCAL):
        """Canonical list arrays (which=0 outer, 1 inner) for bit-exact comparison."""
        s = self.list_sizes(which_list)
        sci = np.empty(s["n_sci"], SCI_DTYPE)
        cj = np.empty(s["n_cj_outer"] if which == 0 else s["n_cj_inner"], CJ_DTYPE)
        pool = np.empty(s["n_pool"], POOL_DTYPE)
        check(lib().nbx_list_export(self.ctx.h, which_list, which, _ptr(sci), _ptr(cj), _ptr(pool)))
        return dict(sci=sci, cj=cj, pool=pool)

    def count_pairs(self, which_list=LIST_LOCAL, stream=None):
        """(interacting pairs inside rc, computed pair slots) of the inner list."""
        p, s = C.c_int64(), C.c_int64()
        check(lib().nbx_count_pairs(self.ctx.h, which_list, C.byref(p), C.byref(s),
                                    _stream(self.torch, stream)))
        return p.value, s.value

    def fma_peak_tflops(self):
        v = C.c_double()
        check(lib().nbx_fma_peak(self.ctx.h, C.byref(v), _stream(self.torch, None)))
        return v.value

    def launch_count(self):
        return lib().nbx_launch_count(self.ctx.h)

    @staticmethod
    def alloc_count():
        """Device allocations made by libnbx so far (process-wide; none in steady state)."""
        return lib().nbx_alloc_count()

    def close(self):
        self.ctx.close()
