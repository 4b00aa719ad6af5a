"""Row f4: smooth particle-mesh Ewald and the leap-frog update on the
GPU, through the C-ABI of libnbx.so (include/nbx.h, nbx_pme_* / nbx_leapfrog).

The reciprocal-space half of the Ewald electrostatics whose real-space half is the EWALD /
EWALD_TAB nonbonded kernel: the reference's PME_SPREAD -> FFT_3D_FORWARD -> PME_SOLVE ->
FFT_3D_INVERSE -> PME_GATHER kernels (pipeline.py:241-246, costs.py:33-37), GRID_MEMSET
(pipeline.py:256-257) and LEAP_FROG (pipeline.py:249-251).  Conventions: oracle/pme.py.

    pme = Pme.for_system(system)                  # beta of the system's Ewald real space
    f = pme.compute(x, q)                         # torch CUDA tensors, f [N,3] (new)
    pme.compute(x, q, out=f)                      # accumulate into f
    f, (e, vir) = pme.compute(x, q, energy=True)  # reciprocal energy + virial (3x3)
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import nbx

FOURIER_SPACING = 0.12  # nm (GROMACS default fourierspacing)


class PmeParams(C.Structure):
    _fields_ = [("nk", C.c_int32 * 3), ("order", C.c_int32), ("beta", C.c_float), ("epsfac", C.c_float)]


def nice_fft_size(n: int) -> int:
    """Smallest even size >= n whose prime factors are 2, 3, 5 and 7 (cuFFT-friendly)."""
    m = max(int(n), 1)
    while True:
        r = m
        for p in (2, 3, 5, 7):
            while r % p == 0:
                r //= p
        if r == 1 and m % 2 == 0:
            return m
        m += 1


def grid_dims(box, spacing=FOURIER_SPACING, order=4):
    return tuple(max(nice_fft_size(math.ceil(float(L) / spacing)), 2 * order) for L in box)


class Pme:
    def __init__(self, box, beta, epsfac=138.935458, nk=None, order=4, device=0):
        self.box = np.asarray(box, dtype=np.float32)
        self.nk = tuple(int(k) for k in (nk if nk is not None else grid_dims(self.box, order=order)))
        self.device = device
        p = PmeParams((C.c_int32 * 3)(*self.nk), order, float(beta), float(epsfac))
        h = C.c_void_p()
        nbx.check(nbx.lib().nbx_pme_create(device, C.byref(p), C.byref(h)))
        self.h = h
        nbx.check(nbx.lib().nbx_pme_set_box(self.h, self.box.ctypes.data_as(C.c_void_p)))

    @classmethod
    def for_system(cls, system, device=0, **kw):
        c = nbx.derive_consts(nbx.make_params(**system.params()))
        if not c["beta"] > 0.0:
            raise ValueError(f"{system.name}: PME needs Ewald electrostatics (coulomb={system.coulomb!r})")
        return cls(system.box, c["beta"], c["epsfac"], device=device, **kw)

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            nbx.lib().nbx_pme_destroy(h)
            self.h = None

    def set_box(self, box):
        self.box = np.asarray(box, dtype=np.float32)
        nbx.check(nbx.lib().nbx_pme_set_box(self.h, self.box.ctypes.data_as(C.c_void_p)))

    def compute(self, x, q, out=None, energy=False, virial=False, stream=None):
        import torch
        assert x.is_cuda and x.dtype == torch.float32 and x.is_contiguous() and x.shape[1] == 3
        assert q.is_cuda and q.dtype == torch.float32 and q.is_contiguous()
        f = torch.zeros_like(x) if out is None else out
        st = torch.cuda.current_stream().cuda_stream if stream is None else stream
        flags = (1 if energy else 0) | (2 if virial else 0)
        nbx.check(nbx.lib().nbx_pme_compute(self.h, int(x.shape[0]), C.c_void_p(x.data_ptr()),
                                            C.c_void_p(q.data_ptr()), C.c_void_p(f.data_ptr()), flags,
                                            C.c_void_p(st)))
        if not (energy or virial):
            return f
        e = np.zeros(1)
        v = np.zeros(9)
        nbx.check(nbx.lib().nbx_pme_energy(self.h, e.ctypes.data_as(C.c_void_p), v.ctypes.data_as(C.c_void_p),
                                           C.c_void_p(st)))
        return f, (float(e[0]), v.reshape(3, 3))

    def compute_grid(self, nb, energy=False, virial=False, grid=0, stream=None):
        """Reciprocal-space forces on the atoms of Nonbonded `nb`'s grid (cluster order, after
        its X op of this step), added to its cluster force buffer: nb.get_f() then returns
        nonbonded + PME forces.  Energy / virial accumulate here (read with energy())."""
        import torch
        st = torch.cuda.current_stream().cuda_stream if stream is None else stream
        flags = (1 if energy else 0) | (2 if virial else 0)
        nbx.check(nbx.lib().nbx_pme_compute_grid(self.h, nb.ctx.h, grid, flags, C.c_void_p(st)))

    def energy(self, stream=None):
        import torch
        st = torch.cuda.current_stream().cuda_stream if stream is None else stream
        e = np.zeros(1)
        v = np.zeros(9)
        nbx.check(nbx.lib().nbx_pme_energy(self.h, e.ctypes.data_as(C.c_void_p), v.ctypes.data_as(C.c_void_p),
                                           C.c_void_p(st)))
        return float(e[0]), v.reshape(3, 3)

    STAGES = ("grid_memset", "pme_spread", "fft_3d_forward", "pme_solve", "fft_3d_inverse", "pme_gather")

    def profile(self, x, q, out=None):
        """Per-stage milliseconds of one force-only evaluation (reference KernelKind names)."""
        import torch
        f = torch.zeros_like(x) if out is None else out
        ms = np.zeros(6, dtype=np.float32)
        nbx.check(nbx.lib().nbx_pme_profile(self.h, int(x.shape[0]), C.c_void_p(x.data_ptr()),
                                            C.c_void_p(q.data_ptr()), C.c_void_p(f.data_ptr()),
                                            ms.ctypes.data_as(C.c_void_p),
                                            C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return dict(zip(self.STAGES, (float(v) for v in ms)))

    def launch_count(self):
        return int(nbx.lib().nbx_pme_launch_count(self.h))


def leapfrog(x, v, f, inv_mass, dt, stream=None):
    """v += f inv_mass dt; x += v dt in place (torch CUDA float32 tensors)."""
    import torch
    st = torch.cuda.current_stream().cuda_stream if stream is None else stream
    nbx.check(nbx.lib().nbx_leapfrog(int(x.shape[0]), C.c_void_p(x.data_ptr()), C.c_void_p(v.data_ptr()),
                                     C.c_void_p(f.data_ptr()), C.c_void_p(inv_mass.data_ptr()), float(dt),
                                     C.c_void_p(st)))
