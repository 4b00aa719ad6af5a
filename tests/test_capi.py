"""CPU checks of the C-ABI boundary: libnbx.so loads, exports every symbol include/nbx.h
declares, derives constants identically to the oracle, and fails loudly without a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_2405_01420_b200 import nbx

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "nbx.h")).read()
    return sorted(set(re.findall(r"NBX_API\s+[\w\s\*]+?\b(nbx_\w+)\s*\(", txt)))


def test_header_symbols_listed():
    assert header_symbols() == sorted(nbx.EXPORTS)


def test_library_exports_every_symbol():
    lib = C.CDLL(nbx.LIB_PATH)
    for s in header_symbols():
        assert hasattr(lib, s), f"{s} not exported by libnbx.so"


def test_exports_are_only_the_abi():
    out = os.popen(f"nm -D --defined-only {nbx.LIB_PATH}").read().split("\n")
    syms = {l.split()[-1] for l in out if " T " in l}
    assert {s for s in syms if s.startswith("nbx_")} == set(header_symbols())


@pytest.mark.parametrize("kw", [dict(coulomb="rf", rc=0.9, rlist_outer=1.0, rlist_inner=0.92),
                                dict(coulomb="ewald", rc=1.0, rlist_outer=1.1, rlist_inner=1.02),
                                dict(coulomb="ewald", rc=1.2, rlist_outer=1.3, rlist_inner=1.22, ewald_rtol=1e-6),
                                dict(coulomb="rf", rc=1.0, rlist_outer=1.2, rlist_inner=1.05, epsilon_r=2.0, epsilon_rf=78.0),
                                dict(coulomb="ewald-tab", rc=1.2, rlist_outer=1.3, rlist_inner=1.22,
                                     lj_modifier="force-switch", rvdw_switch=1.0),
                                dict(coulomb="ewald-tab", rc=0.9, rlist_outer=1.0, rlist_inner=0.92, ewald_rtol=1e-3)])
def test_derived_constants_bit_identical(kw):
    a = nbx.derive_consts(nbx.make_params(**kw))
    b = O.derive_consts(O.make_params(**kw))
    for k in a:
        assert np.float32(a[k]).tobytes() == np.float32(b[k]).tobytes(), k


@pytest.mark.parametrize("rc, rtol", [(1.2, 1e-5), (1.0, 1e-5), (0.9, 1e-3)])
def test_ewald_tables_bit_identical(rc, rtol):
    """EWALD_TAB tables: library (host side, no GPU needed) == oracle, and accurate."""
    import ctypes as C
    from scipy.special import erf
    kw = dict(coulomb="ewald-tab", rc=rc, rlist_outer=rc + 0.1, rlist_inner=rc + 0.02, ewald_rtol=rtol)
    c = nbx.Consts()
    nbx.check(nbx.lib().nbx_derive_consts(C.byref(nbx.make_params(**kw)), C.byref(c)))
    assert c.tab_scale >= 600.0 and c.tab_n == int(np.ceil(rc * np.float64(c.tab_scale))) + 2
    ft = np.zeros((c.tab_n, 2), np.float32)
    vt = np.zeros((c.tab_n, 2), np.float32)
    nbx.check(nbx.lib().nbx_ewald_table(C.byref(c), nbx._ptr(ft), nbx._ptr(vt)))
    fo, vo = O.ewald_table(O.make_params(**kw))
    assert ft.tobytes() == fo.tobytes() and vt.tobytes() == vo.tobytes()
    # interpolation error at mid-points against the exact correction terms
    b = np.float64(c.beta)
    r = (np.arange(1, c.tab_n - 2) + 0.5) / np.float64(c.tab_scale)
    fex = (erf(b * r) / r - 2 * b / np.sqrt(np.pi) * np.exp(-b * b * r * r)) / (r * r)
    vex = erf(b * r) / r
    k = np.arange(1, c.tab_n - 2)
    fin = ft[k, 0] + 0.5 * ft[k, 1]
    vin = vt[k, 0] + 0.5 * vt[k, 1]
    assert np.abs(fin - fex).max() / fex.max() < 2e-6
    assert np.abs(vin - vex).max() / vex.max() < 2e-6


def test_invalid_params_rejected():
    with pytest.raises(nbx.NbxError) as ei:
        nbx.derive_consts(nbx.make_params(rc=1.0, rlist_outer=1.1, rlist_inner=0.9))
    assert ei.value.code == 1


def test_no_cpu_fallback():
    """Without a usable sm_100 GPU, context creation fails with NBX_ECUDA -- never a CPU path."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(nbx.NbxError) as ei:
        nbx.Context(nbx.make_params())
    assert ei.value.code == 2
    assert "no CPU fallback" in str(ei.value)


def test_halo_entry_points_validate_arguments():
    lib = nbx.lib()
    assert lib.nbx_halo_pack_x(None, None, -1, None, None, None) == 1
    assert lib.nbx_halo_unpack_add_f(None, None, 5, None, None) == 1
    assert lib.nbx_halo_pack_x(None, None, 0, None, None, None) == 0
    # the overlapped DD search step rejects a missing context before touching any stream
    assert lib.nbx_grid_search_pair(None, 0, None, None, None, None, 0, None, None, None, None, None, None) != 0


def test_pme_no_cpu_fallback_and_validation():
    """Row f4 entry points: parameter validation happens before device checks, and without a
    usable sm_100 GPU a PME context fails with NBX_ECUDA; the leap-frog validates arguments."""
    import torch

    from paper_2405_01420_b200 import pme
    with pytest.raises(nbx.NbxError) as ei:
        pme.Pme([3.0, 3.0, 3.0], 3.0, nk=(25, 24, 24))
    assert ei.value.code == 1
    with pytest.raises(nbx.NbxError):
        pme.Pme([3.0, 3.0, 3.0], 3.0, order=6)
    if not torch.cuda.is_available():
        with pytest.raises(nbx.NbxError) as ei:
            pme.Pme([3.0, 3.0, 3.0], 3.0)
        assert ei.value.code == 2 and "no CPU fallback" in str(ei.value)
    lib = nbx.lib()
    assert lib.nbx_leapfrog(-1, None, None, None, None, 0.0, None) == 1
    assert lib.nbx_leapfrog(0, None, None, None, None, 0.0, None) == 0
    assert lib.nbx_pme_compute(None, 0, None, None, None, 0, None) == 1
