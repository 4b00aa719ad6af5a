"""Shared comparison helpers and tolerances (north_star: forces rel RMS <= 1e-5, max <= 1e-4;
energies and virial relative error <= 1e-6; pair lists and masks bit-exact)."""
import numpy as np

FORCE_RMS_TOL = 1e-5
FORCE_MAX_TOL = 1e-4  # max_a |df_a| / rms_a |f_a|
ENERGY_TOL = 1e-6
VIRIAL_TOL = 1e-6  # max |dXi| / max |Xi|


def force_errors(f, fref):
    f = np.asarray(f, np.float64)
    fref = np.asarray(fref, np.float64)
    d = f - fref
    if not np.any(fref):
        return float(np.abs(d).max(initial=0.0)), float(np.abs(d).max(initial=0.0))
    rms_ref = np.sqrt((fref**2).sum(axis=1).mean())
    rel_rms = np.sqrt((d**2).sum() / (fref**2).sum())
    rel_max = np.sqrt((d**2).sum(axis=1)).max() / rms_ref
    return rel_rms, rel_max


def assert_forces(f, fref, rms_tol=FORCE_RMS_TOL, max_tol=FORCE_MAX_TOL):
    rel_rms, rel_max = force_errors(f, fref)
    assert rel_rms <= rms_tol, f"force rel RMS {rel_rms:.3e} > {rms_tol}"
    assert rel_max <= max_tol, f"force rel max {rel_max:.3e} > {max_tol}"
    return rel_rms, rel_max


def assert_energies(e, eref, tol=ENERGY_TOL):
    e = np.asarray(e, np.float64)
    eref = np.asarray(eref, np.float64)
    rel = np.abs(e - eref) / np.maximum(np.abs(eref), 1e-300)
    assert np.all(rel <= tol), f"energy rel err {rel} > {tol} (got {e}, ref {eref})"
    return rel


def assert_virial(v, vref, tol=VIRIAL_TOL):
    v = np.asarray(v, np.float64)
    vref = np.asarray(vref, np.float64)
    rel = np.abs(v - vref).max() / np.abs(vref).max()
    assert rel <= tol, f"virial rel err {rel:.3e} > {tol}"
    return rel


def assert_lists_equal(a, b, what=""):
    for k in ("sci", "cj", "pool"):
        assert a[k].shape == b[k].shape, f"{what} {k} shape {a[k].shape} != {b[k].shape}"
        if not np.array_equal(a[k], b[k]):
            bad = np.nonzero(a[k].reshape(len(a[k]), -1).view(np.uint8).reshape(len(a[k]), -1)
                             != b[k].reshape(len(b[k]), -1).view(np.uint8).reshape(len(b[k]), -1))[0]
            raise AssertionError(f"{what} {k} differs at {len(np.unique(bad))} entries, first {bad[:5]}: "
                                 f"{a[k][bad[:3]]} vs {b[k][bad[:3]]}")


def flatten_pairs(lst):
    """(ci, cj, shift, int_mask, corr_mask) per active tile -- the human-readable canonical form."""
    sci, cj, pool = lst["sci"], lst["cj"], lst["pool"]
    rows = []
    for e in sci:
        for q in range(e["cj_start"], e["cj_end"]):
            meta = int(cj[q]["meta"])
            im, p = meta & 0xFF, meta >> 8
            for k in range(8):
                if im >> k & 1:
                    m = pool[p][k] if p else (0xFFFFFFFF, 0)
                    rows.append((8 * int(e["sci"]) + k, int(cj[q]["cj"]), int(e["shift"]), int(m[0]), int(m[1])))
    return np.array(rows, dtype=np.int64).reshape(-1, 5)
