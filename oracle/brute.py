"""float64 all-pairs brute force with exact erfc/erf.  TEST INFRASTRUCTURE ONLY.

Independent of the cluster machinery: minimum image (box >= 2 rc), every unordered pair once,
exclusions from the CSR topology.  Used to pin the C oracle's physics
to the exact functions, and for two-particle known answers.
"""
from __future__ import annotations

import numpy as np
from scipy.special import erf, erfc


def excluded_pairs(excl_offsets, excl_gids):
    n = len(excl_offsets) - 1
    a = np.repeat(np.arange(n), np.diff(excl_offsets))
    b = np.asarray(excl_gids)
    m = a < b
    return set(zip(a[m].tolist(), b[m].tolist()))


def _fsw_terms(r, rc, r1, a):
    """GROMACS force switch for r^-a on [r1, rc): (F_a(r), V_a(r)) incl. the a r^-(a+1) part."""
    d = rc - r1
    A = -a * ((a + 4) * rc - (a + 1) * r1) / (rc ** (a + 2) * d * d)
    B = a * ((a + 3) * rc - (a + 1) * r1) / (rc ** (a + 2) * d ** 3)
    C = rc ** -a - A / 3 * d ** 3 - B / 4 * d ** 4
    t = np.maximum(r - r1, 0.0)
    F = a * r ** (-(a + 1)) + A * t * t + B * t ** 3
    V = r ** -a - A / 3 * t ** 3 - B / 4 * t ** 4 - C
    return F, V


def brute_force(x, q, typ, c6c12, excl_offsets, excl_gids, box, consts, coulomb, rc,
                chunk=2048, lj_modifier="pot-shift", rvdw_switch=0.0):
    """Returns (f[N,3] float64, (E_lj, E_coul incl. self), virial[3,3])."""
    x = np.asarray(x, np.float64)
    q = np.asarray(q, np.float64)
    box = np.asarray(box, np.float64)
    N = x.shape[0]
    epsfac = float(consts["epsfac"])
    krf, crf = float(consts["k_rf"]), float(consts["c_rf"])
    beta = float(consts["beta"])
    c6t = np.asarray(c6c12[..., 0], np.float64)
    c12t = np.asarray(c6c12[..., 1], np.float64)
    exclset = excluded_pairs(excl_offsets, excl_gids)
    f = np.zeros((N, 3))
    elj = ec = 0.0
    vir = np.zeros((3, 3))
    rc2 = rc * rc
    sh6, sh12 = rc**-6, rc**-12
    sh_ew = erfc(beta * rc) / rc
    for a0 in range(0, N, chunk):
        a1 = min(N, a0 + chunk)
        ia = np.arange(a0, a1)
        d = x[ia, None, :] - x[None, :, :]
        d -= box * np.round(d / box)
        r2 = (d * d).sum(-1)
        upper = ia[:, None] < np.arange(N)[None, :]
        m = upper & (r2 < rc2)
        ai, bj = np.nonzero(m)
        ai = ai + a0
        dd = d[ai - a0, bj]
        rr2 = r2[ai - a0, bj]
        r = np.sqrt(rr2)
        ex = np.array([(int(u), int(v)) in exclset for u, v in zip(ai, bj)], dtype=bool) if exclset else np.zeros(len(ai), bool)
        c6 = c6t[typ[ai], typ[bj]]
        c12 = c12t[typ[ai], typ[bj]]
        qq = epsfac * q[ai] * q[bj]
        inv = 1.0 / r
        rinv6 = inv**6
        if lj_modifier == "force-switch":
            F12, V12 = _fsw_terms(r, rc, rvdw_switch, 12.0)
            F6, V6 = _fsw_terms(r, rc, rvdw_switch, 6.0)
            flj = np.where(ex, 0.0, (c12 * F12 - c6 * F6) * inv)  # F/r
            vlj = np.where(ex, 0.0, c12 * V12 - c6 * V6)
        else:
            flj = np.where(ex, 0.0, (12 * c12 * rinv6 * rinv6 - 6 * c6 * rinv6) * inv * inv)  # F/r
            vlj = np.where(ex, 0.0, c12 * (rinv6 * rinv6 - sh12) - c6 * (rinv6 - sh6))
        if coulomb == "rf":
            fc = qq * (np.where(ex, 0.0, inv**3) - 2 * krf)
            vc = qq * (np.where(ex, 0.0, inv) + krf * rr2 - crf)
        else:
            g = 2 * beta / np.sqrt(np.pi) * np.exp(-beta * beta * rr2)
            fc_ne = qq * (erfc(beta * r) * inv + g) * inv * inv
            fc_ex = qq * (-erf(beta * r) * inv + g) * inv * inv
            fc = np.where(ex, fc_ex, fc_ne)
            vc = np.where(ex, -qq * erf(beta * r) * inv, qq * (erfc(beta * r) * inv - sh_ew))
        fs = (flj + fc)[:, None] * dd
        np.add.at(f, ai, fs)
        np.add.at(f, bj, -fs)
        elj += vlj.sum()
        ec += vc.sum()
        vir += -0.5 * np.einsum("pa,pb->ab", dd, fs)
    sumq2 = float((q * q).sum())
    if coulomb == "rf":
        ec += -0.5 * epsfac * crf * sumq2
    else:
        ec += -epsfac * beta / np.sqrt(np.pi) * sumq2
    return f, (elj, ec), vir
