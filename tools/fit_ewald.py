"""Fit the fp32 rational approximations used for Ewald real-space electrostatics.

G(z) = erf(sqrt z)/z^1.5 - (2/sqrt(pi)) exp(-z)/z   (force:  F/r = -beta^3 G(beta^2 r^2) for -erf(beta r)/r)
H(z) = erf(sqrt z)/sqrt z                            (energy: -erf(beta r)/r = -beta H(beta^2 r^2))

Both are entire functions of z.  We fit p(z)/q(z) (q(0)=1) by iteratively re-weighted linear
least squares on the relative error over z in [0, ZMAX] and print fp32 coefficients for
paper_2405_01420_b200/csrc/pairmath.h.  The same coefficients are used by the CPU oracle
(oracle/nbx_oracle.c), so parity does not depend on this fit's accuracy; DESIGN.md states
the accuracy against the exact functions.
"""
import numpy as np
from math import erf, sqrt, pi, exp

ZMAX = 12.5  # beta*rc up to 3.54 (ewald_rtol down to ~3e-7)


def G_exact(z):
    z = np.asarray(z, dtype=np.float64)
    out = np.empty_like(z)
    small = z < 1e-3
    zs = z[small]
    # series: 2/sqrt(pi) * (2/3 - 2/5 z + 1/7 z^2 - 1/27 z^3 ...)  (from erf/exp series)
    c = 2 / sqrt(pi)
    out[small] = c * (2 / 3 - 2 / 5 * zs + 1 / 7 * zs**2 - 1 / 27 * zs**3)
    zl = z[~small]
    out[~small] = np.array([erf(sqrt(v)) for v in zl]) / zl**1.5 - c * np.exp(-zl) / zl
    return out


def H_exact(z):
    z = np.asarray(z, dtype=np.float64)
    out = np.empty_like(z)
    small = z < 1e-6
    out[small] = 2 / sqrt(pi) * (1 - z[small] / 3)
    zl = z[~small]
    out[~small] = np.array([erf(sqrt(v)) for v in zl]) / np.sqrt(zl)
    return out


def fit_rational(f, n, m, zmax=ZMAX, iters=30):
    z = 0.5 * zmax * (1 - np.cos(np.linspace(0, pi, 4000)))
    y = f(z)
    w = 1 / np.abs(y)
    qz = np.ones_like(z)
    for _ in range(iters):
        # p(z) - y*(q(z)-1) = y ; unknowns p0..pn, q1..qm ; weight by 1/(|y| q_prev)
        A = np.hstack([z[:, None] ** np.arange(n + 1), -(y[:, None]) * z[:, None] ** np.arange(1, m + 1)])
        ww = w / np.abs(qz)
        sol, *_ = np.linalg.lstsq(A * ww[:, None], y * ww, rcond=None)
        p = sol[: n + 1]
        q = np.concatenate([[1.0], sol[n + 1 :]])
        qz = np.polyval(q[::-1], z)
        err = (np.polyval(p[::-1], z) / qz - y) / y
        w = w * (1 + 50 * np.abs(err) / np.abs(err).max())  # push towards minimax
        w /= w.max()
    return p, q


def eval32(p, q, z):
    """Horner in fp32 with fma, exactly as pairmath.h evaluates it."""
    z = z.astype(np.float32)
    p32 = p.astype(np.float32)
    q32 = q.astype(np.float32)
    num = np.full_like(z, p32[-1])
    for c in p32[-2::-1]:
        num = (num.astype(np.float64) * z + c).astype(np.float32)
    den = np.full_like(z, q32[-1])
    for c in q32[-2::-1]:
        den = (den.astype(np.float64) * z + c).astype(np.float32)
    return (num / den).astype(np.float32)


if __name__ == "__main__":
    zt = np.linspace(0, ZMAX, 200001)
    for name, f, (n, m) in (("G", G_exact, (5, 5)), ("H", H_exact, (6, 5))):
        p, q = fit_rational(f, n, m, iters=60)
        ref = f(zt)
        approx = eval32(p, q, zt).astype(np.float64)
        rel = np.abs(approx - ref) / np.abs(ref)
        print(f"{name}: n={n} m={m} max rel err (fp32 eval) = {rel.max():.3e}  rms = {np.sqrt((rel**2).mean()):.3e}")
        print("  P =", ", ".join(f"{np.float32(c)!r}" for c in p))
        print("  Q =", ", ".join(f"{np.float32(c)!r}" for c in q))
