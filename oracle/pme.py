"""CPU oracle (test infrastructure only) for SURVEY.md row f4: smooth particle-mesh Ewald.

The reference models this part of the step as five kernel kinds submitted after the
nonbonded kernels when the system uses PME (pipeline.py:241-246: PME_SPREAD,
FFT_3D_FORWARD, PME_SOLVE, FFT_3D_INVERSE, PME_GATHER; costs.py:33-37), plus GRID_MEMSET
(pipeline.py:256-257) and LEAP_FROG (pipeline.py:249-251).  It computes nothing; this module
restates the algorithm (Essmann et al. 1995, GROMACS conventions) in float64 numpy so that
the sm_100a implementation (paper_2405_01420_b200/csrc/pme.cu) can be checked on identical
inputs.  Only tests/ and bench.py's CPU baseline may import it.

Conventions (identical in pme.cu):
  u_d = K_d frac(x_d / L_d);  w = u - floor(u);  theta_j = M_n(w + j) placed at grid index
  floor(u) - j (mod K), j = 0..n-1;  dtheta_j = M_{n-1}(w + j) - M_{n-1}(w + j - 1).
  Q(k) = sum_i q_i prod_d theta;  S = FFT(Q) (unnormalised, e^{-2 pi i m.k/K}).
  G(m) = exp(-pi^2 |mt|^2 / beta^2) / (pi V |mt|^2) prod_d |b_d(m_d)|^2,  mt_d = m_d / L_d with
  m_d signed in (-K/2, K/2];  |b_d(m)|^-2 = |sum_{k=0}^{n-2} M_n(k+1) e^{2 pi i m k / K}|^2.
  E = epsfac/2 sum_m G |S|^2;  phi = IFFT_unnormalised(G S);
  F_i,a = -epsfac q_i (K_a / L_a) sum_k dtheta_a theta_b theta_c phi(k);
  Xi_ab = -1/2 sum_m E_m (delta_ab - 2 (1 + pi^2 |mt|^2 / beta^2) mt_a mt_b / |mt|^2)
  (the same virial convention as the nonbonded path: Xi = -1/2 sum x (x) f).
"""
from __future__ import annotations

import math

import numpy as np

FOURIER_SPACING = 0.12  # nm, GROMACS default fourierspacing


def nice_fft_size(n: int) -> int:
    """Smallest size >= n whose prime factors are 2, 3, 5, 7 (cuFFT-friendly)."""
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


def bspline_m(x, n):
    """Cardinal B-spline M_n(x) (support (0, n)), vectorised, by the standard recursion."""
    x = np.asarray(x, dtype=np.float64)
    m = np.where((x > 0) & (x < 2), 1.0 - np.abs(x - 1.0), 0.0)  # M_2
    for k in range(3, n + 1):
        m = (x * m + (k - x) * _shift_eval(x - 1.0, k - 1)) / (k - 1)
    return m


def _shift_eval(x, n):
    return bspline_m(x, n) if n > 2 else np.where((x > 0) & (x < 2), 1.0 - np.abs(x - 1.0), 0.0)


def splines(x, box, nk, order=4):
    """theta, dtheta [N, 3, order] and base index floor(u) [N, 3]."""
    x = np.asarray(x, dtype=np.float64)
    box = np.asarray(box, dtype=np.float64)
    nk = np.asarray(nk)
    frac = x / box
    frac = frac - np.floor(frac)
    u = frac * nk
    base = np.floor(u).astype(np.int64)
    base = np.minimum(base, nk - 1)
    w = u - base
    j = np.arange(order)
    arg = w[:, :, None] + j[None, None, :]
    theta = bspline_m(arg, order)
    dtheta = bspline_m(arg, order - 1) - bspline_m(arg - 1.0, order - 1)
    return theta, dtheta, base


def bsp_moduli(K, order=4):
    """|b(m)|^2 for m = 0..K-1."""
    mk = bspline_m(np.arange(1, order, dtype=np.float64), order)  # M_n(1..n-1)
    m = np.arange(K)[:, None]
    k = np.arange(order - 1)[None, :]
    s = (mk[None, :] * np.exp(2j * np.pi * m * k / K)).sum(axis=1)
    return 1.0 / np.abs(s) ** 2


def influence(box, nk, beta, order=4):
    """G(m) on the half spectrum [Kx, Ky, Kz//2+1] and mt components."""
    Kx, Ky, Kz = nk
    L = np.asarray(box, dtype=np.float64)
    V = float(np.prod(L))

    def signed(K, n):
        m = np.arange(n)
        return np.where(m <= K // 2, m, m - K)

    mx = signed(Kx, Kx)[:, None, None] / L[0]
    my = signed(Ky, Ky)[None, :, None] / L[1]
    mz = np.arange(Kz // 2 + 1)[None, None, :] / L[2]
    m2 = mx**2 + my**2 + mz**2
    bx, by, bz = bsp_moduli(Kx, order), bsp_moduli(Ky, order), bsp_moduli(Kz, order)[: Kz // 2 + 1]
    with np.errstate(divide="ignore", invalid="ignore"):
        G = np.exp(-np.pi**2 * m2 / beta**2) / (np.pi * V * m2)
    G = G * bx[:, None, None] * by[None, :, None] * bz[None, None, :]
    G[0, 0, 0] = 0.0
    return G, (mx, my, mz), m2


def pme(x, q, box, beta, epsfac, nk=None, order=4):
    """Reciprocal-space energy, forces [N,3] and virial [3,3] (float64)."""
    x = np.asarray(x, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    nk = tuple(nk) if nk is not None else grid_dims(box, order=order)
    Kx, Ky, Kz = nk
    theta, dtheta, base = splines(x, box, nk, order)
    j = np.arange(order)
    ix = (base[:, 0, None] - j[None, :]) % Kx
    iy = (base[:, 1, None] - j[None, :]) % Ky
    iz = (base[:, 2, None] - j[None, :]) % Kz
    # spread (pme_spread)
    Q = np.zeros(nk)
    w = q[:, None, None, None] * theta[:, 0, :, None, None] * theta[:, 1, None, :, None] * theta[:, 2, None, None, :]
    np.add.at(Q, (ix[:, :, None, None], iy[:, None, :, None], iz[:, None, None, :]), w)
    # forward FFT, solve, inverse FFT
    S = np.fft.rfftn(Q)
    G, (mx, my, mz), m2 = influence(box, nk, beta, order)
    wgt = np.full(Kz // 2 + 1, 2.0)
    wgt[0] = 1.0
    if Kz % 2 == 0:
        wgt[-1] = 1.0
    Em = 0.5 * epsfac * G * np.abs(S) ** 2 * wgt[None, None, :]
    E = float(Em.sum())
    with np.errstate(divide="ignore", invalid="ignore"):
        fac = 2.0 * (1.0 + np.pi**2 * m2 / beta**2) / m2
    fac[0, 0, 0] = 0.0
    comps = [np.broadcast_to(c, m2.shape) for c in (mx, my, mz)]
    vir = np.zeros((3, 3))
    for a in range(3):
        for b in range(3):
            vir[a, b] = -0.5 * float((Em * ((1.0 if a == b else 0.0) - fac * comps[a] * comps[b])).sum())
    phi = np.fft.irfftn(G * S, s=nk, axes=(0, 1, 2)) * (Kx * Ky * Kz)
    # gather (pme_gather)
    P = phi[ix[:, :, None, None], iy[:, None, :, None], iz[:, None, None, :]]  # [N, o, o, o]
    tx, ty, tz = theta[:, 0], theta[:, 1], theta[:, 2]
    dx, dy, dz = dtheta[:, 0], dtheta[:, 1], dtheta[:, 2]
    L = np.asarray(box, dtype=np.float64)
    f = np.empty((len(q), 3))
    f[:, 0] = np.einsum("ni,nj,nk,nijk->n", dx, ty, tz, P) * (Kx / L[0])
    f[:, 1] = np.einsum("ni,nj,nk,nijk->n", tx, dy, tz, P) * (Ky / L[1])
    f[:, 2] = np.einsum("ni,nj,nk,nijk->n", tx, ty, dz, P) * (Kz / L[2])
    f *= -epsfac * q[:, None]
    return E, f, vir


def ewald_recip_direct(x, q, box, beta, epsfac, tol=1e-12):
    """Exact reciprocal-space Ewald sum (float64, explicit k vectors): the physics check."""
    x = np.asarray(x, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    L = np.asarray(box, dtype=np.float64)
    V = float(np.prod(L))
    mmax = beta * math.sqrt(-math.log(tol)) / math.pi
    n = [int(math.ceil(mmax * l)) for l in L]
    E = 0.0
    f = np.zeros_like(x)
    vir = np.zeros((3, 3))
    for a in range(-n[0], n[0] + 1):
        for b in range(-n[1], n[1] + 1):
            cs = []
            for c in range(-n[2], n[2] + 1):
                if a == 0 and b == 0 and c == 0:
                    continue
                cs.append(c)
            if not cs:
                continue
            mt = np.stack([np.full(len(cs), a / L[0]), np.full(len(cs), b / L[1]), np.array(cs) / L[2]], 1)
            m2 = (mt**2).sum(1)
            keep = m2 <= mmax**2
            mt, m2 = mt[keep], m2[keep]
            if len(m2) == 0:
                continue
            ph = 2.0 * np.pi * x @ mt.T  # [N, M]
            Sr = (q[:, None] * np.cos(ph)).sum(0)
            Si = (q[:, None] * np.sin(ph)).sum(0)
            g = np.exp(-np.pi**2 * m2 / beta**2) / (np.pi * V * m2)
            Em = 0.5 * epsfac * g * (Sr**2 + Si**2)
            E += float(Em.sum())
            # F_i = -dE/dx_i = epsfac * sum_m g * 2 pi m q_i (sin(ph_i) Sr - cos(ph_i) Si)
            coef = epsfac * g * 2.0 * np.pi * (np.sin(ph) * Sr[None, :] - np.cos(ph) * Si[None, :])
            f += q[:, None] * (coef @ mt)
            fac = 2.0 * (1.0 + np.pi**2 * m2 / beta**2) / m2
            for i in range(3):
                for j in range(3):
                    vir[i, j] += -0.5 * float((Em * ((1.0 if i == j else 0.0) - fac * mt[:, i] * mt[:, j])).sum())
    return E, f, vir
