"""Exact solutions of the further workloads, used as pins of
the oracle.  Plain textbook gas dynamics, independent of the oracle and the CUDA path.

* exact_riemann: the ideal-gas Riemann problem (two shocks / rarefactions meeting at a
  contact), star pressure by bisection on f_L(p) + f_R(p) + (u_R - u_L) = 0 and the
  self-similar sampling of the wave fan (the standard construction, e.g. Toro,
  "Riemann Solvers and Numerical Methods for Fluid Dynamics", ch. 4).  g may be a
  pair (gamma_L, gamma_R): two ideal gases meeting at the contact (each wave
  function f_K and each side's fan only involve that side's gamma).
* noh_planar: the planar Noh solution -- a strong shock reflecting off the wall at
  speed D = (gamma-1)/2 |u0|, gas at rest behind it with rho = rho0 (gamma+1)/(gamma-1),
  p = rho0 |u0| (D + |u0|) ... i.e. all kinetic energy turned into internal energy.
"""
from __future__ import annotations

import math

import numpy as np


def _f(p, r, pk, ck, g):
    if p > pk:  # shock
        A, B = 2.0 / ((g + 1.0) * r), (g - 1.0) / (g + 1.0) * pk
        return (p - pk) * math.sqrt(A / (p + B))
    return 2.0 * ck / (g - 1.0) * ((p / pk) ** ((g - 1.0) / (2.0 * g)) - 1.0)  # rarefaction


def _gammas(g):
    return (float(g[0]), float(g[1])) if isinstance(g, (tuple, list)) else (float(g), float(g))


def star_state(WL, WR, g):
    rL, uL, pL = WL
    rR, uR, pR = WR
    gL, gR = _gammas(g)
    cL, cR = math.sqrt(gL * pL / rL), math.sqrt(gR * pR / rR)
    lo, hi = 1e-12, 1e3 * max(pL, pR)
    for _ in range(200):
        pm = 0.5 * (lo + hi)
        if _f(pm, rL, pL, cL, gL) + _f(pm, rR, pR, cR, gR) + uR - uL > 0.0:
            hi = pm
        else:
            lo = pm
    ps = 0.5 * (lo + hi)
    us = 0.5 * (uL + uR) + 0.5 * (_f(ps, rR, pR, cR, gR) - _f(ps, rL, pL, cL, gL))
    return ps, us


def exact_riemann(x, t, WL=(1.0, 0.0, 1.0), WR=(0.125, 0.0, 0.1), g=1.4, x0=0.5):
    """(rho, u, p) at positions x and time t > 0 for the initial discontinuity at x0."""
    rL, uL, pL = WL
    rR, uR, pR = WR
    gL, gR = _gammas(g)
    cL, cR = math.sqrt(gL * pL / rL), math.sqrt(gR * pR / rR)
    ps, us = star_state(WL, WR, (gL, gR))
    out = np.zeros((3, len(x)))
    for n, xx in enumerate(np.asarray(x, dtype=float)):
        S = (xx - x0) / t
        if S < us:
            g = gL
            if ps > pL:
                rs = rL * ((ps / pL + (g - 1) / (g + 1)) / ((g - 1) / (g + 1) * ps / pL + 1))
                SL = uL - cL * math.sqrt((g + 1) / (2 * g) * ps / pL + (g - 1) / (2 * g))
                W = (rL, uL, pL) if S < SL else (rs, us, ps)
            else:
                rs = rL * (ps / pL) ** (1 / g)
                cs = cL * (ps / pL) ** ((g - 1) / (2 * g))
                if S < uL - cL:
                    W = (rL, uL, pL)
                elif S > us - cs:
                    W = (rs, us, ps)
                else:  # inside the left rarefaction fan
                    u = 2 / (g + 1) * (cL + (g - 1) / 2 * uL + S)
                    c = 2 / (g + 1) * (cL + (g - 1) / 2 * (uL - S))
                    W = (rL * (c / cL) ** (2 / (g - 1)), u, pL * (c / cL) ** (2 * g / (g - 1)))
        else:
            g = gR
            if ps > pR:
                rs = rR * ((ps / pR + (g - 1) / (g + 1)) / ((g - 1) / (g + 1) * ps / pR + 1))
                SR = uR + cR * math.sqrt((g + 1) / (2 * g) * ps / pR + (g - 1) / (2 * g))
                W = (rR, uR, pR) if S > SR else (rs, us, ps)
            else:
                rs = rR * (ps / pR) ** (1 / g)
                cs = cR * (ps / pR) ** ((g - 1) / (2 * g))
                if S > uR + cR:
                    W = (rR, uR, pR)
                elif S < us + cs:
                    W = (rs, us, ps)
                else:
                    u = 2 / (g + 1) * (-cR + (g - 1) / 2 * uR + S)
                    c = 2 / (g + 1) * (cR - (g - 1) / 2 * (uR - S))
                    W = (rR * (c / cR) ** (2 / (g - 1)), u, pR * (c / cR) ** (2 * g / (g - 1)))
        out[:, n] = W
    return out


def noh_planar(t, g, u0=-1.0, rho0=1.0):
    """Shock position, post-shock (rho, p, e) of the planar Noh problem."""
    D = 0.5 * (g - 1.0) * abs(u0)
    rho2 = rho0 * (g + 1.0) / (g - 1.0)
    p2 = rho0 * (D + abs(u0)) * abs(u0)
    return D * t, rho2, p2, 0.5 * u0 * u0


def noh_spherical(r, t, g, u0=-1.0, rho0=1.0):
    """Noh's spherical problem (3D, cold gas at u0 r_hat): the shock at r_s = D t with
    D = (g - 1) |u0| / 2; inside rho = rho0 ((g + 1)/(g - 1))^3, u = 0, p = (g - 1) rho e
    with e = u0^2 / 2; outside the cold gas compressed by convergence, rho = rho0 (1 +
    |u0| t / r)^2, u = u0, p = 0.  Returns (r_s, rho(r))."""
    D = 0.5 * (g - 1.0) * abs(u0)
    rs = D * t
    r = np.asarray(r, dtype=float)
    inside = rho0 * ((g + 1.0) / (g - 1.0)) ** 3
    ahead = rho0 * (1.0 + abs(u0) * t / np.where(r < rs, 1.0, r)) ** 2
    rho = np.where(r < rs, inside, ahead)
    return rs, rho
