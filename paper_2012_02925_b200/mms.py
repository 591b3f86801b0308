"""Manufactured solutions and their Euler source terms (setup-time only).

Restates blockflow/physics.py:359-453: sinusoidal primitive fields on the
unit square (w = 0, z-independent) and the steady source S = div F(Q_exact)
derived symbolically with sympy.  The expression trees are built with the
same sympy operations as the reference so that, on one machine, the
lambdified numpy code and therefore the per-cell values agree; the device
path consumes the host-evaluated arrays (S * V per interior cell and the
Dirichlet ghost values), never the symbolic form.
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np

MMS_IDS = ("constant", "euler_2d", "ns_2d")

# (base, amplitude_x, wavenumber_x, amplitude_y, wavenumber_y), physics.py:362-367
_COEFFS = {
    "rho": (1.0, 0.15, 0.75, 0.10, 1.00),
    "u": (70.0, 7.0, 1.00, 4.0, 1.25),
    "v": (90.0, 6.0, 1.25, 5.0, 0.75),
    "p": (1.0e5, 2.0e4, 1.00, 1.0e4, 0.75),
}


def _symbolic(ms_id):
    import sympy as sp
    x, y = sp.symbols("x y", real=True)
    if ms_id == "constant":
        return x, y, {"rho": sp.Float(1.0), "u": sp.Float(50.0), "v": sp.Float(-30.0),
                      "w": sp.Float(0.0), "p": sp.Float(8.0e4)}
    pi = sp.pi
    fields = {}
    for name, (base, ax, kx, ay, ky) in _COEFFS.items():
        fx, fy = {"rho": (sp.sin, sp.cos), "u": (sp.cos, sp.sin),
                  "v": (sp.sin, sp.cos), "p": (sp.cos, sp.sin)}[name]
        fields[name] = base + ax * fx(kx * pi * x) + ay * fy(ky * pi * y)
    fields = {"rho": fields["rho"], "u": fields["u"], "v": fields["v"],
              "w": sp.Float(0.0), "p": fields["p"]}
    return x, y, fields


def _numpy_fn(x, y, expr):
    import sympy as sp
    f = sp.lambdify((x, y), expr, modules="numpy")

    def call(xa, ya, za=None):
        xa = np.asarray(xa, float)
        return np.broadcast_to(np.asarray(f(xa, ya), float), xa.shape).copy()
    return call


@lru_cache(maxsize=None)
def _solution(ms_id):
    if ms_id not in MMS_IDS:
        raise ValueError(f"unknown manufactured solution id {ms_id!r}")
    x, y, f = _symbolic(ms_id)
    return {n: _numpy_fn(x, y, e) for n, e in f.items()}


def manufactured_solution(ms_id):
    """{rho,u,v,w,p}(x, y, z) callables (physics.py:409-411)."""
    return _solution(ms_id)


@lru_cache(maxsize=None)
def _sources(ms_id, gamma, R, mu, prandtl):
    import sympy as sp
    if ms_id not in MMS_IDS:
        raise ValueError(f"unknown manufactured solution id {ms_id!r}")
    x, y, f = _symbolic(ms_id)
    rho, u, v, p = f["rho"], f["u"], f["v"], f["p"]
    et = p / ((gamma - 1) * rho) + (u ** 2 + v ** 2) / 2
    ht = et + p / rho
    s = [sp.diff(rho * u, x) + sp.diff(rho * v, y),
         sp.diff(rho * u * u + p, x) + sp.diff(rho * u * v, y),
         sp.diff(rho * u * v, x) + sp.diff(rho * v * v + p, y),
         sp.Float(0.0),
         sp.diff(rho * u * ht, x) + sp.diff(rho * v * ht, y)]
    if ms_id == "ns_2d":
        T = p / (rho * R)
        k = mu * (gamma * R / (gamma - 1)) / prandtl
        div = sp.diff(u, x) + sp.diff(v, y)
        txx = 2 * mu * sp.diff(u, x) - sp.Rational(2, 3) * mu * div
        tyy = 2 * mu * sp.diff(v, y) - sp.Rational(2, 3) * mu * div
        txy = mu * (sp.diff(u, y) + sp.diff(v, x))
        s[1] -= sp.diff(txx, x) + sp.diff(txy, y)
        s[2] -= sp.diff(txy, x) + sp.diff(tyy, y)
        qx = u * txx + v * txy + k * sp.diff(T, x)
        qy = u * txy + v * tyy + k * sp.diff(T, y)
        s[4] -= sp.diff(qx, x) + sp.diff(qy, y)
    s = [s[0], s[1], s[2], s[3], s[4]]
    return [_numpy_fn(x, y, sp.together(e.doit())) for e in s]


def mms_source(x, y, z, ms_id, gas):
    """Source components (mass, x/y/z-momentum, energy) at cell centres."""
    fns = _sources(ms_id, gas.gamma, gas.R, getattr(gas, "mu", 0.0), getattr(gas, "prandtl", 0.72))
    return tuple(fn(x, y, z) for fn in fns)
