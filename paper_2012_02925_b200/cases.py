"""The BASELINE.json workloads as plan builders.

Each builder returns (plan, schedule, gas, scheme, freestream, init) built
with this package's host mirrors only, so the same case runs on a box without
the reference installed.  Grid recipes, freestream tables and scheme defaults
follow SURVEY.md §8d and blockflow/cli.py:33-61.
"""

from __future__ import annotations

import numpy as np

from . import geometry, planning
from .model import FreestreamState, GasModel, SchemeConfig

# cli.py:33-44
CASE_TABLES = {
    "inlet_ramp_2d": dict(mach=4.0, pressure=12270.0, temperature=217.0, alpha_deg=0.0),
    "c_annulus_2d": dict(mach=0.25, pressure=84307.0, temperature=300.0, alpha_deg=5.0),
    "multiblock_box_3d": dict(mach=0.8395, pressure=315979.763, temperature=255.556,
                              alpha_deg=3.06),
    "cartesian_box": dict(mach=0.3, pressure=1.0e5, temperature=300.0, alpha_deg=0.0),
}


def freestream_for(case, gas, ndim):
    t = CASE_TABLES[case]
    return FreestreamState.from_mach(gas, t["mach"], t["pressure"], t["temperature"],
                                     t["alpha_deg"], ndim)


def make_plan(grid, np_ranks):
    """aggregate when np < parents, else decompose (test_solver.py:22-31)."""
    if np_ranks < grid.parent_count:
        return planning.aggregate(grid, np_ranks)
    return planning.decompose(grid, np_ranks, grid.ndim)


def c1_inlet(flux="van_leer", ni=128, nj=64):
    """C1: 2D inlet ramp, 128x64 cells, single block, M=4 (cli.py CLI defaults)."""
    gas = GasModel()
    grid = geometry.inlet_ramp_2d(ni=ni, nj=nj)
    plan = make_plan(grid, 1)
    cfg = SchemeConfig(flux=flux, limiter="van_albada", epsilon=1.0, kappa=-1.0, rk_stages=2,
                       cfl=0.8)
    return plan, planning.reorder_boundaries(plan), gas, cfg, freestream_for("inlet_ramp_2d", gas, 2), "uniform"


def c2_channel(np_ranks=4, flux="van_leer", parents=4, ni=512, nj=256, subsonic=False):
    """C2: 4 parents of 512x256 cells cut from one ramp lattice, connected i faces."""
    gas = GasModel()
    grid = geometry.ramp_channel_2d(parents=parents, ni=ni, nj=nj, subsonic=subsonic)
    plan = make_plan(grid, np_ranks)
    cfg = SchemeConfig(flux=flux, limiter="van_albada", rk_stages=2, cfl=0.8)
    if subsonic:
        fs = FreestreamState.from_mach(gas, 0.5, 12270.0, 217.0, 0.0, 2)
    else:
        fs = freestream_for("inlet_ramp_2d", gas, 2)
    return plan, planning.reorder_boundaries(plan), gas, cfg, fs, "uniform"


def c3_mms(n=128, np_ranks=8):
    """C3: 3D n^3 box, Roe, no limiter, z-invariant euler_2d manufactured solution."""
    gas = GasModel()
    grid = geometry.cartesian_box_3d(n, mms=True)
    plan = planning.decompose(grid, np_ranks, 3)
    cfg = SchemeConfig(flux="roe", limiter="none", rk_stages=2, cfl=0.5, mms_id="euler_2d")
    fs = freestream_for("cartesian_box", gas, 3)
    return plan, planning.reorder_boundaries(plan), gas, cfg, fs, "manufactured"


def c4_box(level=15, np_ranks=1, flux="van_leer", cfl=0.8):
    """C4/C5: multiblock_box_3d (level 15 = 256^3 cells), farfield, M=0.8395."""
    gas = GasModel()
    grid = geometry.multiblock_box_3d(level)
    plan = make_plan(grid, np_ranks)
    cfg = SchemeConfig(flux=flux, limiter="van_albada", rk_stages=2, cfl=cfl)
    fs = freestream_for("multiblock_box_3d", gas, 3)
    return plan, planning.reorder_boundaries(plan), gas, cfg, fs, "perturbed"


def perturbed_state(block, fs, gas, rng):
    """C4 initial condition: freestream with interior rho and p
    scaled by (1 + 0.01 N(0,1)); T = p/(rho R).  Returns padded fields."""
    f = {n: block.allocate_field(getattr(fs, n)) for n in ("rho", "u", "v", "w", "p", "T")}
    inner = block.interior()
    for n in ("rho", "p"):
        base = f[n][inner]
        f[n][inner] = base * (1.0 + 0.01 * rng.standard_normal(base.shape))
    f["T"][inner] = f["p"][inner] / (f["rho"][inner] * gas.R)
    return f
