"""Generate the golden vectors from the REFERENCE package (development container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every case is built and run with the reference's own public API
(blockflow.mesh / decomp / solver), then stored as a small .npz:
case description, residual-norm history, final padded fields and conserved
variables of every child (and the limiter arrays of the freeze case).  The
fixtures pin the CPU oracle (tests/test_oracle_golden.py) and the GPU path
(tests/test_gpu_golden.py) without the reference being present.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from blockflow import decomp, mesh, physics, solver  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

TABLES = {
    "inlet_ramp_2d": (4.0, 12270.0, 217.0, 0.0),
    "c_annulus_2d": (0.25, 84307.0, 300.0, 5.0),
    "multiblock_box_3d": (0.8395, 315979.763, 255.556, 3.06),
    "cartesian_box": (0.3, 1.0e5, 300.0, 0.0),
    "channel": (2.0, 1.0e5, 250.0, 0.0),
}

# laminar Navier-Stokes cases: (gas kwargs) per case name
GAS = {
    "ns_channel2d_noslip_tw_np3": dict(mu=0.5),
    "ns_channel3d_noslip_np4": dict(mu=0.3),
    "ns_mms2d_l1": dict(mu=0.01),
    "ns_box3d_sutherland_np8": dict(sutherland=(0.05, 273.15, 110.4)),
}

# name: (grid, level, np, scheme kwargs, init, steps, farfield?)
CASES = {
    "inlet_vl_va_rk2": ("inlet_ramp_2d", 0, 1, dict(flux="van_leer", limiter="van_albada", cfl=0.8),
                        "uniform", 10),
    "inlet_roe_minmod_rk4_np2": ("inlet_ramp_2d", 0, 2,
                                 dict(flux="roe", limiter="minmod", rk_stages=4, cfl=0.6),
                                 "uniform", 5),
    "inlet_vl_vanleer_freeze": ("inlet_ramp_2d", 0, 1,
                                dict(flux="van_leer", limiter="van_leer", cfl=0.6,
                                     limiter_freeze_at=2), "uniform", 4),
    "annulus_roe_va_np4": ("c_annulus_2d", 0, 4, dict(flux="roe", limiter="van_albada", cfl=0.5),
                           "uniform", 5),
    "box3d_vl_va_np8": ("multiblock_box_3d", 0, 8, dict(flux="van_leer", limiter="van_albada",
                                                         cfl=0.8), "perturbed", 3),
    "box3d_roe_none_np2_l1": ("multiblock_box_3d", 1, 2, dict(flux="roe", limiter="none", cfl=0.5),
                              "perturbed", 3),
    "mms2d_roe_l1": ("cartesian_box", 1, 1, dict(flux="roe", limiter="none", cfl=0.5,
                                                 mms_id="euler_2d"), "manufactured", 5),
    "mms3d_cube8_np2": ("cube3d_8", None, 2, dict(flux="roe", limiter="none", cfl=0.5,
                                                  mms_id="euler_2d"), "manufactured", 3),
    "inlet_eps0_kappa": ("inlet_ramp_2d", 0, 1, dict(flux="roe", limiter="none", epsilon=0.0,
                                                     cfl=0.5), "uniform", 4),
    "ns_channel2d_noslip_tw_np3": ("channel2d", None, 3,
                                   dict(flux="van_leer", limiter="van_albada", cfl=0.5,
                                        viscous=True, wall_temperature=300.0), "uniform", 6),
    "ns_channel3d_noslip_np4": ("channel3d", None, 4,
                                dict(flux="roe", limiter="minmod", cfl=0.5, viscous=True),
                                "perturbed", 4),
    "ns_mms2d_l1": ("cartesian_box", 1, 2, dict(flux="roe", limiter="none", cfl=0.5,
                                                viscous=True, mms_id="ns_2d"), "manufactured", 4),
    "ns_box3d_sutherland_np8": ("multiblock_box_3d", 0, 8,
                                dict(flux="van_leer", limiter="van_albada", cfl=0.6, viscous=True),
                                "perturbed", 3),
}


def build_grid(name, level):
    if name in ("channel2d", "channel3d"):
        # duct: supersonic in/outflow in i, no-slip j_min, slip j_max (+ no-slip k_min,
        # slip k_max in 3D); dims not multiples of the device tile
        if name == "channel2d":
            blk = mesh.make_cartesian_block(0, (30, 12), (0.0, 0.0), (1.5, 0.5), 2)
            faces = [("i_min", "supersonic_inflow"), ("i_max", "supersonic_outflow"),
                     ("j_min", "noslip_wall"), ("j_max", "slip_wall")]
        else:
            blk = mesh.make_cartesian_block(0, (20, 10, 8), (0.0, 0.0, 0.0), (1.5, 0.6, 0.5), 3)
            faces = [("i_min", "supersonic_inflow"), ("i_max", "supersonic_outflow"),
                     ("j_min", "noslip_wall"), ("j_max", "slip_wall"),
                     ("k_min", "noslip_wall"), ("k_max", "slip_wall")]
        specs = [mesh._physical(0, f, blk.dims, t) for f, t in faces]
        return mesh.MultiBlockGrid(blocks=[blk], boundaries=specs)
    if name == "cube3d_8":
        blk = mesh.make_cartesian_block(0, (8, 8, 8), (0.0, 0.0, 0.0), (1.0, 1.0, 1.0), 3)
        specs = [mesh._physical(0, f, blk.dims, "mms_dirichlet")
                 for f in ("i_min", "i_max", "j_min", "j_max", "k_min", "k_max")]
        return mesh.MultiBlockGrid(blocks=[blk], boundaries=specs)
    return mesh.generate_case_grid(name, level)


def freestream(name, gas, ndim):
    key = "cartesian_box" if name == "cube3d_8" else name
    key = "channel" if name.startswith("channel") else key
    m, p, T, a = TABLES[key]
    return solver.FreestreamState.from_mach(gas, m, p, T, a, ndim)


def perturb(solvers, fs, gas, seed=0):
    """SURVEY §8d C4 initial state through the reference objects."""
    rng = np.random.default_rng(seed)
    for cid in sorted(solvers):
        s = solvers[cid]
        s.init_uniform()
        inner = s.block.interior()
        for n in ("rho", "p"):
            base = s.fields[n][inner]
            s.fields[n][inner] = base * (1.0 + 0.01 * rng.standard_normal(base.shape))
        s.fields["T"][inner] = s.fields["p"][inner] / (s.fields["rho"][inner] * gas.R)
        s.sync_conserved()


def run_case(name):
    grid_name, level, npr, kw, init, steps = CASES[name]
    gas = physics.GasModel(**GAS.get(name, {}))
    grid = build_grid(grid_name, level)
    plan = decomp.aggregate(grid, npr) if npr < grid.parent_count else \
        decomp.decompose(grid, npr, grid.ndim)
    sched = decomp.reorder_boundaries(plan)
    fs = freestream(grid_name, gas, grid.ndim)
    cfg = solver.SchemeConfig(**kw)
    solvers = solver.build_block_solvers(plan, gas, cfg, fs)
    if init == "perturbed":
        perturb(solvers, fs, gas)
    else:
        for s in solvers.values():
            s.init_manufactured() if init == "manufactured" else s.init_uniform()
    stepper = solver.RankStepper(solvers, solver.make_serial_exchange(plan, sched, solvers), cfg)
    hist = [solver.residual_norms(stepper.step(k + 1)[0]) for k in range(steps)]
    out = {"history": np.array(hist)}
    for cid, s in solvers.items():
        for n in ("rho", "u", "v", "w", "p", "T"):
            out[f"c{cid}_{n}"] = s.fields[n]
        for e in range(5):
            out[f"c{cid}_q{e}"] = s.q[e]
        if cfg.limiter_freeze_at:
            for d in s.dirs:
                out[f"c{cid}_psi{d}_plus"] = s.psi[d][0]
                out[f"c{cid}_psi{d}_minus"] = s.psi[d][1]
    desc = {"grid": grid_name, "level": level, "np": npr, "scheme": kw, "init": init,
            "gas": GAS.get(name, {}),
            "steps": steps, "children": [c.id for c in plan.children],
            "numpy": np.__version__}
    out["desc"] = np.array(json.dumps(desc))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    return desc


if __name__ == "__main__":
    for name in (sys.argv[1:] or CASES):
        d = run_case(name)
        print(name, d["children"])
