"""Rebuild the golden-fixture cases (tests/golden/make_golden.py) with this
repo's host mirror only, so fixtures can be checked where the reference is
not installed (the GPU box)."""

from __future__ import annotations

import glob
import json
import os

import numpy as np

from paper_2012_02925_b200 import cases, geometry, planning
from paper_2012_02925_b200.model import FIELD_NAMES, FreestreamState, GasModel, SchemeConfig

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TABLES = {
    "inlet_ramp_2d": (4.0, 12270.0, 217.0, 0.0),
    "c_annulus_2d": (0.25, 84307.0, 300.0, 5.0),
    "multiblock_box_3d": (0.8395, 315979.763, 255.556, 3.06),
    "cartesian_box": (0.3, 1.0e5, 300.0, 0.0),
    "channel": (2.0, 1.0e5, 250.0, 0.0),
}
FARFIELD = ("c_annulus_2d", "multiblock_box_3d")   # libm pow on the path


def names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(HERE, "*.npz")))


def load(name):
    z = np.load(os.path.join(HERE, name + ".npz"))
    desc = json.loads(str(z["desc"]))
    return desc, z


def channel(name):
    """Same ducts as make_golden.build_grid, through this repo's mirror."""
    from paper_2012_02925_b200.geometry import MultiBlockGrid, make_cartesian_block, physical_patch
    if name == "channel2d":
        blk = make_cartesian_block(0, (30, 12), (0.0, 0.0), (1.5, 0.5), 2)
        faces = [("i_min", "supersonic_inflow"), ("i_max", "supersonic_outflow"),
                 ("j_min", "noslip_wall"), ("j_max", "slip_wall")]
    else:
        blk = make_cartesian_block(0, (20, 10, 8), (0.0, 0.0, 0.0), (1.5, 0.6, 0.5), 3)
        faces = [("i_min", "supersonic_inflow"), ("i_max", "supersonic_outflow"),
                 ("j_min", "noslip_wall"), ("j_max", "slip_wall"),
                 ("k_min", "noslip_wall"), ("k_max", "slip_wall")]
    return MultiBlockGrid(blocks=[blk], boundaries=[physical_patch(0, f, blk.dims, t)
                                                    for f, t in faces])


def build(desc):
    gas_kw = dict(desc.get("gas", {}))
    if "sutherland" in gas_kw:
        gas_kw["sutherland"] = tuple(gas_kw["sutherland"])
    gas = GasModel(**gas_kw)
    gname, level = desc["grid"], desc["level"]
    if gname.startswith("channel"):
        grid = channel(gname)
        fkey = "channel"
    elif gname == "cube3d_8":
        grid = geometry.cartesian_box_3d(8, mms=True)
        fkey = "cartesian_box"
    else:
        grid = geometry.generate_case_grid(gname, level)
        fkey = gname
    npr = desc["np"]
    plan = cases.make_plan(grid, npr)
    sched = planning.reorder_boundaries(plan)
    m, p, T, a = TABLES[fkey]
    fs = FreestreamState.from_mach(gas, m, p, T, a, grid.ndim)
    cfg = SchemeConfig(**desc["scheme"])
    return plan, sched, gas, cfg, fs


def bitwise_case(desc):
    """Cases whose path avoids libm pow (no farfield patches, no Sutherland law)
    are bitwise."""
    return desc["grid"] not in FARFIELD and "sutherland" not in desc.get("gas", {})


def fields_of(z, cid):
    return {n: z[f"c{cid}_{n}"] for n in FIELD_NAMES}


def run_oracle(desc):
    import oracle
    plan, sched, gas, cfg, fs = build(desc)
    blocks = oracle.build_blocks(plan, gas, cfg, fs)
    oracle.blockflow_oracle._init(blocks, desc["init"])
    st = oracle.OracleStepper(blocks, oracle.make_serial_exchange(plan, sched, blocks), cfg)
    hist = np.array([np.sqrt(st.step(k + 1)[0]) for k in range(desc["steps"])])
    return plan, hist, blocks


def history_ok(got, ref, tol=1e-12):
    base = ref[0]
    scale = np.where(base > 1e-12 * base.max(), base, base.max())
    return float(np.max(np.abs(got - ref) / scale)) <= tol


def field_err(a, b, fs, name):
    speed = max(abs(fs.u), abs(fs.v), abs(fs.w))
    scale = speed if name in ("u", "v", "w") else max(abs(getattr(fs, name)), 1e-300)
    return float(np.max(np.abs(a - b))) / scale
