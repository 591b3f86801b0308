"""Laminar Navier-Stokes on the device vs the CPU oracle.

The oracle's viscous restatement is pinned bitwise to the reference by the
ns_* golden cases (tests/test_oracle_golden.py).  Here: EXACT builds bitwise
(padded fields included: edge and corner ghosts follow the reference's ghost
round 2 and extended-BC order) where no libm pow is on the path, the 1e-12
bar otherwise; FAST within 1e-12; the in-process multi-rank driver equal to
the serial one on the interior."""

import numpy as np
import pytest

from paper_2012_02925_b200 import cases, geometry, planning
from paper_2012_02925_b200.geometry import MultiBlockGrid, make_cartesian_block, physical_patch
from paper_2012_02925_b200.model import FIELD_NAMES, FreestreamState, GasModel, SchemeConfig

from test_gpu_parity import compare, run_pair

pytestmark = pytest.mark.gpu


def duct3d(dims, kmin="noslip_wall"):
    blk = make_cartesian_block(0, dims, (0.0, 0.0, 0.0), (1.5, 0.6, 0.5), 3)
    d = blk.dims
    return MultiBlockGrid(blocks=[blk], boundaries=[
        physical_patch(0, "i_min", d, "supersonic_inflow"),
        physical_patch(0, "i_max", d, "supersonic_outflow"),
        physical_patch(0, "j_min", d, "noslip_wall"),
        physical_patch(0, "j_max", d, "slip_wall"),
        physical_patch(0, "k_min", d, kmin),
        physical_patch(0, "k_max", d, "slip_wall")])


@pytest.mark.parametrize("npr", [1, 6])
def test_duct3d_exact_bitwise(npr):
    gas = GasModel(mu=0.2)
    grid = duct3d((40, 24, 18))
    plan = planning.decompose(grid, npr, 3) if npr > 1 else cases.make_plan(grid, 1)
    fs = FreestreamState.from_mach(gas, 2.0, 1.0e5, 250.0, 0.0, 3)
    cfg = SchemeConfig(flux="roe", limiter="van_albada", cfl=0.5, viscous=True,
                       wall_temperature=280.0)
    ref, got = run_pair(plan, cfg, fs, 4, init="perturbed", precision="exact", gas=gas)
    compare(ref, got, fs, bitwise=True)


def test_duct3d_fast_van_leer():
    gas = GasModel(mu=0.2)
    plan = planning.decompose(duct3d((40, 24, 18)), 3, 3)
    fs = FreestreamState.from_mach(gas, 2.0, 1.0e5, 250.0, 0.0, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.5, viscous=True)
    ref, got = run_pair(plan, cfg, fs, 5, init="perturbed", precision="fast", gas=gas)
    compare(ref, got, fs, bitwise=False)


def test_annulus_noslip_self_connected():
    """Self-connected block (round-2 pack and unpack on the same block)."""
    gas = GasModel(mu=5.0)
    plan = planning.decompose(geometry.c_annulus_2d(0, wall="noslip_wall"), 1, 2)
    fs = cases.freestream_for("c_annulus_2d", gas, 2)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.5, viscous=True)
    ref, got = run_pair(plan, cfg, fs, 5, init="uniform", precision="exact", gas=gas)
    compare(ref, got, fs, bitwise=False)   # farfield j_max: libm pow


def test_group_driver_matches_serial_interior():
    from paper_2012_02925_b200.stepper import iterate_gpu, run_distributed_gpu
    gas = GasModel(mu=0.2)
    grid = duct3d((24, 16, 12))
    plan = planning.decompose(grid, 4, 3)
    sched = planning.reorder_boundaries(plan)
    fs = FreestreamState.from_mach(gas, 2.0, 1.0e5, 250.0, 0.0, 3)
    cfg = SchemeConfig(flux="roe", limiter="minmod", cfl=0.5, viscous=True)
    dist = run_distributed_gpu(plan, sched, gas, cfg, fs, max_steps=4, init="perturbed",
                               precision="exact")
    serial = iterate_gpu(plan, sched, gas, cfg, fs, 4, init="perturbed", precision="exact")
    np.testing.assert_array_equal(dist.history, serial.history)
    for pid, flds in dist.fields.items():
        for cid, view in serial.solvers.items():
            c = plan.child(cid)
            if c.parent != pid:
                continue
            (i0, i1), (j0, j1), (k0, k1) = c.cell_box()
            for n in FIELD_NAMES:
                np.testing.assert_array_equal(flds[n][i0:i1, j0:j1, k0:k1],
                                              view.fields[n][view.block.interior()])
