"""FAST Van Leer cell-split kernel (csrc/bf_vl.cuh) vs the CPU oracle.

The split kernel evaluates each face flux as F+(qL) + F-(qR) with both halves
computed by the cells that own the MUSCL states (physics.py:293-297,
solver.py:437-474).  Every case here runs precision="fast" with the Van Leer
flux, so it goes through that kernel, and is held to the north-star bar:
fields within 1e-12 of the freestream scale, residual norms |dH_k| <= 1e-12 H_1.
Cases cover every limiter, general MUSCL (kappa, epsilon), partial tiles in
i/j/k, walls / in- / outflow / farfield / MMS patches in 3D, and the
non-physical face-state error text.
"""

import numpy as np
import pytest

from paper_2012_02925_b200 import cases, geometry, planning
from paper_2012_02925_b200.errors import NonPhysicalStateError
from paper_2012_02925_b200.geometry import MultiBlockGrid, make_cartesian_block, physical_patch
from paper_2012_02925_b200.model import FIELD_NAMES, FreestreamState, GasModel, SchemeConfig

import oracle
from test_gpu_parity import compare, run_pair

pytestmark = pytest.mark.gpu
GAS = GasModel()


def channel_3d(dims=(37, 21, 19), kwall="noslip_wall"):
    """Skewed-free 3D duct: supersonic in/outflow in i, slip walls in j, `kwall`
    in k.  Dimensions deliberately not multiples of the 32 x 16 x KC tile."""
    blk = make_cartesian_block(0, dims, (0.0, 0.0, 0.0), (1.5, 0.7, 0.6), 3)
    d = blk.dims
    return MultiBlockGrid(blocks=[blk], boundaries=[
        physical_patch(0, "i_min", d, "supersonic_inflow"),
        physical_patch(0, "i_max", d, "supersonic_outflow"),
        physical_patch(0, "j_min", d, "slip_wall"),
        physical_patch(0, "j_max", d, "slip_wall"),
        physical_patch(0, "k_min", d, kwall),
        physical_patch(0, "k_max", d, "farfield")])


@pytest.mark.parametrize("limiter", ["van_albada", "minmod", "van_leer", "none"])
@pytest.mark.parametrize("muscl", [(1.0, -1.0), (1.0, 1.0 / 3.0), (0.0, -1.0)])
def test_box3d_split_all_limiters(limiter, muscl):
    eps, kappa = muscl
    plan = cases.make_plan(geometry.multiblock_box_3d(3), 1)
    fs = cases.freestream_for("multiblock_box_3d", GAS, 3)
    cfg = SchemeConfig(flux="van_leer", limiter=limiter, epsilon=eps, kappa=kappa, cfl=0.8)
    ref, got = run_pair(plan, cfg, fs, 8, init="perturbed", precision="fast")
    compare(ref, got, fs, bitwise=False)


@pytest.mark.parametrize("kwall", ["noslip_wall", "slip_wall"])
def test_channel3d_walls_partial_tiles(kwall):
    grid = channel_3d(kwall=kwall)
    plan = cases.make_plan(grid, 1)
    fs = FreestreamState.from_mach(GAS, 2.5, 50000.0, 250.0, 4.0, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.6)
    ref, got = run_pair(plan, cfg, fs, 10, init="perturbed", precision="fast")
    compare(ref, got, fs, bitwise=False)


def test_channel3d_decomposed_rk4():
    grid = channel_3d(dims=(70, 40, 33))
    plan = planning.decompose(grid, 4, 3)
    fs = FreestreamState.from_mach(GAS, 2.5, 50000.0, 250.0, 4.0, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="minmod", rk_stages=4, cfl=0.6)
    ref, got = run_pair(plan, cfg, fs, 4, init="perturbed", precision="fast")
    compare(ref, got, fs, bitwise=False)


def test_mms3d_split():
    plan = planning.decompose(geometry.cartesian_box_3d(20, mms=True), 2, 3)
    fs = FreestreamState.from_mach(GAS, 0.3, 1.0e5, 300.0, 0.0, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="none", mms_id="euler_2d", cfl=0.5)
    ref, got = run_pair(plan, cfg, fs, 5, init="manufactured", precision="fast")
    compare(ref, got, fs, bitwise=False)


@pytest.mark.parametrize("limiter", ["van_albada", "minmod"])
def test_inlet2d_split(limiter):
    plan = planning.decompose(geometry.inlet_ramp_2d(1), 2, 2)
    fs = cases.freestream_for("inlet_ramp_2d", GAS, 2)
    cfg = SchemeConfig(flux="van_leer", limiter=limiter, cfl=0.8)
    ref, got = run_pair(plan, cfg, fs, 30, init="uniform", precision="fast")
    compare(ref, got, fs, bitwise=False)


def test_annulus_farfield_split():
    plan = planning.decompose(geometry.c_annulus_2d(1), 3, 2)
    fs = cases.freestream_for("c_annulus_2d", GAS, 2)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.7)
    ref, got = run_pair(plan, cfg, fs, 15, init="perturbed", precision="fast")
    compare(ref, got, fs, bitwise=False)


@pytest.mark.parametrize("where", [(10, 10, 0), (0, 3, 0), (51, 15, 0)])
def test_split_non_physical_face_state_message(where):
    """Same NonPhysicalStateError text as the oracle (direction, side, face index)."""
    from paper_2012_02925_b200 import stepper as st
    plan = planning.decompose(geometry.inlet_ramp_2d(0), 1, 2)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.5)
    fs = cases.freestream_for("inlet_ramp_2d", GAS, 2)
    gpu = st.GpuContext(plan, [0], GAS, cfg, fs, precision="fast")
    gpu.finalize()
    f6, q5 = gpu.setups[0].initial_state("uniform")
    g = gpu.setups[0].block.ghost
    idx = tuple(w + gg for w, gg in zip(where, g))
    f6[4][idx] = -2.0e5
    gpu.upload(0, f6, q5)
    stepper = st.GpuRankStepper(gpu, cfg)
    with pytest.raises(NonPhysicalStateError, match="face state") as ei:
        stepper.step(1)
    blocks = oracle.build_blocks(plan, GAS, cfg, fs)
    blocks[0].init_uniform()
    blocks[0].fields["p"][idx] = -2.0e5
    sched = planning.reorder_boundaries(plan)
    ost = oracle.OracleStepper(blocks, oracle.make_serial_exchange(plan, sched, blocks), cfg)
    with pytest.raises(NonPhysicalStateError) as eo:
        ost.step(1)
    assert str(ei.value) == str(eo.value)


def test_split_matches_reference_order_kernel():
    """FAST split kernel vs the FAST face kernel (BF_VL=0 path is exercised by
    EXACT runs; here: split FAST vs EXACT on the bench configuration, small)."""
    plan = cases.make_plan(geometry.multiblock_box_3d(4), 1)
    fs = cases.freestream_for("multiblock_box_3d", GAS, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.8)
    from paper_2012_02925_b200.stepper import iterate_gpu
    sched = planning.reorder_boundaries(plan)
    a = iterate_gpu(plan, sched, GAS, cfg, fs, 10, init="perturbed", precision="fast")
    b = iterate_gpu(plan, sched, GAS, cfg, fs, 10, init="perturbed", precision="exact")
    base = b.history[0]
    assert np.max(np.abs(a.history - b.history) / base) <= 1e-12
    for cid in a.solvers:
        for n in FIELD_NAMES:
            x, y = a.solvers[cid].fields[n], b.solvers[cid].fields[n]
            inner = a.solvers[cid].block.interior()
            scale = max(abs(getattr(fs, n)), abs(fs.u)) if n in ("u", "v", "w") else abs(getattr(fs, n))
            assert np.max(np.abs(x[inner] - y[inner])) <= 1e-12 * scale


@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 3, 1), (5, 1, 4), (33, 17, 3), (3, 40, 2)])
@pytest.mark.parametrize("precision", ["fast", "exact"])
def test_thin_and_tiny_blocks(dims, precision):
    """Degenerate shapes: one-cell-thick blocks (the stencil reads only ghosts
    across them, and a wall's second ghost layer mirrors the opposite face's
    ghost: BCs then run in the reference's patch order), partial tiles in every
    axis, tiles thinner than the k-chunk."""
    grid = channel_3d(dims=dims, kwall="slip_wall")
    plan = cases.make_plan(grid, 1)
    fs = FreestreamState.from_mach(GAS, 2.5, 50000.0, 250.0, 4.0, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.5)
    ref, got = run_pair(plan, cfg, fs, 4, init="perturbed", precision=precision)
    compare(ref, got, fs, bitwise=False)


@pytest.mark.parametrize("dims", [(1, 1), (2, 5), (70, 3)])
def test_thin_blocks_2d(dims):
    from paper_2012_02925_b200.geometry import MultiBlockGrid, make_cartesian_block, physical_patch
    blk = make_cartesian_block(0, dims, (0.0, 0.0), (1.0, 0.4), 2)
    d = blk.dims
    grid = MultiBlockGrid(blocks=[blk], boundaries=[
        physical_patch(0, "i_min", d, "supersonic_inflow"),
        physical_patch(0, "i_max", d, "supersonic_outflow"),
        physical_patch(0, "j_min", d, "slip_wall"), physical_patch(0, "j_max", d, "slip_wall")])
    plan = cases.make_plan(grid, 1)
    fs = cases.freestream_for("inlet_ramp_2d", GAS, 2)
    cfg = SchemeConfig(flux="van_leer", limiter="minmod", cfl=0.5)
    ref, got = run_pair(plan, cfg, fs, 5, init="perturbed", precision="fast")
    compare(ref, got, fs, bitwise=False)
