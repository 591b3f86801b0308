"""FAST Roe face-owner kernel (csrc/bf_roe.cuh) vs the CPU oracle.

Each cell computes the Roe flux of its high face in every direction
(physics.py:190-255 with the MUSCL states of solver.py:437-474) and takes its
low faces' fluxes from the neighbours (x: shuffles, y: shared memory, z:
registers); the tile's low x / low y / high x edge faces are extra items.
Every case here runs precision="fast" with the Roe flux, so it goes through
that kernel, and is held to the north-star bar: fields within 1e-12 of the
freestream scale, residual norms |dH_k| <= 1e-12 H_1.  Cases cover every
limiter, general MUSCL (kappa, epsilon), partial tiles in i/j/k, walls / in- /
outflow / farfield / MMS patches in 2D and 3D, decomposed plans, thin blocks
and the error texts (non-physical face state; Roe a^2 <= 0 in
test_gpu_parity_r2.py)."""

import numpy as np
import pytest

from paper_2012_02925_b200 import cases, geometry, planning
from paper_2012_02925_b200.errors import NonPhysicalStateError
from paper_2012_02925_b200.model import FIELD_NAMES, FreestreamState, GasModel, SchemeConfig

import oracle
from test_gpu_parity import compare, run_pair
from test_gpu_vl_split import channel_3d

pytestmark = pytest.mark.gpu
GAS = GasModel()


@pytest.mark.parametrize("limiter", ["van_albada", "minmod", "van_leer", "none"])
@pytest.mark.parametrize("muscl", [(1.0, -1.0), (1.0, 1.0 / 3.0), (0.0, -1.0)])
def test_box3d_roe_all_limiters(limiter, muscl):
    eps, kappa = muscl
    plan = cases.make_plan(geometry.multiblock_box_3d(3), 1)
    fs = cases.freestream_for("multiblock_box_3d", GAS, 3)
    cfg = SchemeConfig(flux="roe", limiter=limiter, epsilon=eps, kappa=kappa, cfl=0.8)
    ref, got = run_pair(plan, cfg, fs, 8, init="perturbed", precision="fast")
    compare(ref, got, fs, bitwise=False)


@pytest.mark.parametrize("kwall", ["noslip_wall", "slip_wall"])
def test_channel3d_roe_walls_partial_tiles(kwall):
    plan = cases.make_plan(channel_3d(kwall=kwall), 1)
    fs = FreestreamState.from_mach(GAS, 2.5, 50000.0, 250.0, 4.0, 3)
    cfg = SchemeConfig(flux="roe", limiter="van_albada", cfl=0.6)
    ref, got = run_pair(plan, cfg, fs, 10, init="perturbed", precision="fast")
    compare(ref, got, fs, bitwise=False)


def test_channel3d_roe_decomposed_rk4():
    plan = planning.decompose(channel_3d(dims=(70, 40, 33)), 4, 3)
    fs = FreestreamState.from_mach(GAS, 2.5, 50000.0, 250.0, 4.0, 3)
    cfg = SchemeConfig(flux="roe", limiter="minmod", rk_stages=4, cfl=0.6)
    ref, got = run_pair(plan, cfg, fs, 4, init="perturbed", precision="fast")
    compare(ref, got, fs, bitwise=False)


def test_c3_mms_roe_split():
    plan, sched, gas, cfg, fs, init = cases.c3_mms(32, 8)
    ref, got = run_pair(plan, cfg, fs, 6, init=init, precision="fast", gas=gas)
    compare(ref, got, fs, bitwise=False)


@pytest.mark.parametrize("limiter", ["van_albada", "minmod", "none"])
def test_inlet2d_roe(limiter):
    plan = planning.decompose(geometry.inlet_ramp_2d(1), 2, 2)
    fs = cases.freestream_for("inlet_ramp_2d", GAS, 2)
    cfg = SchemeConfig(flux="roe", limiter=limiter, epsilon=0.0 if limiter == "none" else 1.0,
                       cfl=0.6)
    ref, got = run_pair(plan, cfg, fs, 30, init="uniform", precision="fast")
    compare(ref, got, fs, bitwise=False)


def test_c1_roe_and_annulus_farfield():
    plan, sched, gas, cfg, fs, init = cases.c1_inlet(flux="roe")
    ref, got = run_pair(plan, cfg, fs, 40, init=init, precision="fast", gas=gas)
    compare(ref, got, fs, bitwise=False)
    plan = planning.decompose(geometry.c_annulus_2d(1), 3, 2)
    fs = cases.freestream_for("c_annulus_2d", GAS, 2)
    cfg = SchemeConfig(flux="roe", limiter="van_albada", cfl=0.7)
    ref, got = run_pair(plan, cfg, fs, 15, init="perturbed", precision="fast")
    compare(ref, got, fs, bitwise=False)


@pytest.mark.parametrize("where", [(10, 10, 0), (0, 3, 0), (51, 15, 0), (31, 7, 0), (32, 0, 0)])
def test_roe_split_non_physical_face_state_message(where):
    """Same NonPhysicalStateError text as the oracle (direction, side, face
    index), poisoned cells inside tiles, on tile edges and on block faces."""
    from paper_2012_02925_b200 import stepper as st
    plan = planning.decompose(geometry.inlet_ramp_2d(0), 1, 2)
    cfg = SchemeConfig(flux="roe", limiter="van_albada", cfl=0.5)
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


@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 3, 1), (5, 1, 4), (33, 17, 3), (3, 40, 2)])
def test_roe_thin_and_tiny_blocks(dims):
    plan = cases.make_plan(channel_3d(dims=dims, kwall="slip_wall"), 1)
    fs = FreestreamState.from_mach(GAS, 2.5, 50000.0, 250.0, 4.0, 3)
    cfg = SchemeConfig(flux="roe", limiter="van_albada", cfl=0.5)
    ref, got = run_pair(plan, cfg, fs, 4, init="perturbed", precision="fast")
    compare(ref, got, fs, bitwise=False)


def test_roe_c4_geometry_level12():
    plan, sched, gas, cfg, fs, init = cases.c4_box(level=12, np_ranks=1, flux="roe")
    ref, got = run_pair(plan, cfg, fs, 2, init=init, precision="fast", gas=gas)
    compare(ref, got, fs, bitwise=False)
