"""Interior / boundary tile split (the launch structure used to overlap the
NCCL halo exchange with interior compute).

On one GPU there is no communicator, so BF_SPLIT_TILES=1 forces the split on
every block face: each stage runs as two stage-kernel launches over disjoint
tile lists (interior tiles, then boundary tiles), with per-tile partials
indexed by tile id.  Results must be unchanged: bitwise vs the oracle in
EXACT mode, within 1e-12 in FAST mode, and the group driver identical."""

import numpy as np
import pytest

from paper_2012_02925_b200 import cases, geometry, planning
from paper_2012_02925_b200.model import GasModel, SchemeConfig

from test_gpu_parity import compare, run_pair

pytestmark = pytest.mark.gpu
GAS = GasModel()


@pytest.fixture(autouse=True)
def split_tiles(monkeypatch):
    monkeypatch.setenv("BF_SPLIT_TILES", "1")


@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_split_tiles_box3d(precision):
    plan = planning.decompose(geometry.multiblock_box_3d(3), 4, 3)
    fs = cases.freestream_for("multiblock_box_3d", GAS, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.8)
    ref, got = run_pair(plan, cfg, fs, 6, init="perturbed", precision=precision)
    compare(ref, got, fs, bitwise=False)


def test_split_tiles_inlet_bitwise():
    plan = planning.decompose(geometry.inlet_ramp_2d(1), 3, 2)
    fs = cases.freestream_for("inlet_ramp_2d", GAS, 2)
    cfg = SchemeConfig(flux="roe", limiter="minmod", cfl=0.5)
    ref, got = run_pair(plan, cfg, fs, 10, init="uniform", precision="exact")
    compare(ref, got, fs, bitwise=True)


def test_split_tiles_group_matches_serial():
    from paper_2012_02925_b200.stepper import iterate_gpu, run_distributed_gpu
    grid = geometry.multiblock_box_3d(2)
    fs = cases.freestream_for("multiblock_box_3d", GAS, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.8)
    plan = planning.decompose(grid, 4, 3)
    sched = planning.reorder_boundaries(plan)
    dist = run_distributed_gpu(plan, sched, GAS, cfg, fs, max_steps=5, init="perturbed",
                               precision="exact")
    serial = iterate_gpu(plan, sched, GAS, cfg, fs, 5, init="perturbed", precision="exact")
    np.testing.assert_array_equal(dist.history, serial.history)
