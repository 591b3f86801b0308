"""Device metrics (bf_add_block_nodes) vs the host compute_metrics.

The device computes face unit normals, areas and cell volumes from the padded
node coordinates with the reference's operation order (mesh.py:250-331,
solver.py:212-220); they must be bitwise equal to the host arrays, and an
inverted cell must raise the reference's MetricError text."""

import numpy as np
import pytest

from paper_2012_02925_b200 import cases, geometry, planning
from paper_2012_02925_b200.errors import MetricError
from paper_2012_02925_b200.geometry import Block, MultiBlockGrid, physical_patch
from paper_2012_02925_b200.model import FIELD_NAMES, GasModel, SchemeConfig

pytestmark = pytest.mark.gpu
GAS = GasModel()


def warped_box_3d(dims=(19, 13, 11), seed=3):
    """Smoothly warped, non-orthogonal 3D block (all metric terms non-trivial)."""
    n = [d + 1 for d in dims]
    s = [np.linspace(0.0, 1.0, m) for m in n]
    X, Y, Z = np.meshgrid(*s, indexing="ij")
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.02, 0.05, size=6)
    x = X + a[0] * np.sin(2 * np.pi * Y) * np.cos(np.pi * Z) + 0.3 * Y
    y = Y + a[1] * np.sin(2 * np.pi * Z) + a[2] * X * X
    z = Z + a[3] * np.sin(np.pi * X) * np.sin(np.pi * Y) + 0.1 * X
    blk = Block(0, np.stack([x, y, z]), 3)
    d = blk.dims
    return MultiBlockGrid(blocks=[blk], boundaries=[
        physical_patch(0, f, d, "farfield") for f in
        ("i_min", "i_max", "j_min", "j_max", "k_min", "k_max")])


def _host_face(metrics, block, d):
    g = block.ghost
    sv = metrics.face_vectors[d]
    sl = tuple(slice(None) if a == d else slice(g[a], g[a] + block.dims[a]) for a in range(3))
    sx, sy, sz = (np.asarray(sv[c])[sl] for c in range(3))
    A = np.sqrt((sx * sx + sy * sy) + sz * sz)
    with np.errstate(invalid="ignore", divide="ignore"):
        n = [np.where(A > 0, c / A, 0.0) for c in (sx, sy, sz)]
    return n + [A]


@pytest.mark.parametrize("grid", ["warped3d", "box3d", "inlet2d", "annulus2d"])
def test_device_metrics_bitwise(grid):
    from paper_2012_02925_b200 import native, stepper
    g = {"warped3d": lambda: warped_box_3d(),
         "box3d": lambda: geometry.multiblock_box_3d(2),
         "inlet2d": lambda: geometry.inlet_ramp_2d(1),
         "annulus2d": lambda: geometry.c_annulus_2d(1)}[grid]()
    plan = cases.make_plan(g, 1)
    fs = cases.freestream_for("multiblock_box_3d" if g.ndim == 3 else "c_annulus_2d", GAS, g.ndim)
    cfg = SchemeConfig(flux="van_leer", cfl=0.5)
    ids = [c.id for c in plan.children]
    gpu = stepper.GpuContext(plan, ids, GAS, cfg, fs, precision="exact")
    try:
        gpu.finalize()
        for cid in ids:
            s = gpu.setups[cid]
            assert s.device_metrics
            host = geometry.compute_metrics(s.block)
            vol = gpu.download(cid, native.FIELD_VOL)
            np.testing.assert_array_equal(vol, host.volume[s.block.interior()])
            for d in range(g.ndim):
                want = _host_face(host, s.block, d)
                for c in range(4):
                    got = gpu.download(cid, native.FIELD_FACE + 4 * d + c)
                    np.testing.assert_array_equal(got, want[c], err_msg=f"d={d} c={c}")
    finally:
        gpu.close()


def test_device_metrics_inverted_cell_message():
    from paper_2012_02925_b200 import stepper
    grid = warped_box_3d(dims=(6, 5, 4))
    blk = grid.blocks[0]
    g = blk.ghost_depth
    nodes = blk.nodes.copy()
    nodes[0, g + 3, g + 2, g + 2] += 5.0          # fold one interior node through its neighbours
    bad = Block.from_padded_nodes(0, nodes, blk.dims, 3)
    with pytest.raises(MetricError) as host_err:
        geometry.compute_metrics(bad)
    grid2 = MultiBlockGrid(blocks=[bad], boundaries=grid.boundaries)
    plan = cases.make_plan(grid2, 1)
    fs = cases.freestream_for("multiblock_box_3d", GAS, 3)
    with pytest.raises(MetricError) as dev_err:
        stepper.GpuContext(plan, [0], GAS, SchemeConfig(flux="van_leer"), fs)
    assert str(dev_err.value) == str(host_err.value)


@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_device_and_host_metrics_runs_identical(precision):
    """Same run with device metrics and with host metrics uploaded: bitwise."""
    from paper_2012_02925_b200.stepper import iterate_gpu
    plan = planning.decompose(warped_box_3d(dims=(24, 17, 15)), 2, 3)
    sched = planning.reorder_boundaries(plan)
    fs = cases.freestream_for("multiblock_box_3d", GAS, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.6)
    a = iterate_gpu(plan, sched, GAS, cfg, fs, 4, init="perturbed", precision=precision)
    b = iterate_gpu(plan, sched, GAS, cfg, fs, 4, init="perturbed", precision=precision,
                    metrics_fn=geometry.compute_metrics)
    np.testing.assert_array_equal(a.history, b.history)
    for cid in a.solvers:
        for n in FIELD_NAMES:
            np.testing.assert_array_equal(a.solvers[cid].fields[n], b.solvers[cid].fields[n])


def test_async_registration_reports_the_inverted_block():
    """bf_add_block_nodes returns before its metric kernels finish (the next
    block's node copy overlaps them); bf_sync_blocks, called at the end of
    GpuContext construction, reports the first registered block with an
    inverted cell — here the second of two children — with the reference text."""
    from paper_2012_02925_b200 import stepper
    grid = warped_box_3d(dims=(12, 5, 4))
    plan = planning.decompose(grid, 2, 3)
    cid = sorted(c.id for c in plan.children)[1]
    setups = stepper.host_setups(plan, [c.id for c in plan.children], GAS,
                                 SchemeConfig(flux="van_leer"),
                                 cases.freestream_for("multiblock_box_3d", GAS, 3))
    blk = setups[cid].block
    g = blk.ghost_depth
    blk.nodes = blk.nodes.copy()
    blk.nodes[0, g + 3, g + 2, g + 2] += 5.0
    with pytest.raises(MetricError) as host_err:
        geometry.compute_metrics(blk)
    fs = cases.freestream_for("multiblock_box_3d", GAS, 3)
    with pytest.raises(MetricError) as dev_err:
        stepper.GpuContext(plan, [c.id for c in plan.children], GAS, SchemeConfig(flux="van_leer"),
                           fs, setups=setups)
    assert str(dev_err.value) == str(host_err.value)
    assert str(dev_err.value).startswith(f"block {cid}:")
