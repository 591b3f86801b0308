"""Fused ghost fill (StageArgs::fill_ctas): the FAST cell-split
Van Leer launch fills the ghosts of W[cur] itself — fill CTAs first, the
tiles that read no ghost cell beside them, boundary tiles after a device-side
acquire of the fill's completion counter — instead of one ghost_kernel launch
before every stage.  Every ghost value is the double the separate launch
writes, so fused and separate runs must be bitwise identical (fields and
residual history), for any number of fill CTAs, and the fused path must agree
with the CPU oracle as the separate one does.  BF_FUSED_FILL / BF_FILL_CTAS
are read at context creation."""

import numpy as np
import pytest

from paper_2012_02925_b200 import cases, geometry, planning
from paper_2012_02925_b200.model import FIELD_NAMES, GasModel, SchemeConfig

from test_gpu_parity import compare, run_pair

pytestmark = pytest.mark.gpu
GAS = GasModel()


def _run(monkeypatch, fused, plan, cfg, fs, steps, ctas=None, init="perturbed"):
    from paper_2012_02925_b200.stepper import iterate_gpu
    monkeypatch.setenv("BF_FUSED_FILL", "1" if fused else "0")
    if ctas is None:
        monkeypatch.delenv("BF_FILL_CTAS", raising=False)
    else:
        monkeypatch.setenv("BF_FILL_CTAS", str(ctas))
    sched = planning.reorder_boundaries(plan)
    return iterate_gpu(plan, sched, GAS, cfg, fs, steps, init=init, precision="fast")


def _same(a, b):
    np.testing.assert_array_equal(a.history, b.history)
    for cid, va in a.solvers.items():
        vb = b.solvers[cid]
        for n in FIELD_NAMES:
            np.testing.assert_array_equal(va.fields[n], vb.fields[n], err_msg=f"{cid} {n}")


CASES = {
    # 3D: farfield on every outer face, connected faces between 8 children
    "box3d_8": lambda: (planning.decompose(geometry.multiblock_box_3d(3), 8, 3),
                        SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.8),
                        cases.freestream_for("multiblock_box_3d", GAS, 3)),
    # C4's geometry and scheme at level 6 (4 parents)
    "c4_l6": lambda: cases.c4_box(level=6, np_ranks=1)[0:1] + cases.c4_box(level=6, np_ranks=1)[3:5],
    # 2D: inflow / outflow / walls, 2 children
    "ramp2d": lambda: (planning.decompose(geometry.inlet_ramp_2d(1), 2, 2),
                       SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.5),
                       cases.freestream_for("inlet_ramp_2d", GAS, 2)),
    # C1 (the SPEC case), single block
    "c1": lambda: (cases.c1_inlet()[0], cases.c1_inlet()[3], cases.c1_inlet()[4]),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_fused_fill_bitwise_vs_separate_launch(monkeypatch, name):
    plan, cfg, fs = CASES[name]()
    init = "uniform" if name == "c1" else "perturbed"
    a = _run(monkeypatch, True, plan, cfg, fs, 9, init=init)
    b = _run(monkeypatch, False, plan, cfg, fs, 9, init=init)
    _same(a, b)


@pytest.mark.parametrize("ctas", [1, 2, 7, 64])
def test_fused_fill_any_number_of_fill_ctas(monkeypatch, ctas):
    plan, cfg, fs = CASES["box3d_8"]()
    a = _run(monkeypatch, True, plan, cfg, fs, 5, ctas=ctas)
    b = _run(monkeypatch, False, plan, cfg, fs, 5)
    _same(a, b)


def test_fused_fill_matches_oracle(monkeypatch):
    monkeypatch.setenv("BF_FUSED_FILL", "1")
    plan, cfg, fs = CASES["box3d_8"]()
    ref, got = run_pair(plan, cfg, fs, 6, init="perturbed", precision="fast")
    compare(ref, got, fs, bitwise=False)


def test_fused_fill_replaces_the_ghost_launches(monkeypatch):
    """With the fused fill on, ghost launches happen only for the first fill
    after the upload (both buffers); every later stage is one launch."""
    from paper_2012_02925_b200 import stepper
    monkeypatch.setenv("BF_FUSED_FILL", "1")
    plan, cfg, fs = CASES["box3d_8"]()
    gpu = stepper.GpuContext(plan, [c.id for c in plan.children], GAS, cfg, fs, precision="fast",
                             schedule=planning.reorder_boundaries(plan))
    try:
        gpu.upload_initial("perturbed")
        gpu.set_profiling(True)
        st = stepper.GpuRankStepper(gpu, cfg)
        st.run(1, 6)
        n_stage, _ = gpu.kernel_stats(0)
        n_ghost, _ = gpu.kernel_stats(1)
        assert n_stage == 12
        assert n_ghost <= 2, n_ghost
    finally:
        gpu.close()


def test_ghost_block_order_does_not_change_values(monkeypatch):
    """The ghost launch's CUDA blocks are spread over the launch across tasks
    (and 2 items per thread); the tasks of one launch write disjoint ghost
    cells, so the order is invisible in the results: bitwise equal to the task
    order (BF_GHOST_INTERLEAVE=0) with the separate fill launch."""
    plan, cfg, fs = CASES["c4_l6"]()
    monkeypatch.setenv("BF_GHOST_INTERLEAVE", "1")
    a = _run(monkeypatch, False, plan, cfg, fs, 6)
    monkeypatch.setenv("BF_GHOST_INTERLEAVE", "0")
    b = _run(monkeypatch, False, plan, cfg, fs, 6)
    _same(a, b)
