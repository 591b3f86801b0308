"""One RK step replayed from a CUDA graph (bf_step).

Steps after the first are captured once per starting buffer and replayed;
BF_GRAPH=0 (read at context creation) keeps every launch on the stream.  The
two paths must give identical histories and fields, bitwise, and agree with
the oracle as the plain path does."""

import numpy as np
import pytest

from paper_2012_02925_b200 import cases, geometry, planning
from paper_2012_02925_b200.model import FIELD_NAMES, GasModel, SchemeConfig

from test_gpu_parity import compare, run_pair

pytestmark = pytest.mark.gpu
GAS = GasModel()


def _run(monkeypatch, graph, plan, cfg, fs, steps, precision):
    from paper_2012_02925_b200.stepper import iterate_gpu
    monkeypatch.setenv("BF_GRAPH", graph)
    sched = planning.reorder_boundaries(plan)
    return iterate_gpu(plan, sched, GAS, cfg, fs, steps, init="uniform", precision=precision)


@pytest.mark.parametrize("precision,rk", [("exact", 2), ("fast", 2), ("fast", 1), ("exact", 4)])
def test_graph_replay_bitwise(monkeypatch, precision, rk):
    plan = planning.decompose(geometry.inlet_ramp_2d(1), 2, 2)
    fs = cases.freestream_for("inlet_ramp_2d", GAS, 2)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.5, rk_stages=rk)
    a = _run(monkeypatch, "1", plan, cfg, fs, 7, precision)
    b = _run(monkeypatch, "0", plan, cfg, fs, 7, precision)
    np.testing.assert_array_equal(a.history, b.history)
    for cid, va in a.solvers.items():
        vb = b.solvers[cid]
        for n in FIELD_NAMES:
            np.testing.assert_array_equal(va.fields[n], vb.fields[n])


def test_graph_replay_matches_oracle_3d(monkeypatch):
    monkeypatch.setenv("BF_GRAPH", "1")
    plan = planning.decompose(geometry.multiblock_box_3d(2), 4, 3)
    fs = cases.freestream_for("multiblock_box_3d", GAS, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.8)
    ref, got = run_pair(plan, cfg, fs, 6, init="perturbed", precision="fast")
    compare(ref, got, fs, bitwise=False)


@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_graph_reused_after_reupload(precision):
    """The graphs captured in a first run replay correctly after the state is
    uploaded again (buffer parity and derived-T state reset by the upload)."""
    from paper_2012_02925_b200 import stepper
    plan = planning.decompose(geometry.inlet_ramp_2d(1), 2, 2)
    fs = cases.freestream_for("inlet_ramp_2d", GAS, 2)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.5, rk_stages=1)
    gpu = stepper.GpuContext(plan, [c.id for c in plan.children], GAS, cfg, fs,
                             precision=precision)
    try:
        runs = []
        for _ in range(2):
            gpu.upload_initial("uniform")
            st = stepper.GpuRankStepper(gpu, cfg)
            hist = [st.step(k + 1)[0] for k in range(6)]
            fields = {c.id: gpu.download(c.id, "p") for c in plan.children}
            runs.append((np.array(hist), fields))
        np.testing.assert_array_equal(runs[0][0], runs[1][0])
        for cid in runs[0][1]:
            np.testing.assert_array_equal(runs[0][1][cid], runs[1][1][cid])
    finally:
        gpu.close()
