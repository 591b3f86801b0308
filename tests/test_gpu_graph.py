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
