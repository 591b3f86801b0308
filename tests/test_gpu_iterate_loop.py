"""iterate_gpu drives the step loop from C (bf_iterate) with the history
guards of solver.py:836-855 evaluated after every step.  Against the per-step
Python loop (GpuRankStepper.step + check_history_guards): the same steps, the
same norms, the same convergence flag, the same DivergenceError."""

import numpy as np
import pytest

from paper_2012_02925_b200 import cases, geometry, planning
from paper_2012_02925_b200.model import GasModel, SchemeConfig

pytestmark = pytest.mark.gpu
GAS = GasModel()


def _python_loop(plan, cfg, fs, max_steps, target=None, floor=None, init="uniform"):
    from paper_2012_02925_b200 import stepper as S
    gpu = S.GpuContext(plan, [c.id for c in plan.children], GAS, cfg, fs, precision="fast")
    try:
        gpu.upload_initial(init)
        st = S.GpuRankStepper(gpu, cfg)
        hist, conv = [], False
        for k in range(max_steps):
            hist.append(S.residual_norms(st.step(k + 1)[0]))
            if S.check_history_guards(hist, k, target, residual_floor=floor):
                conv = True
                break
        return np.array(hist), conv
    finally:
        gpu.close()


def _case():
    plan = planning.decompose(geometry.inlet_ramp_2d(1), 2, 2)
    return plan, planning.reorder_boundaries(plan), cases.freestream_for("inlet_ramp_2d", GAS, 2)


@pytest.mark.parametrize("target,floor", [(None, None), (0.5, None), (None, 1e30), (1e-30, None)])
def test_c_loop_matches_python_loop(target, floor):
    from paper_2012_02925_b200.stepper import iterate_gpu
    plan, sched, fs = _case()
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.5)
    ref_h, ref_c = _python_loop(plan, cfg, fs, 40, target, floor)
    got = iterate_gpu(plan, sched, GAS, cfg, fs, 40, residual_target=target,
                      residual_floor=floor, precision="fast")
    np.testing.assert_array_equal(got.history, ref_h)
    assert got.converged == ref_c and got.steps == len(ref_h)


def test_c_loop_divergence_raises_like_python_loop():
    from paper_2012_02925_b200.stepper import iterate_gpu
    plan, sched, fs = _case()
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=50.0)
    msgs = []
    for run in ("python", "c"):
        try:
            if run == "python":
                _python_loop(plan, cfg, fs, 30)
            else:
                iterate_gpu(plan, sched, GAS, cfg, fs, 30, precision="fast")
            msgs.append(None)
        except Exception as exc:  # noqa: BLE001 - same type and text on both paths
            msgs.append((type(exc).__name__, str(exc)))
    assert msgs[0] == msgs[1]
    assert msgs[0] is not None
