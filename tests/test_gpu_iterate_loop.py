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


def _fields(res):
    from paper_2012_02925_b200.model import FIELD_NAMES
    return {cid: {n: v.fields[n].copy() for n in FIELD_NAMES} for cid, v in res.solvers.items()}


@pytest.mark.parametrize("flux", ["van_leer", "roe"])
def test_batched_loop_matches_unbatched(monkeypatch, flux):
    """bf_iterate batches graph-replayed steps with the norms and guards on the
    device (RunState, guard_kernel); a guard that fires mid-batch turns the
    rest of the batch into no-ops.  Against BF_BATCH=0 (one host round trip per
    step): same steps (a target first reached after the 256-step batch
    boundary), bitwise the same norms and padded fields (ghost layers
    included)."""
    from paper_2012_02925_b200.stepper import iterate_gpu
    plan, sched, fs = _case()
    cfg = SchemeConfig(flux=flux, limiter="van_albada", cfl=0.5)
    monkeypatch.setenv("BF_BATCH", "0")
    probe = iterate_gpu(plan, sched, GAS, cfg, fs, 400, precision="fast")
    rel = probe.history / probe.history[0]
    active = probe.history[0] > 1e-12 * probe.history[0].max()
    target = float(np.max(rel[300][active]))   # reached first at or before step 301
    runs = {}
    for batch in ("0", "1"):
        monkeypatch.setenv("BF_BATCH", batch)
        r = iterate_gpu(plan, sched, GAS, cfg, fs, 400, residual_target=target, precision="fast")
        runs[batch] = (r.history.copy(), r.steps, r.converged, _fields(r))
    (h0, s0, c0, f0), (h1, s1, c1, f1) = runs["0"], runs["1"]
    assert s0 == s1 and c0 == c1 and c0 and s0 > 256
    np.testing.assert_array_equal(h1, h0)
    for cid in f0:
        for n in f0[cid]:
            np.testing.assert_array_equal(f1[cid][n], f0[cid][n], err_msg=f"{cid} {n}")


def test_batched_loop_error_mid_batch(monkeypatch):
    """A non-physical state in the middle of a batch: the same error text as
    the per-step loop, raised after the same step."""
    from paper_2012_02925_b200.stepper import iterate_gpu
    plan, sched, fs = _case()
    cfg = SchemeConfig(flux="roe", limiter="none", rk_stages=1, cfl=3.0)
    out = {}
    for batch in ("0", "1"):
        monkeypatch.setenv("BF_BATCH", batch)
        try:
            iterate_gpu(plan, sched, GAS, cfg, fs, 200, precision="fast")
            out[batch] = None
        except Exception as exc:  # noqa: BLE001
            out[batch] = (type(exc).__name__, str(exc))
    assert out["0"] == out["1"] and out["0"] is not None
