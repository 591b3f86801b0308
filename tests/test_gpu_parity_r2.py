"""Parity on the benchmarked configuration and the remaining reference behaviours
(VERDICT r1 "what's missing" 6 and "what's weak" 1):

* the FAST build (the one bench.py times) against the CPU oracle on the C4
  geometry itself at level 13 (4.2M cells in the 4 parents), 2 RK2 steps;
* a long horizon: C1 (the SPEC case) for 2000 steps against the oracle — EXACT
  bitwise; FAST |dH_k| <= 1e-12 H_1 at every step and the state within 1e-12
  of the freestream scale through step 1000 (3e-12 at step 2000, see the test);
* the C2 subsonic variant (M = 0.5, farfield ends), full size;
* the C3 order-of-accuracy study at 32^3 / 64^3 / 128^3 on 8 blocks
  (cli.py:410-434), the 128^3 case also at np = 1 (1 -> 8 blocks);
* the Roe a^2 <= 0 error (physics.py:213-217), same text as the oracle."""

import io

import numpy as np
import pytest

import oracle
from paper_2012_02925_b200 import cases, cli, geometry, planning
from paper_2012_02925_b200.errors import NonPhysicalStateError
from paper_2012_02925_b200.model import FIELD_NAMES, FreestreamState, GasModel, SchemeConfig

from test_gpu_parity import _gpu, _init_perturbed, compare, history_close, run_pair

pytestmark = pytest.mark.gpu
GAS = GasModel()


@pytest.mark.slow
def test_c4_level13_fast_vs_oracle():
    plan, sched, gas, cfg, fs, init = cases.c4_box(level=13, np_ranks=1)
    assert plan.grid.total_cells() == 4 * 1024 * 1024
    ref, got = run_pair(plan, cfg, fs, 2, init=init, precision="fast", gas=gas)
    compare(ref, got, fs, bitwise=False)


def _state_diff(blocks, got, fs):
    """max |d| / freestream scale over the interior primitives (cli.py:302-315)."""
    scale = {n: abs(getattr(fs, n)) for n in ("rho", "p", "T")}
    for n in "uvw":
        scale[n] = max(abs(fs.u), abs(fs.v), abs(fs.w))
    out = 0.0
    for cid, view in got.solvers.items():
        inner = view.block.interior()
        for n in FIELD_NAMES:
            out = max(out, float(np.max(np.abs(blocks[cid][n][inner] - view.fields[n][inner])))
                      / scale[n])
    return out


@pytest.mark.slow
def test_c1_2000_steps_vs_oracle():
    """Long horizon on the SPEC case (C1, 2000 RK2 steps; SURVEY §0 finding 5).
    EXACT: fields bitwise equal to the oracle after 1000 and 2000 steps.
    FAST: residual norms |dH_k| <= 1e-12 H_1 at every step; state within 1e-12
    of the freestream scale through step 1000.  At 2000 steps the FAST state
    sits at ~2e-12 (profiles/r02_fast_drift_c1.jsonl: a converging steady state
    amplifies the build's ulp-level residual differences J^-1 dR; every
    non-bitwise variant measured lands at 0.9-1.8e-12 there), held here to 3e-12."""
    plan, sched, gas, cfg, fs, init = cases.c1_inlet()
    blocks = oracle.build_blocks(plan, gas, cfg, fs)
    for b in blocks.values():
        b.init_uniform()
    ost = oracle.OracleStepper(blocks, oracle.make_serial_exchange(plan, sched, blocks), cfg)
    hist, snaps = [], {}
    for k in range(2000):
        hist.append(np.sqrt(ost.step(k + 1)[0]))
        if k + 1 in (1000, 2000):
            snaps[k + 1] = {cid: {n: b.fields[n].copy() for n in FIELD_NAMES}
                            for cid, b in blocks.items()}
    hist = np.array(hist)
    st = _gpu()
    for steps in (1000, 2000):
        ex = st.iterate_gpu(plan, sched, gas, cfg, fs, steps, init=init, precision="exact")
        for cid, view in ex.solvers.items():
            for n in FIELD_NAMES:
                np.testing.assert_array_equal(view.fields[n], snaps[steps][cid][n],
                                              err_msg=f"EXACT step {steps} field {n}")
        fa = st.iterate_gpu(plan, sched, gas, cfg, fs, steps, init=init, precision="fast")
        assert fa.steps == steps
        history_close(fa.history, hist[:steps], 1e-12)
        d = _state_diff(snaps[steps], fa, fs)
        assert d <= (1e-12 if steps == 1000 else 3e-12), f"FAST state after {steps}: {d:.3e}"
    # the run really moved: the mass and momentum residuals fell
    assert np.all(hist[-1][[0, 1]] < 0.2 * hist[0][[0, 1]])


@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_c2_subsonic_full_size_vs_oracle(precision):
    plan, sched, gas, cfg, fs, init = cases.c2_channel(subsonic=True)
    assert plan.grid.total_cells() == 4 * 512 * 256
    assert any(s.kind == "physical" and s.bc_type == "farfield"
               for specs in plan.boundaries.values() for s in specs)
    ref, got = run_pair(plan, cfg, fs, 3, init=init, precision=precision, gas=gas)
    compare(ref, got, fs, bitwise=False, check_q=False)


def test_c3_order_study_32_64_128_on_8_blocks():
    """cli.py:410-434 on the 3D cube split into 8 children:
    the converged L2 solution error falls at second order."""
    cfg = cli.RunConfig(case="cartesian_box", flux="roe", limiter="none", cfl=0.5,
                        max_steps=40000, residual_target=1e-7, mms_levels="32,64,128")
    buf = io.StringIO()
    out = cli.run_mms_study(cfg, cli.build_gas(cfg), buf, precision="fast", ndim=3, np_ranks=8)
    assert all(conv for _, _, _, conv in out), buf.getvalue()
    errs = [e for _, e, _, _ in out]
    orders = [np.log(a / b) / np.log(2.0) for a, b in zip(errs, errs[1:])]
    assert min(orders) > 1.9, buf.getvalue()
    # 1 -> 8 blocks: the 128^3 cube as one block and as 8 children gives the same
    # cells bitwise (FAST; every face flux has one owner, independent of the
    # tiling); the error metric itself is plan-dependent (cli.py:458 normalises
    # per block), so the fields are compared, not the errors
    from paper_2012_02925_b200.stepper import iterate_gpu
    runs = []
    for npr in (1, 8):
        plan, sched, gas, c3cfg, fs, init = cases.c3_mms(128, npr)
        r = iterate_gpu(plan, sched, gas, c3cfg, fs, 50, init=init, precision="fast")
        parent = {}
        for cid, view in r.solvers.items():
            (i0, i1), (j0, j1), (k0, k1) = plan.child(cid).cell_box()
            for n in FIELD_NAMES:
                parent.setdefault(n, np.zeros((128, 128, 128)))[i0:i1, j0:j1, k0:k1] = \
                    view.fields[n][view.block.interior()]
        runs.append(parent)
    for n in FIELD_NAMES:
        np.testing.assert_array_equal(runs[0][n], runs[1][n], err_msg=n)


def _roe_a2_state(block, fs):
    """Uniform u = 1000 m/s with p = 1e-20 in a patch of cells: the face states
    pass the positivity check but the Roe-averaged h - |u|^2/2 cancels to 0."""
    f = {n: block.allocate_field(getattr(fs, n)) for n in FIELD_NAMES}
    g = block.ghost[0]
    sl = (slice(g + 5, g + 10), slice(g + 3, g + 7), slice(None))
    f["u"][sl] = 1000.0
    f["v"][sl] = 0.0
    f["rho"][sl] = 1.0
    f["p"][sl] = 1e-20
    f["T"][sl] = f["p"][sl] / (f["rho"][sl] * GAS.R)
    return f


@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_roe_nonpositive_sound_speed_message(precision):
    grid = geometry.inlet_ramp_2d(0)
    plan = planning.decompose(grid, 1, 2)
    cfg = SchemeConfig(flux="roe", limiter="none", epsilon=0.0, cfl=0.5)
    fs = cases.freestream_for("inlet_ramp_2d", GAS, 2)
    st = _gpu()
    gpu = st.GpuContext(plan, [0], GAS, cfg, fs, precision=precision)
    gpu.finalize()
    f = _roe_a2_state(plan.child_block(0), fs)
    gpu.upload(0, [f[n] for n in FIELD_NAMES])
    with pytest.raises(NonPhysicalStateError, match="Roe-averaged state") as ei:
        st.GpuRankStepper(gpu, cfg).step(1)
    gpu.close()
    blocks = oracle.build_blocks(plan, GAS, cfg, fs)
    for n, arr in f.items():
        blocks[0].fields[n][...] = arr
    blocks[0].sync_conserved()
    sched = planning.reorder_boundaries(plan)
    ost = oracle.OracleStepper(blocks, oracle.make_serial_exchange(plan, sched, blocks), cfg)
    with pytest.raises(NonPhysicalStateError) as eo:
        ost.step(1)
    assert str(ei.value) == str(eo.value)
