"""BASELINE configurations at their full sizes (SURVEY §8d C2–C4).

The CPU oracle finishes C2 (4 x 512 x 256 cells) and C3 (128^3 in 8 blocks)
in seconds per step, so those are compared with it directly.  C4 (256^3,
16.8M cells) is checked through size-independent properties:

* plan invariance: the same parent-level initial state stepped under
  `aggregate(grid, 1)` (4 blocks) and `decompose(grid, 8, 3)` (8 x 128^3) gives
  bitwise-equal interior fields in the EXACT build — the reference's own
  serial == decomposed property (tests/test_solver.py:489-512);
* freestream preservation over the farfield box;
* run-to-run determinism of the FAST build (fields and norms bitwise)."""

import numpy as np
import pytest

from paper_2012_02925_b200 import cases, planning
from paper_2012_02925_b200.model import FIELD_NAMES

from test_gpu_parity import compare, run_pair

pytestmark = pytest.mark.gpu
G = 2   # ghost depth on every stencil axis


def test_c2_full_size_vs_oracle():
    plan, sched, gas, cfg, fs, init = cases.c2_channel()
    assert plan.grid.total_cells() == 4 * 512 * 256
    ref, got = run_pair(plan, cfg, fs, 3, init=init, precision="fast", gas=gas)
    compare(ref, got, fs, bitwise=False)


def test_c3_full_size_bitwise():
    plan, sched, gas, cfg, fs, init = cases.c3_mms(128, 8)
    assert len(plan.children) == 8 and plan.grid.total_cells() == 128 ** 3
    ref, got = run_pair(plan, cfg, fs, 2, init=init, precision="exact", gas=gas)
    compare(ref, got, fs, bitwise=True)


def _parent_state(plan, gas, fs):
    """Perturbed C4 state per PARENT block (rng seeded by parent id), so every
    plan of the grid starts from the same cells."""
    out = {}
    for blk in plan.grid.blocks:
        out[blk.id] = cases.perturbed_state(blk, fs, gas, np.random.default_rng(1000 + blk.id))
    return out


def _run_plan(plan, gas, cfg, fs, parents, steps, precision):
    from paper_2012_02925_b200 import stepper
    ids = [c.id for c in plan.children]
    gpu = stepper.GpuContext(plan, ids, gas, cfg, fs, precision=precision)
    try:
        gpu.finalize()
        for c in plan.children:
            (i0, i1), (j0, j1), (k0, k1) = c.cell_box()
            pf = parents[c.parent]
            gpu.upload(c.id, [pf[n][i0:i1 + 2 * G, j0:j1 + 2 * G, k0:k1 + 2 * G]
                              for n in FIELD_NAMES])
        st = stepper.GpuRankStepper(gpu, cfg)
        hist = np.array([np.sqrt(st.step(k + 1)[0]) for k in range(steps)])
        interior = {}
        for c in plan.children:
            (i0, i1), (j0, j1), (k0, k1) = c.cell_box()
            for n in FIELD_NAMES:
                a = gpu.download(c.id, n)
                interior[(c.parent, n, i0, j0, k0)] = a[G:-G, G:-G, G:-G].copy()
        return hist, interior
    finally:
        gpu.close()


def _assemble(plan, interior):
    """Parent interiors from the children's interiors."""
    out = {}
    for blk in plan.grid.blocks:
        for n in FIELD_NAMES:
            out[(blk.id, n)] = np.empty(tuple(blk.dims))
    for (pid, n, i0, j0, k0), a in interior.items():
        out[(pid, n)][i0:i0 + a.shape[0], j0:j0 + a.shape[1], k0:k0 + a.shape[2]] = a
    return out


def test_c4_plan_invariance_exact():
    plan1, _, gas, cfg, fs, _ = cases.c4_box(15, 1)
    assert plan1.grid.total_cells() == 256 ** 3
    plan8 = planning.decompose(plan1.grid, 8, 3)
    assert len(plan8.children) == 8
    parents = _parent_state(plan1, gas, fs)
    h1, f1 = _run_plan(plan1, gas, cfg, fs, parents, 2, "exact")
    h8, f8 = _run_plan(plan8, gas, cfg, fs, parents, 2, "exact")
    a1, a8 = _assemble(plan1, f1), _assemble(plan8, f8)
    for key in a1:
        np.testing.assert_array_equal(a8[key], a1[key], err_msg=str(key))
    # Σ R² is summed per block: 4 vs 8 partial sums
    np.testing.assert_allclose(h8, h1, rtol=1e-13, atol=0)
    assert np.all(h1 > 0)


def test_c4_freestream_preserved_fast():
    from paper_2012_02925_b200.stepper import iterate_gpu
    plan, sched, gas, cfg, fs, _ = cases.c4_box(15, 1)
    res = iterate_gpu(plan, sched, gas, cfg, fs, 4, init="uniform", precision="fast")
    for view in res.solvers.values():
        inner = view.block.interior()
        for n in ("rho", "u", "v", "w", "p"):
            ref = getattr(fs, n)
            scale = max(abs(ref), abs(fs.u), 1e-300) if n in ("u", "v", "w") else abs(ref)
            err = np.abs(view.fields[n][inner] - ref).max() / scale
            assert err <= 1e-12, (n, err)


def test_c4_deterministic_fast():
    from paper_2012_02925_b200.stepper import iterate_gpu
    plan, sched, gas, cfg, fs, init = cases.c4_box(15, 1)
    a = iterate_gpu(plan, sched, gas, cfg, fs, 3, init=init, precision="fast")
    ha = a.history.copy()
    fa = {cid: v.fields["p"].copy() for cid, v in a.solvers.items()}
    del a
    b = iterate_gpu(plan, sched, gas, cfg, fs, 3, init=init, precision="fast")
    np.testing.assert_array_equal(b.history, ha)
    for cid, v in b.solvers.items():
        np.testing.assert_array_equal(v.fields["p"], fa[cid])
