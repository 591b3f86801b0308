"""Block arenas recycled across contexts (BF_ARENA_CACHE=1, bf_release_cache,
DESIGN.md §5): a context built on cached arenas (stale contents) and one built
after the cache was released give bitwise-identical runs; without the opt-in
the arenas go back to the driver when the last context of the device closes."""

import numpy as np
import pytest

from paper_2012_02925_b200 import cases, geometry, native, planning
from paper_2012_02925_b200.model import FIELD_NAMES, GasModel, SchemeConfig

pytestmark = pytest.mark.gpu


def test_recycled_arenas_do_not_leak_state(monkeypatch):
    monkeypatch.setenv("BF_ARENA_CACHE", "1")
    from paper_2012_02925_b200.stepper import iterate_gpu
    gas = GasModel()
    plan = planning.decompose(geometry.multiblock_box_3d(2), 4, 3)
    sched = planning.reorder_boundaries(plan)
    fs = cases.freestream_for("multiblock_box_3d", gas, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.8)
    runs = []
    for release in (True, False, False):
        if release:
            native.lib().bf_release_cache(-1)
        r = iterate_gpu(plan, sched, gas, cfg, fs, 3, init="perturbed", precision="exact")
        runs.append((r.history.copy(),
                     {cid: {n: v.fields[n].copy() for n in FIELD_NAMES}
                      for cid, v in r.solvers.items()}))
    for h, f in runs[1:]:
        np.testing.assert_array_equal(h, runs[0][0])
        for cid in f:
            for n in FIELD_NAMES:
                np.testing.assert_array_equal(f[cid][n], runs[0][1][cid][n])
    native.lib().bf_release_cache(-1)


def test_cache_released_with_last_context(monkeypatch):
    from paper_2012_02925_b200 import stepper
    import gc
    monkeypatch.delenv("BF_ARENA_CACHE", raising=False)
    gc.collect()                   # contexts of earlier tests (results keep them alive)
    gas = GasModel()
    plan = cases.make_plan(geometry.multiblock_box_3d(2), 1)
    sched = planning.reorder_boundaries(plan)
    fs = cases.freestream_for("multiblock_box_3d", gas, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.8)
    native.lib().bf_release_cache(-1)
    ids = [c.id for c in plan.children]
    a = stepper.GpuContext(plan, ids, gas, cfg, fs, schedule=sched)
    b = stepper.GpuContext(plan, ids, gas, cfg, fs, schedule=sched)
    a.close()                      # b still alive: a's arenas are kept for reuse
    assert native.lib().bf_cache_bytes(-1) > 0
    b.close()                      # last context of the device: handed back
    assert native.lib().bf_cache_bytes(-1) == 0
    monkeypatch.setenv("BF_ARENA_CACHE", "1")
    c = stepper.GpuContext(plan, ids, gas, cfg, fs, schedule=sched)
    c.close()
    assert native.lib().bf_cache_bytes(-1) > 0
    stepper.release_cache()
    assert native.lib().bf_cache_bytes(-1) == 0
