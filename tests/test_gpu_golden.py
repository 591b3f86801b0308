"""Device path vs the reference's golden vectors (no reference needed).

EXACT build: fields, conserved variables and frozen limiter arrays bitwise
equal to the reference wherever the path avoids libm pow, residual norms to
1e-13 (the device sums R^2 per tile, numpy pairwise); farfield cases within
1e-12.  FAST build: within the 1e-12 bar on every case."""

import numpy as np
import pytest

import golden_cases as gc
from paper_2012_02925_b200.model import FIELD_NAMES

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision", ["exact", "fast", "auto"])
@pytest.mark.parametrize("name", gc.names())
def test_gpu_matches_reference_golden(name, precision):
    from paper_2012_02925_b200.stepper import iterate_gpu, resolve_precision
    desc, z = gc.load(name)
    plan, sched, gas, cfg, fs = gc.build(desc)
    if precision == "fast" and cfg.limiter_freeze_at:
        pytest.skip("fast arithmetic + frozen limiters is outside the 1e-12 bar (DESIGN.md §4); "
                    "'auto' runs such cases in exact arithmetic")
    precision = resolve_precision(precision, cfg)
    res = iterate_gpu(plan, sched, gas, cfg, fs, desc["steps"], init=desc["init"],
                      precision=precision)
    bitwise = precision == "exact" and gc.bitwise_case(desc)
    if bitwise:
        np.testing.assert_allclose(res.history, z["history"], rtol=1e-13, atol=0)
    else:
        assert gc.history_ok(res.history, z["history"])
    for cid, view in res.solvers.items():
        for n in FIELD_NAMES:
            got, want = view.fields[n], z[f"c{cid}_{n}"]
            if bitwise:
                np.testing.assert_array_equal(got, want, err_msg=f"child {cid} {n}")
            else:
                assert gc.field_err(got, want, fs, n) <= 1e-12, (cid, n)
        if bitwise:
            for e in range(5):
                np.testing.assert_array_equal(view.q[e], z[f"c{cid}_q{e}"])
            if cfg.limiter_freeze_at:
                for d in view.dirs:
                    np.testing.assert_array_equal(view.psi[d][0], z[f"c{cid}_psi{d}_plus"])
                    np.testing.assert_array_equal(view.psi[d][1], z[f"c{cid}_psi{d}_minus"])
