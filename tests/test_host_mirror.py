"""The host-side mirrors (geometry, planning, topology, MMS, model) against
the reference package itself, bitwise (skipped where the reference is not
installed; the golden-vector tests cover that case)."""

import numpy as np
import pytest

from paper_2012_02925_b200 import geometry, mms, planning
from paper_2012_02925_b200.model import FreestreamState, GasModel
from paper_2012_02925_b200.topology import halo_regions

PRESETS = [("inlet_ramp_2d", 0), ("inlet_ramp_2d", 1), ("c_annulus_2d", 0), ("c_annulus_2d", 1),
           ("multiblock_box_3d", 0), ("multiblock_box_3d", 2), ("cartesian_box", 2)]


@pytest.mark.parametrize("case,level", PRESETS)
def test_grids_and_metrics_bitwise(ref, case, level):
    g_ref = ref.mesh.generate_case_grid(case, level)
    g_me = geometry.generate_case_grid(case, level)
    assert len(g_ref.blocks) == len(g_me.blocks)
    for b1, b2 in zip(g_ref.blocks, g_me.blocks):
        assert b1.dims == b2.dims and b1.ghost == b2.ghost
        np.testing.assert_array_equal(b1.nodes, b2.nodes)
        m1, m2 = ref.mesh.compute_metrics(b1), geometry.compute_metrics(b2)
        np.testing.assert_array_equal(m1.volume, m2.volume)
        np.testing.assert_array_equal(m1.centers, m2.centers)
        for d in range(b1.ndim):
            np.testing.assert_array_equal(m1.face_vectors[d], m2.face_vectors[d])
    key = lambda s: (s.kind, s.block, s.face, s.box, s.bc_type, s.neighbor_block,
                     s.neighbor_face, s.neighbor_box, s.axis_map, s.link_id)
    assert [key(s) for s in g_ref.boundaries] == [key(s) for s in g_me.boundaries]


@pytest.mark.parametrize("case,level,npr", [
    ("inlet_ramp_2d", 1, 1), ("inlet_ramp_2d", 1, 4), ("c_annulus_2d", 1, 3),
    ("multiblock_box_3d", 0, 1), ("multiblock_box_3d", 0, 2), ("multiblock_box_3d", 0, 3),
    ("multiblock_box_3d", 1, 4), ("multiblock_box_3d", 2, 8), ("multiblock_box_3d", 3, 6),
    ("multiblock_box_3d", 15, 1), ("multiblock_box_3d", 15, 8)])
def test_plans_and_schedules_equal(ref, case, level, npr):
    g_ref = ref.mesh.generate_case_grid(case, level)
    g_me = geometry.generate_case_grid(case, level)
    mk_ref = ref.decomp.aggregate if npr < g_ref.parent_count else \
        (lambda g, n: ref.decomp.decompose(g, n, g.ndim))
    mk_me = planning.aggregate if npr < g_me.parent_count else \
        (lambda g, n: planning.decompose(g, n, g.ndim))
    p1, p2 = mk_ref(g_ref, npr), mk_me(g_me, npr)
    d1, d2 = ref.decomp.plan_to_dict(p1), planning.plan_summary(p2)
    assert d1["children"] == d2["children"]
    assert d1["boundaries"] == d2["boundaries"]
    s1, s2 = ref.decomp.reorder_boundaries(p1), planning.reorder_boundaries(p2)
    for r in range(npr):
        e1 = [(e.child, e.peer_rank, e.peer_child, e.tag, e.local) for e in s1.entries(r)]
        e2 = [(e.child, e.peer_rank, e.peer_child, e.tag, e.local) for e in s2.entries(r)]
        assert e1 == e2
    if level < 10:
        for cid in range(len(p1.children)):
            np.testing.assert_array_equal(p1.child_block(cid).nodes, p2.child_block(cid).nodes)
            for s in p2.boundaries[cid]:
                if s.kind == "connected":
                    rs = [x for x in p1.boundaries[cid] if x.link_id == s.link_id and
                          x.face == s.face and x.box == s.box][0]
                    blk = p2.child_block(cid)
                    for rnd in (1, 2):
                        assert halo_regions(s, blk.dims, blk.ghost, rnd) == \
                            ref.topology.halo_regions(rs, blk.dims, blk.ghost, rnd)


def test_freestream_and_gas(ref):
    for args in ((4.0, 12270.0, 217.0, 0.0, 2), (0.8395, 315979.763, 255.556, 3.06, 3),
                 (0.25, 84307.0, 300.0, 5.0, 2)):
        a = ref.solver.FreestreamState.from_mach(ref.physics.GasModel(), *args)
        b = FreestreamState.from_mach(GasModel(), *args)
        assert a.values() == b.values()


@pytest.mark.parametrize("ms_id", ["constant", "euler_2d", "ns_2d"])
def test_mms_bitwise(ref, ms_id):
    rng = np.random.default_rng(4)
    x, y = rng.random(200), rng.random(200)
    z = np.zeros_like(x)
    s1 = ref.physics.manufactured_solution(ms_id)
    s2 = mms.manufactured_solution(ms_id)
    for n in ("rho", "u", "v", "w", "p"):
        np.testing.assert_array_equal(s1[n](x, y, z), s2[n](x, y, z))
    gas_r = ref.physics.GasModel(mu=1.8e-5)
    gas_m = GasModel(mu=1.8e-5)
    for a, b in zip(ref.physics.mms_source(x, y, z, ms_id, gas_r),
                    mms.mms_source(x, y, z, ms_id, gas_m)):
        np.testing.assert_array_equal(a, b)


def test_oracle_equals_reference_iterate_random_schemes(ref):
    """A few extra scheme combinations straight against blockflow.solver.iterate."""
    import oracle
    rng = np.random.default_rng(11)
    gas_r, gas_m = ref.physics.GasModel(), GasModel()
    for trial in range(4):
        flux = ["roe", "van_leer"][trial % 2]
        lim = ["none", "van_leer", "van_albada", "minmod"][trial]
        kappa = float(rng.choice([-1.0, 0.0, 1.0 / 3.0]))
        rk = [1, 2, 4, 2][trial]
        cfg_r = ref.solver.SchemeConfig(flux=flux, limiter=lim, kappa=kappa, rk_stages=rk, cfl=0.5)
        from paper_2012_02925_b200.model import SchemeConfig
        cfg_m = SchemeConfig(flux=flux, limiter=lim, kappa=kappa, rk_stages=rk, cfl=0.5)
        g1 = ref.mesh.generate_case_grid("inlet_ramp_2d", 0)
        g2 = geometry.generate_case_grid("inlet_ramp_2d", 0)
        p1, p2 = ref.decomp.decompose(g1, 2, 2), planning.decompose(g2, 2, 2)
        fs_r = ref.solver.FreestreamState.from_mach(gas_r, 4.0, 12270.0, 217.0, 0.0, 2)
        fs_m = FreestreamState.from_mach(gas_m, 4.0, 12270.0, 217.0, 0.0, 2)
        try:
            r1 = ref.solver.iterate(p1, ref.decomp.reorder_boundaries(p1), gas_r, cfg_r, fs_r, 4)
        except Exception as exc:  # noqa: BLE001
            with pytest.raises(type(exc).__bases__[0]):
                oracle.iterate(p2, planning.reorder_boundaries(p2), gas_m, cfg_m, fs_m, 4)
            continue
        r2 = oracle.iterate(p2, planning.reorder_boundaries(p2), gas_m, cfg_m, fs_m, 4)
        np.testing.assert_array_equal(r1.history, r2.history)
        for cid in r1.solvers:
            for n in ("rho", "u", "v", "w", "p", "T"):
                np.testing.assert_array_equal(r1.solvers[cid].fields[n], r2.solvers[cid].fields[n])


@pytest.mark.parametrize("case,level", [("c_annulus_2d", 1), ("multiblock_box_3d", 1)])
def test_face_gradient_matrices_bitwise(ref, case, level):
    """geometry.face_gradient_matrix (viscous setup uploaded to the device) and the
    oracle's restatement vs BlockSolver._grad_invT (solver.py:582-642)."""
    import oracle
    g_ref = ref.mesh.generate_case_grid(case, level)
    g_me = geometry.generate_case_grid(case, level)
    gas = ref.physics.GasModel(mu=1.8e-5)
    cfg = ref.solver.SchemeConfig(viscous=True)
    fs = ref.solver.FreestreamState.from_mach(gas, 0.5, 1e5, 300.0, 0.0, g_ref.ndim)
    for b1, b2 in zip(g_ref.blocks, g_me.blocks):
        specs = g_ref.block_boundaries(b1.id)
        s = ref.solver.BlockSolver(b1, specs, gas, cfg, fs)
        m2 = geometry.compute_metrics(b2)
        ob = oracle.blockflow_oracle.OracleBlock(b2, g_me.block_boundaries(b2.id), m2,
                                                 GasModel(mu=1.8e-5), cfg, fs)
        for d in range(b1.ndim):
            np.testing.assert_array_equal(geometry.face_gradient_matrix(b2, m2, d),
                                          s._grad_invT[d])
            np.testing.assert_array_equal(ob.grad_invT[d], s._grad_invT[d])
