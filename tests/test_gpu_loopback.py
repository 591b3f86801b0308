"""The NCCL code path of the multi-rank runtime, N ranks on one GPU.

`run_distributed_gpu(..., transport="loopback")` runs every rank of a plan as
a host thread driving its own context (exchange.run_distributed's structure,
exchange.py:599-682) with the in-process transport of csrc/bf_loopback.h bound
in place of libnccl.  Everything between the transport calls is the code the
NCCL ranks run: pack kernel -> grouped send/recv per remote endpoint in the
C++ order (remote_links_sorted) on the high-priority comm stream -> unpack
kernel, the interior tiles of the stage launched meanwhile and the boundary
tiles after the unpack (ev_unpacked), the per-step rank allgather of the
residual record and the rank-ordered sum.  A message paired with the wrong
endpoint has the wrong size (transport error) or the wrong data (not
bitwise), so these tests also pin the C++ message order.

Held bitwise to the serial driver (EXACT and FAST) and to the lock-step group
driver, on plans whose every rank has remote links."""

import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest

from paper_2012_02925_b200 import cases, geometry, planning
from paper_2012_02925_b200.errors import NonPhysicalStateError
from paper_2012_02925_b200.model import FIELD_NAMES, FreestreamState, GasModel, SchemeConfig

pytestmark = pytest.mark.gpu
GAS = GasModel()
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stepper():
    from paper_2012_02925_b200 import stepper
    return stepper


def assert_same_as_serial(plan, cfg, fs, steps, init, precision, gas=GAS, transport="loopback"):
    st = _stepper()
    sched = planning.reorder_boundaries(plan)
    dist = st.run_distributed_gpu(plan, sched, gas, cfg, fs, max_steps=steps, init=init,
                                  precision=precision, transport=transport)
    serial = st.iterate_gpu(plan, sched, gas, cfg, fs, steps, init=init, precision=precision)
    # the norms are rank-ordered sums of per-rank child-ordered sums
    # (exchange.py:294-309): bitwise equal to the serial id-ordered sum when
    # every rank owns one child, a re-association (~1 ulp) otherwise
    if all(len(plan.rank_children(r)) == 1 for r in range(plan.np_ranks)):
        np.testing.assert_array_equal(dist.history, serial.history)
    else:
        np.testing.assert_allclose(dist.history, serial.history, rtol=1e-15, atol=0)
    for cid, view in serial.solvers.items():
        c = plan.child(cid)
        (i0, i1), (j0, j1), (k0, k1) = c.cell_box()
        for n in FIELD_NAMES:
            np.testing.assert_array_equal(dist.fields[c.parent][n][i0:i1, j0:j1, k0:k1],
                                          view.fields[n][view.block.interior()],
                                          err_msg=f"child {cid} field {n}")
    return dist


@pytest.mark.parametrize("nranks", [2, 4, 8])
@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_loopback_box3d_matches_serial(nranks, precision):
    plan = cases.make_plan(geometry.multiblock_box_3d(3), nranks)   # aggregate at np=2
    assert all(any(plan.child(s.neighbor_block).rank != r
                   for c in plan.rank_children(r) for s in plan.boundaries[c.id]
                   if s.kind == "connected") for r in range(nranks))
    fs = cases.freestream_for("multiblock_box_3d", GAS, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.8)
    assert_same_as_serial(plan, cfg, fs, 5, "perturbed", precision)


@pytest.mark.parametrize("transport", ["loopback", "group"])
def test_transfer_counters_are_the_engines(transport):
    """DistributedResult.counters come from the engine (bf_transfer_counters):
    one concatenated message per remote endpoint and exchange, its bytes, one
    pack + one unpack launch and one wait per exchange, every send and receive
    of the group in flight — equal to native_counters' prediction."""
    plan = cases.make_plan(geometry.multiblock_box_3d(2), 4)
    fs = cases.freestream_for("multiblock_box_3d", GAS, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.8, rk_stages=2)
    dist = _stepper().run_distributed_gpu(plan, planning.reorder_boundaries(plan), GAS, cfg, fs,
                                          max_steps=3, init="perturbed", transport=transport)
    want = _stepper().native_counters(plan, rounds=1, exchanges=3 * 2)
    assert dist.counters == want
    assert all(c["messages"] > 0 and c["staging_copies"] == 0 for c in dist.counters.values())


def test_loopback_c4_level12_eight_ranks_fast():
    """C4's geometry at 128^3 cells decomposed over 8 ranks (the north-star
    np=8 plan, scaled down): 8 children of 64^3, 3 remote faces each."""
    plan, sched, gas, cfg, fs, init = cases.c4_box(level=12, np_ranks=8)
    assert_same_as_serial(plan, cfg, fs, 3, init, "fast", gas=gas)


def test_loopback_inlet_roe_rk4_exact_vs_oracle():
    """2D, several remote links per rank, Roe + RK4: bitwise vs the oracle too."""
    import oracle
    plan = planning.decompose(geometry.inlet_ramp_2d(1), 4, 2)
    sched = planning.reorder_boundaries(plan)
    fs = cases.freestream_for("inlet_ramp_2d", GAS, 2)
    cfg = SchemeConfig(flux="roe", limiter="minmod", rk_stages=4, cfl=0.5)
    dist = assert_same_as_serial(plan, cfg, fs, 6, "uniform", "exact")
    ref = oracle.iterate(plan, sched, GAS, cfg, fs, 6)
    np.testing.assert_allclose(dist.history, ref.history, rtol=1e-13, atol=0)
    for cid, s in ref.solvers.items():
        c = plan.child(cid)
        (i0, i1), (j0, j1), (k0, k1) = c.cell_box()
        for n in ("rho", "u", "v", "p"):
            np.testing.assert_array_equal(dist.fields[c.parent][n][i0:i1, j0:j1, k0:k1],
                                          s.fields[n][s.block.interior()])


def test_loopback_viscous_round2():
    """Laminar NS: ghost round 2 messages through the same transport."""
    from test_gpu_viscous import duct3d
    gas = GasModel(mu=0.2)
    plan = planning.decompose(duct3d((24, 16, 12)), 4, 3)
    fs = FreestreamState.from_mach(gas, 2.0, 1.0e5, 250.0, 0.0, 3)
    cfg = SchemeConfig(flux="roe", limiter="minmod", cfl=0.5, viscous=True)
    assert_same_as_serial(plan, cfg, fs, 4, "perturbed", "exact", gas=gas)


def test_loopback_equals_group_driver():
    plan = planning.decompose(geometry.multiblock_box_3d(2), 4, 3)
    fs = cases.freestream_for("multiblock_box_3d", GAS, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.8)
    st = _stepper()
    sched = planning.reorder_boundaries(plan)
    a = st.run_distributed_gpu(plan, sched, GAS, cfg, fs, max_steps=4, init="perturbed",
                               precision="fast", transport="loopback")
    b = st.run_distributed_gpu(plan, sched, GAS, cfg, fs, max_steps=4, init="perturbed",
                               precision="fast", transport="group")
    np.testing.assert_array_equal(a.history, b.history)
    for pid in a.fields:
        for n in FIELD_NAMES:
            np.testing.assert_array_equal(a.fields[pid][n], b.fields[pid][n])


def test_loopback_no_overlap_same_result(monkeypatch):
    """BF_NO_OVERLAP=1 runs the exchange in line (one stage launch): bitwise equal."""
    plan = planning.decompose(geometry.multiblock_box_3d(2), 4, 3)
    fs = cases.freestream_for("multiblock_box_3d", GAS, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.8)
    st = _stepper()
    sched = planning.reorder_boundaries(plan)
    a = st.run_distributed_gpu(plan, sched, GAS, cfg, fs, max_steps=3, init="perturbed",
                               precision="fast")
    monkeypatch.setenv("BF_NO_OVERLAP", "1")
    b = st.run_distributed_gpu(plan, sched, GAS, cfg, fs, max_steps=3, init="perturbed",
                               precision="fast")
    np.testing.assert_array_equal(a.history, b.history)


def test_loopback_nonphysical_error_matches_serial():
    """A CFL far too high fails on some rank: every rank returns at the same
    step (the error key travels with the residual allgather), the raised error
    is the failing rank's own reference-format message, and no rank hangs."""
    plan = planning.decompose(geometry.inlet_ramp_2d(0), 3, 2)
    sched = planning.reorder_boundaries(plan)
    fs = cases.freestream_for("inlet_ramp_2d", GAS, 2)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=50.0)
    st = _stepper()
    with pytest.raises(NonPhysicalStateError) as serial:
        st.iterate_gpu(plan, sched, GAS, cfg, fs, 20, precision="exact")
    with pytest.raises(NonPhysicalStateError) as dist:
        st.run_distributed_gpu(plan, sched, GAS, cfg, fs, max_steps=20, precision="exact")
    kind = lambda e: "CFL" in str(e) or "face state" in str(e)   # noqa: E731
    assert kind(serial.value) and kind(dist.value), (str(serial.value), str(dist.value))
    assert not str(dist.value).startswith("rank ")


TWO_PROC = textwrap.dedent("""
    import os, numpy as np, torch, torch.distributed as dist
    from paper_2012_02925_b200 import cases, geometry, planning
    from paper_2012_02925_b200.model import GasModel, SchemeConfig
    from paper_2012_02925_b200.stepper import iterate_gpu, run_distributed_gpu
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", init_method="env://")
    gas = GasModel()
    plan = cases.make_plan(geometry.multiblock_box_3d(3), 2)
    sched = planning.reorder_boundaries(plan)
    fs = cases.freestream_for("multiblock_box_3d", gas, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.8)
    d = run_distributed_gpu(plan, sched, gas, cfg, fs, max_steps=4, init="perturbed",
                            precision="fast")
    if rank == 0:
        s = iterate_gpu(plan, sched, gas, cfg, fs, 4, init="perturbed", precision="fast")
        assert np.array_equal(d.history, s.history), (d.history, s.history)
        print("NCCL2-OK")
    dist.destroy_process_group()
""")


def test_two_process_nccl_when_two_gpus(tmp_path):
    """Real NCCL between two processes (skipped on the one-GPU pool)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two visible GPUs")
    script = tmp_path / "nccl2.py"
    script.write_text(TWO_PROC)
    env = dict(os.environ, PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node=2", "--master-addr", "127.0.0.1", "--master-port",
                          "29541", str(script)], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0 and "NCCL2-OK" in out.stdout, out.stdout[-2000:] + out.stderr[-4000:]


@pytest.mark.parametrize("nranks", [2, 4])
def test_loopback_device_guards_equal_host_loop(monkeypatch, nranks):
    """Multi-rank bf_iterate batches: the rank record, its allgather and the
    history guards run on the device (rank_record / rank_guard kernels), every
    rank stops after the same step.  Against BF_BATCH=0 (host collect, host
    allgather and host guard per step): the same steps, bitwise the same norms
    and fields, a target reached mid-batch included."""
    plan = cases.make_plan(geometry.multiblock_box_3d(3), nranks)
    sched = planning.reorder_boundaries(plan)
    fs = cases.freestream_for("multiblock_box_3d", GAS, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.8)
    st = _stepper()
    monkeypatch.setenv("BF_BATCH", "0")
    probe = st.run_distributed_gpu(plan, sched, GAS, cfg, fs, max_steps=30, init="perturbed",
                                   precision="fast")
    target = float(np.max(probe.relative_history()[17]))
    runs = {}
    for batch in ("0", "1"):
        monkeypatch.setenv("BF_BATCH", batch)
        runs[batch] = st.run_distributed_gpu(plan, sched, GAS, cfg, fs, max_steps=30,
                                             residual_target=target, init="perturbed",
                                             precision="fast")
    a, b = runs["0"], runs["1"]
    assert a.steps == b.steps and a.converged == b.converged and a.steps < 30
    np.testing.assert_array_equal(a.history, b.history)
    for cid in a.fields:
        for n in a.fields[cid]:
            np.testing.assert_array_equal(a.fields[cid][n], b.fields[cid][n], err_msg=f"{cid} {n}")


def test_loopback_odd_block_sizes_tile_halo_classification():
    """A tile is interior only if its whole 2-cell halo stays off every remote
    face: with 65 cells along the cut axis the tile at i0 = 32 reads cell 65 —
    a ghost cell the unpack writes while the interior tiles run (the overlap
    path).  Bitwise equal to the serial driver (FAST, 3 steps)."""
    grid = geometry.cartesian_box_3d(130, mms=False)
    plan = planning.decompose(grid, 2, 3)
    assert any(65 in c.dims for c in plan.children), [c.dims for c in plan.children]
    fs = cases.freestream_for("multiblock_box_3d", GAS, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.8)
    assert_same_as_serial(plan, cfg, fs, 3, "perturbed", "fast")
