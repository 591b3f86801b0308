"""The N>1 host path on CPU: two processes over gloo.

Each rank steps only its own children with the CPU oracle; remote halos are
exchanged with torch.distributed point-to-point messages issued in the
NCCL-group order contract of the device runtime
(paper_2012_02925_b200.distributed.remote_links); residual sums are combined
in rank order and fields assembled per parent with the same helpers the GPU
driver uses.  The result must be bitwise identical to the serial run —
which proves the message pairing/order contract and the rank-ordered
reduction without a GPU."""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case(name):
    from paper_2012_02925_b200 import cases, geometry, planning
    from paper_2012_02925_b200.model import GasModel, SchemeConfig
    gas = GasModel()
    if name == "inlet":
        grid = geometry.inlet_ramp_2d(1)
        fs = cases.freestream_for("inlet_ramp_2d", gas, 2)
        cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.8)
        plan = planning.decompose(grid, 2, 2)
        init = "uniform"
    elif name == "annulus":     # self-connection seam split across the two ranks
        grid = geometry.c_annulus_2d(0)
        fs = cases.freestream_for("c_annulus_2d", gas, 2)
        cfg = SchemeConfig(flux="roe", limiter="minmod", cfl=0.5)
        # ring split along the wrap direction (decomp.py:602-617): the seam
        # becomes a remote link between the two ranks
        plan = planning._assemble(grid, 2, {grid.blocks[0].id: [2, 1, 1]}, None).validate()
        init = "uniform"
    else:
        grid = geometry.multiblock_box_3d(0)
        fs = cases.freestream_for("multiblock_box_3d", gas, 3)
        cfg = SchemeConfig(flux="roe", limiter="van_albada", cfl=0.5)
        plan = planning.aggregate(grid, 2)
        init = "perturbed"
    return plan, planning.reorder_boundaries(plan), gas, cfg, fs, init


def _worker(rank, world, port, name, steps, out_path):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from oracle.blockflow_oracle import FACE_NAMES, _init, _peer_spec
    from paper_2012_02925_b200 import distributed as D
    plan, sched, gas, cfg, fs, init = _case(name)
    # every rank builds all children so the perturbed IC consumes the same draws
    blocks = oracle.build_blocks(plan, gas, cfg, fs)
    _init(blocks, init)
    mine = {c.id: blocks[c.id] for c in plan.rank_children(rank)}
    order = D.remote_links(plan, rank)

    def exchange(round_no):
        # local links: direct copies (same-rank neighbours)
        for e in sched.entries(rank):
            if e.local:
                ps = _peer_spec(plan, e)
                src, dst = blocks[e.peer_child], blocks[e.child]
                bufs = oracle.pack_face(src.fields, ps, src.block.dims, src.block.ghost)
                oracle.unpack_face(bufs, dst.fields, e.spec, dst.block.dims, dst.block.ghost,
                                   FACE_NAMES.index(ps.face) % 2)
        # remote links: one message per direction, issued in the NCCL-group order
        ops, recv_bufs = [], []
        for cid, spec, peer, tag in order:
            b = blocks[cid]
            bufs = oracle.pack_face(b.fields, spec, b.block.dims, b.block.ghost)
            names = list(bufs)
            send = torch.from_numpy(np.concatenate([bufs[n] for n in names]).copy())
            recv = torch.empty_like(send)
            ops.append(dist.P2POp(dist.isend, send, peer))
            ops.append(dist.P2POp(dist.irecv, recv, peer))
            recv_bufs.append((cid, spec, names, recv))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        for cid, spec, names, recv in recv_bufs:
            b = blocks[cid]
            flat = recv.numpy()
            n = flat.size // len(names)
            got = {nm: flat[i * n:(i + 1) * n] for i, nm in enumerate(names)}
            partner = None
            for s in plan.boundaries[spec.neighbor_block]:
                if s.kind == "connected" and s.link_id == spec.link_id and s is not spec and \
                        (s.face != spec.face or s.box != spec.box or spec.neighbor_block != cid):
                    partner = s
            oracle.unpack_face(got, b.fields, spec, b.block.dims, b.block.ghost,
                               FACE_NAMES.index(partner.face) % 2)

    st = oracle.OracleStepper(mine, exchange, cfg)
    hist = []
    for k in range(steps):
        local, _ = st.step(k + 1)
        hist.append(np.sqrt(D.allgather_sum(local, dist)))
    parts = [None] * world
    dist.all_gather_object(parts, D.local_interiors(mine))
    if rank == 0:
        fields = D.assemble_parent_fields(plan, parts)
        np.savez(out_path, history=np.array(hist),
                 **{f"{pid}_{n}": v for pid, fl in fields.items() for n, v in fl.items()})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["inlet", "annulus", "box3d"])
def test_two_rank_gloo_run_matches_serial(name, tmp_path):
    sys.path.insert(0, ROOT)
    import oracle
    from paper_2012_02925_b200 import distributed as D
    out = str(tmp_path / "r.npz")
    steps = 4
    mp.start_processes(_worker, args=(2, _free_port(), name, steps, out), nprocs=2,
                       join=True, start_method="spawn")
    got = np.load(out)
    plan, sched, gas, cfg, fs, init = _case(name)
    blocks = oracle.build_blocks(plan, gas, cfg, fs)
    from oracle.blockflow_oracle import _init
    _init(blocks, init)
    st = oracle.OracleStepper(blocks, oracle.make_serial_exchange(plan, sched, blocks), cfg)
    # serial reference: per-rank partial sums combined in rank order, as the reference does
    hist = []
    for k in range(steps):
        s, _ = st.step(k + 1)
        hist.append(s)
    parts = [D.local_interiors({c.id: blocks[c.id] for c in plan.rank_children(r)})
             for r in range(plan.np_ranks)]
    fields = D.assemble_parent_fields(plan, parts)
    for pid, fl in fields.items():
        for n, v in fl.items():
            np.testing.assert_array_equal(got[f"{pid}_{n}"], v, err_msg=f"{pid} {n}")
    np.testing.assert_allclose(got["history"], np.sqrt(np.array(hist)), rtol=1e-14)


def test_remote_link_order_is_symmetric():
    """Both endpoints of every remote link see it at the same position of the
    per-peer message sequence (what NCCL group matching requires)."""
    from paper_2012_02925_b200 import cases, geometry, planning
    from paper_2012_02925_b200 import distributed as D
    for grid, npr in ((geometry.multiblock_box_3d(2), 8), (geometry.c_annulus_2d(1), 4),
                      (geometry.multiblock_box_3d(1), 3)):
        plan = cases.make_plan(grid, npr)
        seq = {}
        for r in range(plan.np_ranks):
            for cid, spec, peer, tag in D.remote_links(plan, r):
                seq.setdefault((r, peer), []).append(tag)
        for (r, peer), tags in seq.items():
            assert tags == seq[(peer, r)], (r, peer)


def test_rank_ordered_sum_matches_reference_fabric(ref):
    parts = [np.array([1e16, 1.0, -1e16, 3.0, 1e-300]), np.array([1.0, 1e16, 1e16, 2.0, 0.0]),
             np.array([-1e16, -1e16, 1.0, 1.0, 1.0])]
    fabric = ref.exchange.MessageFabric(3, timeout_s=1.0)
    import threading
    res = {}

    def go(r):
        res[r] = fabric.allreduce_sum("residual", 0, r, parts[r])
    ts = [threading.Thread(target=go, args=(r,)) for r in range(3)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    from paper_2012_02925_b200 import distributed as D
    np.testing.assert_array_equal(D.rank_ordered_sum(parts), res[0])


def test_cpp_remote_order_matches_python():
    """The C++ issue order (remote_links_sorted, exercised through
    bf_probe_remote_order on the endpoints in GpuContext's bf_add_link order)
    equals distributed.remote_links — the order the gloo runs above use."""
    import ctypes as C
    from paper_2012_02925_b200 import cases, geometry, native
    from paper_2012_02925_b200 import distributed as D
    L = native.lib()
    for grid, npr in ((geometry.multiblock_box_3d(2), 8), (geometry.c_annulus_2d(1), 4),
                      (geometry.multiblock_box_3d(1), 3), (geometry.multiblock_box_3d(3), 2)):
        plan = cases.make_plan(grid, npr)
        for r in range(plan.np_ranks):
            added = []   # (cid, spec, peer_rank, tag) in bf_add_link call order
            for c in sorted(plan.rank_children(r), key=lambda c: c.id):
                for s in plan.boundaries[c.id]:
                    if s.kind == "connected" and plan.child(s.neighbor_block).rank != r:
                        added.append((c.id, s, plan.child(s.neighbor_block).rank,
                                      int(s.link_id)))
            n = len(added)
            out = (C.c_int * max(n, 1))()
            assert L.bf_probe_remote_order(n, native.ints([a[2] for a in added]),
                                           native.ints([a[3] for a in added]),
                                           native.ints([a[0] for a in added]), out) == 0
            got = [(added[out[q]][0], added[out[q]][2], added[out[q]][3]) for q in range(n)]
            want = [(cid, peer, tag) for cid, _, peer, tag in D.remote_links(plan, r)]
            assert got == want, (r, got, want)
