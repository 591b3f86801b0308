"""The NCCL code path on the one GPU this pool provides.

`run_distributed_gpu` under an initialised torch.distributed NCCL group (a
1-rank world here, in a subprocess so the test process stays uninitialised):
bf_nccl_unique_id / bf_nccl_init (dlopen'ed NCCL), the per-step rank
allgather of the residual sums and the all_gather_object field assembly.
Its history and fields must equal the serial driver's bitwise (EXACT).  The
N>1 exchange itself is covered by the in-process group tests on one GPU and
by the gloo tests of the message order (NCCL refuses two ranks on one device)."""

import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent("""
    import numpy as np, torch, torch.distributed as dist
    from paper_2012_02925_b200 import cases, geometry, planning
    from paper_2012_02925_b200.model import GasModel, SchemeConfig
    from paper_2012_02925_b200.stepper import iterate_gpu, run_distributed_gpu
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method="env://")
    gas = GasModel()
    plan = planning.aggregate(geometry.multiblock_box_3d(2), 1)
    sched = planning.reorder_boundaries(plan)
    fs = cases.freestream_for("multiblock_box_3d", gas, 3)
    cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.8)
    d = run_distributed_gpu(plan, sched, gas, cfg, fs, max_steps=4, init="perturbed",
                            precision="exact")
    s = iterate_gpu(plan, sched, gas, cfg, fs, 4, init="perturbed", precision="exact")
    assert np.array_equal(d.history, s.history), (d.history, s.history)
    for cid, view in s.solvers.items():
        c = plan.child(cid)
        (i0, i1), (j0, j1), (k0, k1) = c.cell_box()
        for n in ("rho", "u", "v", "w", "p"):
            a = d.fields[c.parent][n][i0:i1, j0:j1, k0:k1]
            b = view.fields[n][view.block.interior()]
            assert np.array_equal(a, b), (cid, n)
    dist.destroy_process_group()
    print("NCCL-OK")
""")


def test_run_distributed_gpu_nccl_one_rank(tmp_path):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", WORLD_SIZE="1",
               RANK="0", LOCAL_RANK="0", PYTHONPATH=ROOT)
    script = tmp_path / "nccl_one_rank.py"
    script.write_text(SCRIPT)
    out = subprocess.run([sys.executable, str(script)], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and "NCCL-OK" in out.stdout, out.stdout[-2000:] + out.stderr[-4000:]


SCRIPT_N = textwrap.dedent("""
    import os, numpy as np, torch, torch.distributed as dist
    from paper_2012_02925_b200 import cases, geometry, planning
    from paper_2012_02925_b200.model import GasModel, SchemeConfig
    from paper_2012_02925_b200.stepper import iterate_gpu, run_distributed_gpu
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", init_method="env://")
    gas = GasModel()
    plan = cases.make_plan(geometry.multiblock_box_3d(3), world)
    sched = planning.reorder_boundaries(plan)
    fs = cases.freestream_for("multiblock_box_3d", gas, 3)
    for prec in ("exact", "fast"):
        cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.8)
        d = run_distributed_gpu(plan, sched, gas, cfg, fs, max_steps=5, init="perturbed",
                                precision=prec)
        # every rank has the same rank-ordered norms and the whole assembled field
        if rank == 0:
            s = iterate_gpu(plan, sched, gas, cfg, fs, 5, init="perturbed", precision=prec,
                            device=int(os.environ["LOCAL_RANK"]))
            np.testing.assert_allclose(d.history, s.history, rtol=1e-15, atol=0)
            for cid, view in s.solvers.items():
                c = plan.child(cid)
                (i0, i1), (j0, j1), (k0, k1) = c.cell_box()
                for n in ("rho", "u", "v", "w", "p"):
                    assert np.array_equal(d.fields[c.parent][n][i0:i1, j0:j1, k0:k1],
                                          view.fields[n][view.block.interior()]), (prec, cid, n)
            assert all(cnt["messages"] > 0 for cnt in d.counters.values()), d.counters
    dist.destroy_process_group()
    if rank == 0:
        print("NCCL-N-OK")
""")


def _gpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_run_distributed_gpu_nccl_multi_rank(tmp_path, nranks):
    """One process per GPU over NCCL (needs >= nranks visible GPUs; this pool's
    calls have one, the driver's scaling box has eight): halos as grouped NCCL
    send/recv with the interior tiles overlapped, bitwise equal to the serial
    driver on rank 0's device."""
    if _gpus() < nranks:
        pytest.skip(f"needs {nranks} GPUs, {_gpus()} visible")
    script = tmp_path / "nccl_n.py"
    script.write_text(SCRIPT_N)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nranks}", "--master-addr", "127.0.0.1", "--master-port",
           str(29540 + nranks), str(script)]
    out = subprocess.run(cmd, cwd=ROOT, env=dict(os.environ, PYTHONPATH=ROOT),
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0 and "NCCL-N-OK" in out.stdout, out.stdout[-2000:] + out.stderr[-4000:]
