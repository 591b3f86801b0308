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
