import sys, os, numpy as np
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import golden_cases as gc, oracle
from paper_2012_02925_b200 import stepper as stp
from paper_2012_02925_b200.model import FIELD_NAMES
name = sys.argv[1]
desc, z = gc.load(name)
plan, sched, gas, cfg, fs = gc.build(desc)
ids = [c.id for c in plan.children]
gpu = stp.GpuContext(plan, ids, gas, cfg, fs, precision="exact", schedule=sched)
gpu.upload_initial(desc["init"])
st = stp.GpuRankStepper(gpu, cfg)
blocks = oracle.build_blocks(plan, gas, cfg, fs)
oracle.blockflow_oracle._init(blocks, desc["init"])
ost = oracle.OracleStepper(blocks, oracle.make_serial_exchange(plan, sched, blocks), cfg)
def cmp(tag):
    bad = 0
    for cid in ids:
        v = st.solvers[cid]
        v.invalidate() if hasattr(v, "invalidate") else None
        for n in FIELD_NAMES:
            got = gpu.download(cid, n); want = blocks[cid].fields[n]
            d = np.abs(got - want)
            if d.max() > 1e-9 * max(1.0, np.abs(want).max()):
                bad += 1
                print(tag, cid, n, d.max(), np.argwhere(d > 1e-9 * np.abs(want).max())[:8].tolist())
    print(tag, "bad", bad)
gpu.update_ghosts(); ost.update_ghosts(); cmp("ug0")
for k in range(2):
    st.step(k + 1); ost.step(k + 1)
    gpu.update_ghosts(); ost.update_ghosts(); cmp(f"ug{k+1}")
