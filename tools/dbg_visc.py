import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import golden_cases as gc
from paper_2012_02925_b200.stepper import iterate_gpu
from paper_2012_02925_b200.model import FIELD_NAMES
name = sys.argv[1]
desc, z = gc.load(name)
plan, sched, gas, cfg, fs = gc.build(desc)
for steps in range(1, desc["steps"] + 1):
    res = iterate_gpu(plan, sched, gas, cfg, fs, steps, init=desc["init"], precision="exact")
    print("steps", steps, "hist", res.history[-1])
cid_err = []
for cid, view in res.solvers.items():
    for n in FIELD_NAMES:
        got, want = view.fields[n], z[f"c{cid}_{n}"]
        d = np.abs(got - want)
        if d.max() > 0:
            idx = np.argwhere(d > 1e-9 * np.abs(want).max())
            print(cid, n, d.max(), len(idx), idx[:6].tolist(), view.block.dims)
