"""FAST-vs-EXACT state drift on C1 over a long horizon (development probe).
Prints, at checkpoints, the max relative primitive difference (freestream
scale) and the max |dH_k|/H_1 of the FAST build against the EXACT build."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2012_02925_b200 import cases
from paper_2012_02925_b200.stepper import iterate_gpu

case = sys.argv[1] if len(sys.argv) > 1 else "c1"
checks = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "250,500,1000,2000").split(",")]
plan, sched, gas, cfg, fs, init = cases.c1_inlet() if case == "c1" else cases.c4_box(level=int(case[3:]))
scale = {n: max(abs(getattr(fs, n)), 1e-300) for n in ("rho", "p", "T")}
spd = max(abs(fs.u), abs(fs.v), abs(fs.w))
for n in "uvw": scale[n] = spd
out = {"case": case, "lib": os.environ.get("BFGPU_LIB", "default"), "rows": []}
for K in checks:
    e = iterate_gpu(plan, sched, gas, cfg, fs, K, init=init, precision="exact")
    f = iterate_gpu(plan, sched, gas, cfg, fs, K, init=init, precision="fast")
    st = 0.0; where = None
    for cid, v in e.solvers.items():
        for n in ("rho", "u", "v", "p"):
            a = v.fields[n][v.block.interior()]; b = f.solvers[cid].fields[n][v.block.interior()]
            d = np.abs(a - b) / scale[n]
            if d.max() > st:
                st = float(d.max()); where = (n, [int(x) for x in np.unravel_index(np.argmax(d), d.shape)])
    base = e.history[0]; sc = np.where(base > 1e-12 * base.max(), base, base.max())
    h = float(np.max(np.abs(f.history - e.history) / sc))
    out["rows"].append({"steps": K, "state": st, "where": where, "hist_H1": h})
print(json.dumps(out))
