"""Time GpuContext construction (C4, pinned nodes) several times in one process."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2012_02925_b200 import cases, stepper
plan, sched, gas, cfg, fs, init = cases.c4_box(level=15)
ids = [c.id for c in plan.children]
setups = stepper.host_setups(plan, ids, gas, cfg, fs)
for cid, s in setups.items():
    buf = torch.empty(s.block.nodes.size, dtype=torch.float64, pin_memory=True).numpy()
    arr = np.ndarray(s.block.nodes.shape, dtype=np.float64, buffer=buf, order="C")
    arr[...] = s.block.nodes
    s.block.nodes = arr
torch.cuda.synchronize()
keep = stepper.GpuContext(plan, ids, gas, cfg, fs, precision="fast", setups=setups, schedule=sched)
for r in range(4):
    t = time.perf_counter()
    g = stepper.GpuContext(plan, ids, gas, cfg, fs, precision="fast", setups=setups, schedule=sched)
    dt = time.perf_counter() - t
    print("ctx", r, round(dt * 1e3, 2), "ms", {k: (round(v * 1e3, 2) if isinstance(v, float) else [round(x * 1e3, 2) for x in v]) for k, v in g.timing.items()}, flush=True)
    g.close()
