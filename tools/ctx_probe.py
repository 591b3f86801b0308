"""Times the pieces of context creation for the C4 bench workload (e2e 'blocks' phase)."""
import time, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, ctypes as C
torch.cuda.init(); torch.zeros(1, device="cuda")
from paper_2012_02925_b200 import stepper, native, cases
import bench
plan, sched, gas, cfg, fs, init = bench.build_case(15, 1)
ids = [c.id for c in plan.children]
for rep in range(3):
    setups = stepper.host_setups(plan, ids, gas, cfg, fs)
    t0 = time.perf_counter()
    g = stepper.GpuContext(plan, ids, gas, cfg, fs, precision="fast", setups=setups)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    g.finalize(); torch.cuda.synchronize(); t2 = time.perf_counter()
    g.close(); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"rep {rep}: ctx+blocks {t1-t0:.3f} s, finalize {t2-t1:.3f} s, close {t3-t2:.3f} s")
L = native.lib()
for n in (1, 2, 4):
    p = C.c_void_p()
    cr = torch.cuda.cudart()
    t0 = time.perf_counter()
    bufs = [torch.empty(int(1.15e9 // 8), dtype=torch.float64, device="cuda") for _ in range(n)]
    torch.cuda.synchronize()
    print(f"torch alloc {n} x 1.15 GB: {time.perf_counter()-t0:.3f} s")
    del bufs; torch.cuda.empty_cache()
