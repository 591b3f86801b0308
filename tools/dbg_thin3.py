import sys, os, numpy as np
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
from paper_2012_02925_b200 import cases
from paper_2012_02925_b200.model import GasModel, SchemeConfig, FIELD_NAMES, FreestreamState
from test_gpu_parity import run_pair
from test_gpu_vl_split import channel_3d
GAS = GasModel()
dims = tuple(int(x) for x in sys.argv[1].split(","))
prec = sys.argv[2]
grid = channel_3d(dims=dims, kwall="slip_wall")
plan = cases.make_plan(grid, 1)
fs = FreestreamState.from_mach(GAS, 2.5, 50000.0, 250.0, 4.0, 3)
cfg = SchemeConfig(flux="van_leer", limiter="van_albada", cfl=0.5)
for steps in (1, 2):
    ref, got = run_pair(plan, cfg, fs, steps, init="perturbed", precision=prec)
    print("steps", steps, "hist", np.max(np.abs(ref.history - got.history) / ref.history[0]))
    blk = got.solvers[0].block
    for n in FIELD_NAMES:
        a = ref.solvers[0].fields[n]; b = got.solvers[0].fields[n]
        dd = np.abs(a - b)
        if dd.max() > 1e-9 * np.abs(a).max():
            idx = np.argwhere(dd > 1e-9 * np.abs(a).max())
            print(n, dd.max(), len(idx), idx[:8].tolist(), "shape", a.shape)
