import sys, os, numpy as np
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
from paper_2012_02925_b200 import cases, planning
from paper_2012_02925_b200.geometry import MultiBlockGrid, make_cartesian_block, physical_patch
from paper_2012_02925_b200.model import GasModel, SchemeConfig, FIELD_NAMES
from test_gpu_parity import run_pair
GAS = GasModel()
dims = tuple(int(x) for x in sys.argv[1].split(","))
prec = sys.argv[2] if len(sys.argv) > 2 else "exact"
blk = make_cartesian_block(0, dims, (0.0, 0.0), (1.0, 0.4), 2)
d = blk.dims
grid = MultiBlockGrid(blocks=[blk], boundaries=[
    physical_patch(0, "i_min", d, "supersonic_inflow"),
    physical_patch(0, "i_max", d, "supersonic_outflow"),
    physical_patch(0, "j_min", d, "slip_wall"), physical_patch(0, "j_max", d, "slip_wall")])
plan = cases.make_plan(grid, 1)
fs = cases.freestream_for("inlet_ramp_2d", GAS, 2)
cfg = SchemeConfig(flux="van_leer", limiter="minmod", cfl=0.5)
for steps in (1, 2):
    ref, got = run_pair(plan, cfg, fs, steps, init="uniform", precision=prec)
    print("steps", steps, "hist", ref.history[-1], got.history[-1])
    for n in FIELD_NAMES:
        a = ref.solvers[0].fields[n]; b = got.solvers[0].fields[n]
        dd = np.abs(a - b)
        if dd.max() > 1e-9 * np.abs(a).max():
            print(n, dd.max(), np.argwhere(dd > 1e-9 * np.abs(a).max())[:10].tolist())
