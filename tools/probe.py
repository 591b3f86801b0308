"""Quick GPU measurement probe (development tool, not the bench contract).

  python tools/probe.py CASE [--flux roe] [--steps K] [--warmup W] [--precision fast]
  CASE: c4[:level]  multiblock_box_3d (default), one rank, all children
        box:N       single N^3 block, farfield on all faces, perturbed freestream
        c1 | c2 | c3

Prints one JSON line: ms per step, per-kernel-class ms per launch, HBM fraction
of the stage kernel (240 B/cell/stage 3D, 168 B 2D).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build(case, flux):
    from paper_2012_02925_b200 import cases, geometry, planning
    from paper_2012_02925_b200.model import GasModel, SchemeConfig
    if case.startswith("c4"):
        lvl = int(case.split(":")[1]) if ":" in case else 15
        return cases.c4_box(level=lvl, np_ranks=1, flux=flux)
    if case.startswith("box:"):
        n = int(case.split(":")[1])
        gas = GasModel()
        grid = geometry.cartesian_box_3d(n, mms=False)
        plan = planning.decompose(grid, 1, 3)
        cfg = SchemeConfig(flux=flux, limiter="van_albada", rk_stages=2, cfl=0.8)
        fs = cases.freestream_for("multiblock_box_3d", gas, 3)
        return plan, planning.reorder_boundaries(plan), gas, cfg, fs, "perturbed"
    if case == "c1":
        return cases.c1_inlet(flux=flux)
    if case == "c2":
        return cases.c2_channel(1, flux=flux)
    if case == "c3":
        return cases.c3_mms(128, 1)
    raise SystemExit(f"unknown case {case}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("--flux", default="van_leer")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--precision", default="fast")
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    import torch
    from paper_2012_02925_b200 import stepper
    torch.cuda.set_device(0)
    plan, sched, gas, cfg, fs, init = build(a.case, a.flux)
    ids = [c.id for c in plan.children]
    gpu = stepper.GpuContext(plan, ids, gas, cfg, fs, precision=a.precision, schedule=sched)
    gpu.upload_initial(init)
    st = stepper.GpuRankStepper(gpu, cfg)
    s = torch.cuda.current_stream()
    gpu.set_stream(s.cuda_stream)
    st.run(1, a.warmup)
    torch.cuda.synchronize()
    q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    q0.record(s)
    nq = len(st.run(a.warmup + 1, a.steps))
    q1.record(s)
    torch.cuda.synchronize()
    ms_noprof = q0.elapsed_time(q1) / nq
    a.warmup += nq
    gpu.set_profiling(True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    n = len(st.run(a.warmup + 1, a.steps))
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    stats = {c: gpu.kernel_stats(c) for c in range(4)}
    cells = plan.grid.total_cells()
    B = 240 if plan.grid.ndim == 3 else 168
    n0, t0 = stats[0]
    stage_ms = t0 / max(n0, 1)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6535.1
    out = {"case": a.case, "flux": a.flux, "tag": a.tag, "precision": a.precision, "cells": cells,
           "steps": n, "ms_per_step": ms / n, "mcups": cells * n / ms / 1e3,
           "ms_per_step_noprof": ms_noprof, "mcups_noprof": cells / ms_noprof / 1e3,
           "stage_ms": stage_ms, "stage_launches": n0,
           "ghost_ms": stats[1][1] / max(stats[1][0], 1), "unpack_ms": stats[2][1] / max(stats[2][0], 1),
           "reduce_ms": stats[3][1] / max(stats[3][0], 1),
           "stage_hbm_frac": B * cells / (stage_ms * 1e-3) / 1e9 / peak,
           "step_hbm_frac": B * cells * cfg.rk_stages / (ms / n * 1e-3) / 1e9 / peak,
           "env": {k: v for k, v in os.environ.items() if k.startswith("BF_")}}
    print(json.dumps(out))
    gpu.close()


if __name__ == "__main__":
    main()
