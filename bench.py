"""Benchmark: fp64 cell-updates/s (MCUPS) per RK iteration on B200.

Workload at N=1 (BASELINE.json configs[3]): multiblock_box_3d
level 15 = 256^3 cells in 4 parent blocks, one rank (aggregate -> 4 children),
Van Leer flux + Van Albada limiter, MUSCL eps=1 kappa=-1, RK2, CFL 0.8,
farfield M=0.8395, perturbed-freestream initial state.  With --gpus N>1
(torchrun, one rank per GPU, NCCL halos) the weak-scaling sweep C5 is run:
256^3 cells per GPU (level 15 + log2 N).

Printed: ONE JSON line (rank 0).  `value` = total interior cells x K RK steps
/ device time of the K steps (CUDA events on the launching stream, barrier +
synchronize on both sides, max over ranks) / 1e6.  See DESIGN.md §5 for the
roofline arithmetic and the CPU baseline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "fp64 cell-updates/sec (MCUPS) per RK iteration at 1/2/4/8 B200; % HBM roofline"
UNIT = "MCUPS"
# Algorithmic HBM bytes per interior cell per residual evaluation (RK stage),
# 3D reads W 40 + Q0 40 + 3 face vectors 72 + dt/V 8, writes Q 40 + W 40.
ALG_BYTES_3D = 240
ALG_BYTES_2D = 168


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index=0, period=0.1):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:  # noqa: BLE001
            self.nv = None
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def build_case(level, np_ranks, flux="van_leer"):
    from paper_2012_02925_b200 import cases
    return cases.c4_box(level=level, np_ranks=np_ranks, flux=flux, cfl=0.8)


def workload_config(level, nranks, ncells, precision, kc):
    return {
        "workload": ("C4 multiblock_box_3d L15 (256^3 cells), 1 GPU" if nranks == 1 else
                     f"C5 weak scaling: multiblock_box_3d L{level} ({ncells} cells, 256^3 per GPU)"),
        "grid_level": level, "cells": ncells, "ranks": nranks,
        "scheme": "van_leer flux + van_albada limiter, MUSCL eps=1 kappa=-1, RK2, CFL 0.8",
        "bcs": "farfield (M=0.8395, alpha=3.06 deg) + connected block interfaces",
        "init": "freestream with interior rho,p x (1+0.01 N(0,1)), seed 0",
        "precision": precision, "kc": kc,
        "l2": "inputs larger than L2 (device state ~4.6 GB per 256^3 cells vs 126 MB L2)",
        "parallelism": f"block decomposition over {nranks} rank(s)" + (", NCCL halos" if nranks > 1 else ""),
    }


# ---------------------------------------------------------------------------
# CPU baseline: the oracle (numpy restatement of the reference) on host cores
# ---------------------------------------------------------------------------

def cpu_sample(level=9, steps=3, threads=1):
    """MCUPS of the CPU oracle on multiblock_box_3d L`level` (bounded sample of
    the same workload: same scheme, BCs and IC).  threads>1 runs the
    reference's threaded-rank driver (exchange.run_distributed analogue)."""
    import oracle
    from paper_2012_02925_b200 import cases, planning
    plan, sched, gas, cfg, fs, _ = cases.c4_box(level=level, np_ranks=threads)
    ncells = plan.grid.total_cells()
    blocks = oracle.build_blocks(plan, gas, cfg, fs)
    rng = np.random.default_rng(0)
    for cid in sorted(blocks):
        f = cases.perturbed_state(blocks[cid].block, fs, gas, rng)
        for n, arr in f.items():
            blocks[cid].fields[n][...] = arr
        blocks[cid].sync_conserved()
    if threads == 1:
        st = oracle.OracleStepper(blocks, oracle.make_serial_exchange(plan, sched, blocks), cfg)
        st.step(1)      # warm-up
        t0 = time.perf_counter()
        c0 = os.times()
        for k in range(steps):
            st.step(k + 2)
        dt = time.perf_counter() - t0
        c1 = os.times()
    else:
        c0 = os.times()
        res = oracle.run_threaded(plan, sched, gas, cfg, fs, steps, init="perturbed", warmup=1)
        dt = res.solve_seconds
        c1 = os.times()
    busy = ((c1.user - c0.user) + (c1.system - c0.system)) / max(dt, 1e-9)
    return ncells * steps / dt / 1e6, {"cells": ncells, "steps": steps, "seconds": dt,
                                       "cores_busy": round(busy, 2)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        pass
    return "unknown"


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    nthreads = min(os.cpu_count() or 1, 8)
    level = 9
    from paper_2012_02925_b200 import cases
    plan, sched, gas, cfg, fs, _ = cases.c4_box(level=level, np_ranks=nthreads)
    ncells = plan.grid.total_cells()
    import oracle
    # set-up and warm-up steps untimed; timed steps of the threaded reference driver
    c0 = os.times()
    res = oracle.run_threaded(plan, sched, gas, cfg, fs, args.steps, init="perturbed",
                              warmup=args.warmup)
    c1 = os.times()
    dt = res.solve_seconds
    busy = ((c1.user - c0.user) + (c1.system - c0.system)) / max(c1.elapsed - c0.elapsed, 1e-9)
    value = ncells * args.steps / dt / 1e6
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(15, 1, 16777216, "numpy (reference arithmetic)", None),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "port",
                         "cores_busy": round(busy, 2),
                         "sample": f"multiblock_box_3d L{level} ({ncells} cells), {nthreads} "
                                   f"rank threads (run_distributed analogue), {args.steps} RK2 "
                                   f"steps; CPU {cpu_model()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--level", type=int, default=None)
    ap.add_argument("--precision", default="fast", choices=["fast", "exact"])
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--workload", default="c4", choices=["c1", "c2", "c3", "c4"],
                    help="c4 (default, BASELINE configs[3]) is the bench line; c1-c3 are "
                         "informational runs of the other BASELINE configs on one GPU")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    args.warmup = max(args.warmup, 3)

    import torch
    from paper_2012_02925_b200 import stepper

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://")
    else:
        torch.cuda.set_device(0)
    level = args.level if args.level is not None else 15 + int(round(math.log2(world)))
    if args.workload == "c4":
        plan, sched, gas, cfg, fs, init = build_case(level, world)
    else:
        from paper_2012_02925_b200 import cases
        if world > 1:
            raise SystemExit("--workload c1/c2/c3 are single-GPU informational runs")
        plan, sched, gas, cfg, fs, init = {"c1": cases.c1_inlet, "c2": lambda: cases.c2_channel(1),
                                           "c3": lambda: cases.c3_mms(128, 1)}[args.workload]()
        args.skip_e2e = True
    ncells = plan.grid.total_cells()
    my_children = [c.id for c in plan.rank_children(rank)]
    my_cells = sum(plan.child(c).cell_count() for c in my_children)

    t_setup = time.perf_counter()
    setups = stepper.host_setups(plan, my_children, gas, cfg, fs)
    t_setup = time.perf_counter() - t_setup
    gpu = stepper.GpuContext(plan, my_children, gas, cfg, fs, device=local, rank=rank,
                             nranks=world, precision=args.precision, setups=setups)
    if world > 1:
        import ctypes as C
        box = [None]
        if rank == 0:
            buf = (C.c_char * 128)()
            gpu._check(gpu.L.bf_nccl_unique_id(buf))
            box = [bytes(buf.raw)]
        dist.broadcast_object_list(box, src=0)
        gpu._check(gpu.L.bf_nccl_init(gpu.ctx, (C.c_char * 128).from_buffer_copy(box[0])))
    gpu.upload_initial(init)
    stream = torch.cuda.current_stream()
    gpu.set_stream(stream.cuda_stream)
    st = stepper.GpuRankStepper(gpu, cfg)

    for k in range(args.warmup):
        st.step(k + 1)
    gpu.set_profiling(True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        # the drop-in's step loop (iterate_gpu): steps driven from C, each one
        # returning its residual norms to the host
        done = len(st.run(args.warmup + 1, args.steps))
        ev1.record(stream)
        torch.cuda.synchronize()
    if done != args.steps:
        raise SystemExit(f"bench: the history guard stopped the run after {done} steps")
    if dist:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    stats = {cls: gpu.kernel_stats(cls) for cls in range(4)}
    gpu.set_profiling(False)
    value = ncells * args.steps / (ms / 1e3) / 1e6
    n_stage, ms_stage = stats[0]
    launches = sum(n for n, _ in stats.values())
    peak, peak_kind = _peaks()
    alg_bytes = (ALG_BYTES_3D if plan.grid.ndim == 3 else ALG_BYTES_2D) * my_cells
    avg_stage_s = ms_stage / max(n_stage, 1) / 1e3
    achieved = alg_bytes / avg_stage_s / 1e9
    traffic = None
    prof_path = os.path.join(ROOT, "profiles", "stage_kernel_traffic.json")
    if os.path.exists(prof_path):
        try:
            with open(prof_path) as f:
                pj = json.load(f)
            if pj.get("cells") == my_cells and pj.get("precision") == args.precision:
                traffic = pj.get("dram_bytes_per_launch")
        except Exception:  # noqa: BLE001
            traffic = None

    # e2e through the public API with host buffers (rank 0 / N=1 only)
    # the measured context is done: release it before the end-to-end run builds its own
    # (its block arenas are then recycled instead of mapped afresh by the driver)
    gpu.close()
    e2e = None
    if not args.skip_e2e:
        e2e = e2e_run(plan, my_children, gas, cfg, fs, init, local, rank, world, args, dist,
                      setups)

    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        v, info = cpu_sample(level=11, steps=3, threads=1)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"CPU oracle (numpy restatement of blockflow.solver.iterate, 1 thread) "
                         f"on multiblock_box_3d L11 ({info['cells']} cells, same scheme/BCs/IC), "
                         f"{info['steps']} timed RK2 steps after 1 warm-up, {info['seconds']:.1f} s; "
                         f"CPU {cpu_model()}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": (workload_config(level, world, ncells, args.precision, gpu_kc())
                       if args.workload == "c4" else
                       {"workload": {"c1": "C1 inlet ramp 2D 128x64, 1 block",
                                     "c2": "C2 ramp channel 2D 4 x 512x256 connected blocks",
                                     "c3": "C3 3D MMS cube 128^3 (Roe, no limiter), one block"
                                     }[args.workload] + " (informational)",
                        "cells": ncells, "precision": args.precision}),
            "residual_evals_per_s": value * 1e6 * cfg.rk_stages,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": peak_kind,
                         "kernel": "stage_kernel (fused limiter+MUSCL+flux+residual+dt+RK update)",
                         "alg_bytes_per_launch": alg_bytes,
                         "avg_launch_ms": avg_stage_s * 1e3,
                         "stage_share_of_step": ms_stage / max(ms, 1e-9)},
            "step_roofline_frac": (value * 1e6 * 2 * (ALG_BYTES_3D if plan.grid.ndim == 3 else ALG_BYTES_2D)
                                   / world / 1e9) / peak,
            "kernel_ms": {"stage": ms_stage, "ghost_fill": stats[1][1], "unpack": stats[2][1],
                          "reduce": stats[3][1]},
            "gpu_launches": launches,
            "host_setup_s": t_setup,
            "clocks": clocks.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


def gpu_kc():
    return int(os.environ.get("BF_KC", "32"))   # runtime default for the FAST Van Leer path


def e2e_run(plan, children, gas, cfg, fs, init, device, rank, world, args, dist, setups):
    """Same metric through the public API with HOST buffers: geometry and the
    initial state go host->device, every step returns its residual norms to
    the host, the final padded fields come back to the host."""
    import torch
    from paper_2012_02925_b200 import stepper
    from paper_2012_02925_b200.model import FIELD_NAMES
    import ctypes as C
    # host-side setup (metrics, IC) is the reference's excluded setup phase
    from paper_2012_02925_b200.cases import perturbed_state
    def pinned(shape, order="F", like=None):
        n = int(np.prod(shape))
        buf = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
        arr = np.ndarray(shape, dtype=np.float64, buffer=buf, order=order)
        if like is not None:
            arr[...] = like
        return arr

    rng = np.random.default_rng(0)
    host = {}
    outs = {}
    for c in sorted(plan.children, key=lambda c: c.id):
        if c.id not in setups:   # same draws as a serial run, without the arrays
            for _ in range(2):
                left = c.cell_count()
                while left > 0:
                    m = min(left, 1 << 24)
                    rng.standard_normal(m)
                    left -= m
            continue
        blk = setups[c.id].block
        f = perturbed_state(blk, fs, gas, rng)
        if c.id in setups:
            f6 = [f[n] for n in FIELD_NAMES]
            host[c.id] = [pinned(x.shape, like=x) for x in f6]
            outs[c.id] = [pinned(blk.shape) for _ in FIELD_NAMES]
    # the inputs of the run live in pinned host memory: node coordinates of every
    # owned block (the device computes the metrics), initial fields; outputs too
    setups = stepper.host_setups(plan, children, gas, cfg, fs)
    for cid, s in setups.items():
        s.block.nodes = pinned(s.block.nodes.shape, order="C", like=s.block.nodes)
    uid = None
    if world > 1:
        box = [None]
        if rank == 0:
            buf = (C.c_char * 128)()
            stepper.native.lib().bf_nccl_unique_id(buf)
            box = [bytes(buf.raw)]
        dist.broadcast_object_list(box, src=0)
        uid = (C.c_char * 128).from_buffer_copy(box[0])
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    marks = {}

    def mark(name):
        torch.cuda.synchronize()
        marks[name] = time.perf_counter()

    mark("start")
    t0 = marks["start"]
    # device registration: geometry host->device, tables, buffers
    gpu = stepper.GpuContext(plan, children, gas, cfg, fs, device=device, rank=rank,
                             nranks=world, precision=args.precision, setups=setups)
    mark("blocks")
    if uid is not None:
        gpu._check(gpu.L.bf_nccl_init(gpu.ctx, uid))
    gpu.finalize()
    mark("finalize")
    for cid, f6 in host.items():
        gpu.upload(cid, f6)      # conserved variables derived on the device
    mark("upload")
    st = stepper.GpuRankStepper(gpu, cfg)
    st.run(1, args.steps)    # each step ends with the D2H of its residual norms
    mark("steps")
    out = {cid: [gpu.download(cid, n, out=outs[cid][k]) for k, n in enumerate(FIELD_NAMES)]
           for cid in host}
    mark("download")
    dt = marks["download"] - t0
    names = list(marks)
    phases = {n: marks[n] - marks[p] for p, n in zip(names, names[1:])}
    phases["ctx_detail"] = gpu.timing
    if dist:
        t = torch.tensor([dt], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    h2d, d2h = gpu.transfer_bytes()
    gpu.close()
    del out
    ncells = plan.grid.total_cells()
    return {"value": ncells * args.steps / dt / 1e6, "unit": UNIT,
            "h2d_bytes_per_step": h2d / args.steps,
            "d2h_bytes_per_step": d2h / args.steps + 48,
            "seconds": dt,
            "phases_s": phases,
            "note": "through the public API from pinned host buffers: context creation with "
                    "the block node coordinates host->device (metrics computed on the device), "
                    "upload of the initial padded state (6 primitive fields; conserved "
                    "variables derived on the device), K RK steps "
                    "each returning its residual norms to the host, download of the 6 final "
                    "padded fields into pinned host arrays; grid generation and the initial "
                    "condition are built before the timed region (the reference's setup phase)"}


if __name__ == "__main__":
    sys.exit(main())
