"""The multi-rank engine at C4 scale on ONE GPU: C4 (256^3) decomposed over N
ranks, each rank a host thread with its own context driving the NCCL code path
(grouped send/recv of the halo messages on the comm stream beside the interior
tiles, rank-ordered residual allgather) through the in-process transport
(run_distributed_gpu(..., transport="loopback")).  Reports the wall-clock solve
rate and checks the residual history against the one-rank run of the same
partition (serial driver, iterate_gpu), FAST arithmetic.

  python tools/loopback_probe.py N [--steps K]
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("nranks", type=int)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--level", type=int, default=15)
    a = ap.parse_args()
    from paper_2012_02925_b200 import cases
    from paper_2012_02925_b200.stepper import iterate_gpu, run_distributed_gpu
    plan, sched, gas, cfg, fs, init = cases.c4_box(level=a.level, np_ranks=a.nranks)
    cells = plan.grid.total_cells()
    run_distributed_gpu(plan, sched, gas, cfg, fs, max_steps=2, init=init, precision="fast")
    r = run_distributed_gpu(plan, sched, gas, cfg, fs, max_steps=a.steps, init=init,
                            precision="fast")
    ser = iterate_gpu(plan, sched, gas, cfg, fs, a.steps, init=init, precision="fast")
    same = bool(np.array_equal(r.history, ser.history))
    rel = float(np.max(np.abs(r.history - ser.history) / np.maximum(ser.history[0], 1e-300)))
    print(json.dumps({"nranks": a.nranks, "children": len(plan.children), "cells": cells,
                      "steps": r.steps, "solve_s": r.solve_seconds,
                      "mcups_wall": cells * r.steps / r.solve_seconds / 1e6,
                      "history_bitwise_vs_serial": same, "history_max_rel": rel,
                      "messages": int(sum(c.get("messages", 0) for c in r.counters.values()))
                      if isinstance(r.counters, dict) else None}))


if __name__ == "__main__":
    main()
