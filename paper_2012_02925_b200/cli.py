"""`blockflow run` on the device.

    python -m paper_2012_02925_b200.cli run config.txt [--np N] [--output-dir D]
                                        [--compare-serial] [--precision auto|exact|fast]

The configuration is parsed by the reference's own runner code (blockflow.cli
RunConfig / parse_config, loaded from baseline/_ref: every key, default,
coercion and error text is the reference's), same artefacts (cli.py:365-390):
``residuals.csv`` (relative history), ``counters.json`` (per-rank transfer
counters of the native engine as it ran, bf_transfer_counters),
``plan.json`` (decomposition + schedule), ``block_<id>.vtk`` / ``.npy``
solutions, and the same summary line.  The solve runs through
``run_distributed_gpu``: one process per GPU over NCCL under torchrun, else
every rank as a context of the in-process group on the visible devices.
``mms_levels`` runs the order-of-accuracy study on the device (cli.py:410-434);
scaling studies are bench.py's (``--gpus N`` under torchrun).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from dataclasses import replace

import numpy as np

from . import geometry, planning
from .errors import BlockflowError, ConfigError, bridged
from .model import FIELD_NAMES, FreestreamState, GasModel, SchemeConfig

EXIT_OK, EXIT_ERROR, EXIT_CONFIG = 0, 1, 2


def _ref_cli():
    """The reference's own run-config schema and parser (blockflow.cli:
    RunConfig cli.py:50-116, CASE_TABLES cli.py:34-44, parse_config
    cli.py:145-179), consumed as they are: keys, defaults, coercions and error
    texts are the reference's by construction."""
    from . import reference
    return reference.load("cli")


def __getattr__(name):
    if name in ("RunConfig", "CASE_TABLES"):
        return getattr(_ref_cli(), name)
    raise AttributeError(name)


def validated(cfg):
    """cfg.validate() (the reference's RunConfig.validate, cli.py:90-107) with
    its ConfigError re-raised as this package's."""
    rc = _ref_cli()
    try:
        cfg = cfg.validate()
    except rc.ConfigError as e:
        raise bridged(ConfigError)(str(e)) from None
    if cfg.case == "deadlock_demo":
        raise bridged(ConfigError)("deadlock_demo exercises the reference's simulated MPI "
                                   "fabric (out of scope for the device runner)")
    return cfg


def parse_config(source):
    """blockflow.cli.parse_config; its ConfigError is re-raised as this
    package's (bridged to the reference's class)."""
    rc = _ref_cli()
    try:
        return rc.parse_config(source)
    except rc.ConfigError as e:
        raise bridged(ConfigError)(str(e)) from None


# ---- case assembly (cli.py:182-247) -----------------------------------------------

def build_gas(cfg):
    return GasModel(mu=cfg.mu if cfg.physics == "laminar_ns" else 0.0, prandtl=cfg.prandtl)


def build_grid(cfg):
    if cfg.grid_file is not None:
        raise ConfigError("grid_file runs: load the grid with blockflow.mesh.load_grid and "
                          "call stepper.run_distributed_gpu (the device runner reads presets)")
    grid = geometry.generate_case_grid(cfg.case, cfg.level)
    if cfg.case == "c_annulus_2d" and cfg.physics == "laminar_ns":
        grid.boundaries = [s if not (s.kind == "physical" and s.bc_type == "slip_wall")
                           else replace(s, bc_type="noslip_wall") for s in grid.boundaries]
    return grid


def build_freestream(cfg, gas, ndim):
    tables = _ref_cli().CASE_TABLES
    table = dict(tables.get(cfg.case or "", tables["cartesian_box"]))
    for key in ("mach", "pressure", "temperature", "alpha_deg"):
        if getattr(cfg, key) is not None:
            table[key] = getattr(cfg, key)
    return FreestreamState.from_mach(gas, table["mach"], table["pressure"],
                                     table["temperature"], table["alpha_deg"], ndim)


def build_scheme(cfg):
    return SchemeConfig(flux=cfg.flux, epsilon=cfg.epsilon, kappa=cfg.kappa,
                        limiter=cfg.limiter, rk_stages=cfg.rk_stages, cfl=cfg.cfl,
                        limiter_freeze_at=cfg.limiter_freeze_at,
                        entropy_fix_coeff=cfg.entropy_fix_coeff,
                        viscous=(cfg.physics == "laminar_ns"),
                        wall_temperature=cfg.wall_temperature)


STRATEGY_VALUES = (("granularity", ("sliced", "packed")), ("buffers", ("transient", "persistent")),
                   ("transport", ("staged", "direct")), ("wait_policy", ("per_block", "deferred_all")))


def check_strategy(cfg):
    """exchange.py:56-70 validation.  The native engine always runs packed,
    persistent, direct, deferred (the paper's optimised configuration), so the
    values are checked and reported, not switched."""
    for name, allowed in STRATEGY_VALUES:
        value = getattr(cfg, name)
        if value not in allowed:
            raise ConfigError(f"{name} must be one of {allowed}, got {value!r}")


def build_plan(cfg, grid):
    split = cfg.split_dims if cfg.split_dims is not None else grid.ndim
    if cfg.aggregation or cfg.np < grid.parent_count:
        return planning.aggregate(grid, cfg.np)
    return planning.decompose(grid, cfg.np, split)


# ---- writers (cli.py:250-289, decomp.py:620-654, exchange.py:116-119) -------------

def plan_to_dict(plan, schedule=None):
    out = planning.plan_summary(plan)
    out["aggregated"] = bool(getattr(plan, "aggregated", False))
    out["parents"] = [{"id": b.id, "dims": list(b.dims)} for b in plan.grid.blocks]
    out = {k: out[k] for k in ("np", "aggregated", "parents", "children", "boundaries")}
    if schedule is not None:
        out["schedule"] = {
            "reordered": schedule.reordered,
            "order": {str(r): [{"child": e.child, "tag": e.tag, "local": e.local,
                                "peer_rank": e.peer_rank} for e in entries]
                      for r, entries in sorted(schedule.per_rank.items())}}
    return out


def counters_to_json(counters):
    return json.dumps([{"rank": r, **counters[r]} for r in sorted(counters)], indent=2)


def write_solution_vtk(path, block, fields):
    """Legacy structured-grid file of one block: nodes, rho/p/T, velocity."""
    ni, nj, nk = block.dims
    g = block.ghost_depth
    if block.ndim == 2:
        xs = block.nodes[0][g:g + ni + 1, g:g + nj + 1]
        ys = block.nodes[1][g:g + ni + 1, g:g + nj + 1]
        zs = np.zeros_like(xs)
        dims = (ni + 1, nj + 1, 1)
    else:
        cut = tuple(slice(g, g + n + 1) for n in block.dims)
        xs, ys, zs = (block.nodes[c][cut] for c in range(3))
        dims = (ni + 1, nj + 1, nk + 1)
    npts = int(np.prod(dims))
    lines = ["# vtk DataFile Version 3.0", f"blockflow solution block {block.id}", "ASCII",
             "DATASET STRUCTURED_GRID", f"DIMENSIONS {dims[0]} {dims[1]} {dims[2]}",
             f"POINTS {npts} double"]
    lines += [f"{x!r} {y!r} {z!r}" for x, y, z in zip(xs.ravel(order="F"), ys.ravel(order="F"),
                                                      zs.ravel(order="F"))]
    lines.append(f"CELL_DATA {ni * nj * nk}")
    for name in ("rho", "p", "T"):
        lines += [f"SCALARS {name} double 1", "LOOKUP_TABLE default"]
        lines += [repr(v) for v in fields[name].ravel(order="F")]
    lines.append("VECTORS velocity double")
    lines += [f"{u!r} {v!r} {w!r}" for u, v, w in zip(fields["u"].ravel(order="F"),
                                                      fields["v"].ravel(order="F"),
                                                      fields["w"].ravel(order="F"))]
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


def write_solution_npy(path, fields):
    np.save(path, np.stack([fields[n] for n in FIELD_NAMES]))


def max_rel_primitive_diff(fields_a, fields_b, fs):
    """cli.py:302-315: max |a - b| / freestream reference over blocks and fields."""
    vmag = float(np.sqrt(fs.u ** 2 + fs.v ** 2 + fs.w ** 2)) or 1.0
    refs = {"rho": abs(fs.rho), "u": vmag, "v": vmag, "w": vmag, "p": abs(fs.p), "T": abs(fs.T)}
    worst = 0.0
    for bid in fields_a:
        for n, ref in refs.items():
            worst = max(worst, float(np.max(np.abs(fields_a[bid][n] - fields_b[bid][n])) / ref))
    return worst


# ---- run (cli.py:318-407) ---------------------------------------------------------

def mms_solution_error(result):
    """cli.py:447-461: RMS over blocks and cells of the primitive-variable error
    relative to the manufactured fields (rho, u, v, p)."""
    from . import mms
    err2, count = 0.0, 0
    for s in result.solvers.values():
        sol = mms.manufactured_solution(s.config.mms_id)
        c = s.metrics.centers
        cut = s.block.interior()
        x, y, z = (c[i][cut] for i in range(3))
        for name in ("rho", "u", "v", "p"):
            exact = sol[name](x, y, z)
            e = (s.fields[name][cut] - exact) / np.abs(exact).max()
            err2 += float(np.sum(e * e))
            count += e.size
    return float(np.sqrt(err2 / count))


def run_mms_study(cfg, gas, stdout=sys.stdout, precision="auto", ndim=2, np_ranks=1):
    """cli.py:410-434 on the device: converge the manufactured case on the
    cartesian box at each size, report the L2 solution error and the observed
    order.  ndim=3 runs the z-invariant 3D cube split over
    `np_ranks` children.  Returns [(n, error, steps, converged)]."""
    from .stepper import iterate_gpu
    sizes = [int(v) for v in cfg.mms_levels.split(",")]
    ms_id = "ns_2d" if cfg.physics == "laminar_ns" else "euler_2d"
    fs = build_freestream(replace(cfg, case="cartesian_box"), gas, ndim)
    scheme = replace(build_scheme(cfg), mms_id=ms_id)
    out = []
    for n in sizes:
        if ndim == 2:
            level, size = 0, 8
            while size < n:
                level, size = level + 2, size * 2
            if size != n:
                raise ConfigError(f"mms grid size {n} is not 8 * 2^k")
            grid = geometry.generate_case_grid("cartesian_box", level)
        else:
            grid = geometry.cartesian_box_3d(n, mms=True)
        plan = planning.decompose(grid, np_ranks, grid.ndim)
        res = iterate_gpu(plan, planning.reorder_boundaries(plan), gas, scheme, fs,
                          max_steps=cfg.max_steps, residual_target=cfg.residual_target,
                          init="manufactured", precision=precision)
        err = mms_solution_error(res)
        out.append((n, err, res.steps, res.converged))
        print(f"mms {ms_id} {n}^{ndim}: L2 error {err:.6e} ({res.steps} steps, "
              f"converged={res.converged})", file=stdout)
    for (na, a, _, _), (nb, b, _, _) in zip(out, out[1:]):
        print(f"observed order {na}->{nb}: {np.log(a / b) / np.log(nb / na):.3f}", file=stdout)
    return out


def run(cfg, stdout=sys.stdout, precision="auto"):
    from .stepper import run_distributed_gpu
    cfg = validated(cfg)
    if cfg.mms_levels:
        if cfg.case != "cartesian_box":
            raise ConfigError("mms_levels requires case = cartesian_box")
        run_mms_study(cfg, build_gas(cfg), stdout, precision)
        return EXIT_OK
    if cfg.scaling:
        raise ConfigError("scaling studies: bench.py (--gpus N under torchrun) measures them")
    check_strategy(cfg)
    os.makedirs(cfg.output_dir, exist_ok=True)
    gas = build_gas(cfg)
    grid = build_grid(cfg)
    fs = build_freestream(cfg, gas, grid.ndim)
    scheme = build_scheme(cfg)
    plan = build_plan(cfg, grid)
    schedule = planning.reorder_boundaries(plan) if cfg.reorder else planning.naive_schedule(plan)
    out = run_distributed_gpu(plan, schedule, gas, scheme, fs, max_steps=cfg.max_steps,
                              residual_target=cfg.residual_target, timeout_s=cfg.timeout_s,
                              precision=precision)
    rel = out.relative_history()
    with open(os.path.join(cfg.output_dir, "residuals.csv"), "w") as f:
        f.write("step,r_mass,r_xmom,r_ymom,r_zmom,r_energy\n")
        for i, row in enumerate(rel):
            f.write(f"{i + 1}," + ",".join(f"{v:.16e}" for v in row) + "\n")
    # the engine's own counters (bf_transfer_counters), as the reference writes
    # its RankRuntime counters (cli.py:376-378)
    with open(os.path.join(cfg.output_dir, "counters.json"), "w") as f:
        f.write(counters_to_json(out.counters))
    with open(os.path.join(cfg.output_dir, "plan.json"), "w") as f:
        f.write(json.dumps(plan_to_dict(plan, schedule), indent=2))
    if cfg.write_solution:
        for b in grid.blocks:
            write_solution_vtk(os.path.join(cfg.output_dir, f"block_{b.id}.vtk"), b,
                               out.fields[b.id])
            write_solution_npy(os.path.join(cfg.output_dir, f"block_{b.id}.npy"),
                               out.fields[b.id])
    base = out.history[0]
    active = base > 1e-12 * np.max(base)
    final = float(np.max(rel[-1][active])) if np.any(active) else 0.0
    print(f"ran {out.steps} steps on np={cfg.np}; final relative residual {final:.3e}; "
          f"solver time {out.solve_seconds:.3f}s", file=stdout)
    if cfg.compare_serial and cfg.np > 1:
        plan1 = planning.aggregate(grid, 1)
        ref = run_distributed_gpu(plan1, planning.reorder_boundaries(plan1), gas, scheme, fs,
                                  max_steps=out.steps, precision=precision)
        diff = max_rel_primitive_diff(ref.fields, out.fields, fs)
        print(f"serial comparison: max relative primitive difference {diff:.3e}", file=stdout)
    return EXIT_OK


def make_parser():
    p = argparse.ArgumentParser(prog="blockflow-gpu", description=__doc__.splitlines()[0])
    sub = p.add_subparsers(dest="command", required=True)
    r = sub.add_parser("run", help="run one configuration on the device")
    r.add_argument("config", help="path to a key = value config file")
    r.add_argument("--np", type=int, default=None, help="rank count override")
    r.add_argument("--no-reorder", action="store_true")
    r.add_argument("--compare-serial", action="store_true")
    r.add_argument("--output-dir", default=None)
    r.add_argument("--precision", choices=("auto", "exact", "fast"), default="auto")
    return p


def main(argv=None):
    args = make_parser().parse_args(argv)
    try:
        cfg = parse_config(args.config)
        over = {}
        if args.np is not None:
            over["np"] = args.np
        if args.no_reorder:
            over["reorder"] = False
        if args.compare_serial:
            over["compare_serial"] = True
        if args.output_dir is not None:
            over["output_dir"] = args.output_dir
        cfg = validated(replace(cfg, **over))
        return run(cfg, precision=args.precision)
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    except BlockflowError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_ERROR


if __name__ == "__main__":
    sys.exit(main())
