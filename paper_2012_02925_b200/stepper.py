"""Drop-in GPU replacements for the reference's stepping drivers.

Reference seam: ``RankStepper(solvers, exchange_fn, config)``
with ``.step(step_index) -> (sumsq[5], ncells)`` and ``.update_ghosts()``
(blockflow/solver.py:763-814), built internally by ``iterate``
(solver.py:914-936) and ``run_distributed`` (exchange.py:599-682).  This
module provides the same three things backed by libbfgpu.so:

  GpuRankStepper       RankStepper contract for one rank's children on one GPU
  iterate_gpu          same signature/result as solver.iterate
  run_distributed_gpu  same signature/result as exchange.run_distributed;
                       one process per GPU over NCCL when torch.distributed is
                       initialised with world_size == plan.np_ranks, otherwise
                       every rank as a context of an in-process lock-step group

Plans, boundary specs, gas/scheme/freestream objects are read by attribute,
so the reference's own objects and this package's mirrors are both accepted.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import native
from .errors import (ConfigError, DivergenceError, MetricError, NativeLibraryError,
                     NonPhysicalStateError, bridged)
from .model import FIELD_NAMES, PRIM_NAMES, RK_COEFFS, validate_scheme

_SUPPORTED_BC = tuple(native.BC)


def _geometry():
    from . import geometry, mms
    return geometry, mms


def encode_primitive(rho, u, v, w, p, gamma):
    """physics.py:136-140 (setup-time conversion of the initial state)."""
    ke = 0.5 * (u * u + v * v + w * w)
    return rho, rho * u, rho * v, rho * w, p / (gamma - 1.0) + rho * ke


def resolve_precision(precision, config):
    """"exact": reference evaluation order, bitwise where no libm pow is involved.
    "fast": FMA and strength reduction, within 1e-12 of the reference.
    "auto" (default): fast, except exact when limiters are frozen — a frozen
    non-smooth limiter pins O(1) limiter differences that roundoff-level state
    differences produce in flat regions, which later multiply real gradients
    (DESIGN.md §4), so freeze runs keep reference arithmetic."""
    if precision == "auto":
        return "exact" if getattr(config, "limiter_freeze_at", None) else "fast"
    if precision not in ("exact", "fast"):
        raise ConfigError(f"precision must be 'exact', 'fast' or 'auto', got {precision!r}")
    return precision


def host_setups(plan, child_ids, gas, config, freestream, metrics_fn=None):
    """Host-side setup (metrics, MMS data) of children, reusable across contexts."""
    return {cid: _BlockSetup(plan, cid, gas, config, freestream, metrics_fn)
            for cid in child_ids}


class _BlockSetup:
    """Host arrays of one child needed to register it with the device."""

    def __init__(self, plan, cid, gas, config, freestream, metrics_fn):
        geometry, mms = _geometry()
        self.cid = cid
        self.block = plan.child_block(cid)
        self.specs = sorted(plan.boundaries[cid], key=lambda s: s.canonical_key())
        self._metrics_fn = metrics_fn or geometry.compute_metrics
        self._metrics = None
        # host metrics are only needed for a custom metrics_fn and for MMS
        # (cell centres); otherwise the device computes them from the nodes
        self.device_metrics = metrics_fn is None and config.mms_id is None
        self.gas, self.config, self.fs = gas, config, freestream
        self.inner = self.block.interior()
        self.solution = mms.manufactured_solution(config.mms_id) if config.mms_id else None
        self.source = None
        if config.mms_id is not None:
            c = self.metrics.centers
            xs, ys, zs = (c[i][self.inner] for i in range(3))
            self.source = [np.asfortranarray(np.asarray(s) * self.vol)
                           for s in mms.mms_source(xs, ys, zs, config.mms_id, gas)]

    @property
    def metrics(self):
        """Host metrics (mesh.py compute_metrics), computed on first use."""
        if self._metrics is None:
            self._metrics = self._metrics_fn(self.block)
        return self._metrics

    @property
    def vol(self):
        return self.metrics.volume[self.inner]

    def initial_state(self, init):
        """(fields6, q5) padded Fortran arrays (solver.py:258-277)."""
        blk = self.block
        f = {}
        if init == "manufactured":
            c = self.metrics.centers
            for n in PRIM_NAMES:
                f[n] = np.asfortranarray(self.solution[n](c[0], c[1], c[2]))
            f["T"] = np.asfortranarray(f["p"] / (f["rho"] * self.gas.R))
        else:
            for n in FIELD_NAMES:
                f[n] = blk.allocate_field(getattr(self.fs, n))
        q = [np.asfortranarray(x) for x in
             encode_primitive(*(f[n] for n in PRIM_NAMES), self.gas.gamma)]
        return [f[n] for n in FIELD_NAMES], q

    def dirichlet_values(self, spec, extended=False):
        """Cached MMS ghost values of one patch, [layer][6][tangential] (solver.py:385-401);
        extended: tangential ranges widened by the ghost depth (round 2, solver.py:285-305)."""
        g = self.block.ghost
        d = spec.axis
        n = self.block.dims[d]
        tang = []
        for a in range(3):
            if a == d:
                tang.append(None)
            else:
                lo, hi = spec.box[a]
                ext = g[a] if extended else 0
                tang.append(slice(g[a] + lo - ext, g[a] + hi + ext))
        c = self.metrics.centers
        out = []
        for depth in range(self.block.ghost_depth):
            pos = g[d] - 1 - depth if spec.side == 0 else g[d] + n + depth
            cut = list(tang)
            cut[d] = pos
            cut = tuple(cut)
            vals = {nm: self.solution[nm](c[0][cut], c[1][cut], c[2][cut]) for nm in PRIM_NAMES}
            vals["T"] = vals["p"] / (vals["rho"] * self.gas.R)
            for nm in FIELD_NAMES:
                out.append(np.asarray(vals[nm], float).ravel(order="F"))
        return np.ascontiguousarray(np.concatenate(out))


class GpuContext:
    """One libbfgpu context: the children of one rank on one device."""

    def __init__(self, plan, child_ids, gas, config, freestream, device=0, rank=0, nranks=1,
                 precision="auto", metrics_fn=None, setups=None, schedule=None):
        validate_scheme(config)
        precision = resolve_precision(precision, config)
        self.viscous = bool(getattr(config, "viscous", False))
        self.L = native.lib()
        self.plan = plan
        self.gas, self.config, self.fs = gas, config, freestream
        self.rank, self.nranks, self.device = rank, nranks, device
        self.precision = precision
        self.child_ids = sorted(child_ids)
        self.ndim = plan.grid.ndim
        sch = native.Scheme(
            flux=native.FLUX[config.flux], limiter=native.LIMITER[config.limiter],
            epsilon=float(config.epsilon), kappa=float(config.kappa),
            rk_stages=int(config.rk_stages), cfl=float(config.cfl),
            limiter_freeze_at=int(config.limiter_freeze_at or 0),
            entropy_fix_coeff=float(config.entropy_fix_coeff),
            has_wall_temperature=int(config.wall_temperature is not None),
            wall_temperature=float(config.wall_temperature or 0.0),
            precision=native.PRECISION[precision], viscous=int(self.viscous))
        suth = getattr(gas, "sutherland", None)
        gas_s = native.Gas(gamma=float(gas.gamma), R=float(gas.R),
                           mu=float(getattr(gas, "mu", 0.0)),
                           prandtl=float(getattr(gas, "prandtl", 0.72)),
                           has_sutherland=int(suth is not None),
                           sutherland=(C.c_double * 3)(*(suth if suth is not None else (0, 0, 0))))
        fs_s = native.Freestream(*(float(getattr(freestream, n)) for n in FIELD_NAMES))
        t_create = time.perf_counter()
        self.ctx = self.L.bf_create(self.ndim, C.byref(gas_s), C.byref(sch), C.byref(fs_s),
                                    device, rank, nranks)
        self.timing = {"create_s": time.perf_counter() - t_create, "blocks_s": []}
        if not self.ctx:
            raise NativeLibraryError(f"bf_create failed (device {device}, rank {rank}/{nranks})")
        self.setups = {}
        self._keep_nodes = []
        for cid in self.child_ids:
            s = setups[cid] if setups is not None else \
                _BlockSetup(plan, cid, gas, config, freestream, metrics_fn)
            self.setups[cid] = s
            if s.device_metrics and s.source is None:
                nodes = []
                for c in range(self.ndim):
                    x = np.asarray(s.block.nodes[c], dtype=float)
                    if not (x.flags.c_contiguous or x.flags.f_contiguous):
                        x = np.ascontiguousarray(x)
                    nodes.append(x)
                st = [x // 8 for x in nodes[0].strides] + [0] * (3 - self.ndim)
                if any(n.strides != nodes[0].strides for n in nodes):
                    nodes = [np.ascontiguousarray(n) for n in nodes]
                    st = [x // 8 for x in nodes[0].strides] + [0] * (3 - self.ndim)
                t_blk = time.perf_counter()
                self._check(self.L.bf_add_block_nodes(
                    self.ctx, cid, native.ints(s.block.dims), s.block.ghost_depth,
                    native.dptrs(nodes), (C.c_longlong * 3)(*st), None))
                self.timing["blocks_s"].append(time.perf_counter() - t_blk)
                self._keep_nodes.append(nodes)   # read asynchronously until bf_sync_blocks
                continue
            fv = []
            for d in range(self.ndim):
                for comp in range(3):
                    fv.append(np.asfortranarray(s.metrics.face_vectors[d][comp], dtype=float))
            vol = np.asfortranarray(s.vol, dtype=float)
            src = native.dptrs(s.source) if s.source is not None else None
            self._keep = (fv, vol, s.source)
            self._check(self.L.bf_add_block(self.ctx, cid, native.ints(s.block.dims),
                                            s.block.ghost_depth, native.dptrs(fv),
                                            native.dptr(vol), src))
        t_sync = time.perf_counter()
        self._check(self.L.bf_sync_blocks(self.ctx))   # device metrics done; inverted cells raise
        self.timing["sync_s"] = time.perf_counter() - t_sync
        self._keep_nodes = []
        if self.viscous:   # face gradient matrices (solver.py:582-642), host numpy
            geometry, _ = _geometry()
            for cid in self.child_ids:
                s = self.setups[cid]
                mats = [None] * 27
                keep = []
                for d in range(self.ndim):
                    M = geometry.face_gradient_matrix(s.block, s.metrics, d)
                    for r in range(3):
                        for e in range(3):
                            if r < self.ndim and e < self.ndim:
                                arr = np.asfortranarray(M[r, e])
                                keep.append(arr)
                                mats[9 * d + 3 * r + e] = arr
                self._check(self.L.bf_add_viscous_geometry(self.ctx, cid, native.dptrs(mats)))
        added = []   # connected endpoints in bf_add_link order
        for cid in self.child_ids:
            s = self.setups[cid]
            for spec in s.specs:
                box = native.ints([x for r in spec.box for x in r])
                face = native.FACES.index(spec.face)
                if spec.kind == "physical":
                    if spec.bc_type not in native.BC:
                        raise bridged(ConfigError)(f"unknown physical bc type {spec.bc_type!r}")
                    vals = vext = None
                    if spec.bc_type == "mms_dirichlet":
                        if s.solution is None:
                            raise bridged(ConfigError)("mms_dirichlet patch needs config.mms_id")
                        vals = s.dirichlet_values(spec)
                        if self.viscous:
                            vext = s.dirichlet_values(spec, extended=True)
                    self._check(self.L.bf_add_bc_patch_ext(
                        self.ctx, cid, native.BC[spec.bc_type], face, box,
                        native.dptr(vals) if vals is not None else None,
                        native.dptr(vext) if vext is not None else None))
                else:
                    peer = spec.neighbor_block
                    prank = plan.child(peer).rank if nranks > 1 else rank
                    self._check(self.L.bf_add_link(
                        self.ctx, cid, face, box,
                        native.ints([x for e in spec.axis_map for x in e]), peer,
                        native.FACES.index(spec.neighbor_face),
                        native.ints([x for r in spec.neighbor_box for x in r]), prank,
                        int(spec.link_id)))
                    added.append((cid, spec))
        if self.viscous and added:
            # round-2 unpack order = the reference's exchange sequence: the schedule's
            # entries rank-major (solver.py:869-899); the runtime puts remote ones last
            if schedule is None:
                from .planning import reorder_boundaries
                schedule = reorder_boundaries(plan)
            seq = [(e.child, id(e.spec)) for r in sorted(schedule.per_rank)
                   for e in schedule.per_rank[r]]
            pos = {key: q for q, key in enumerate(seq)}
            keyed = [(cid, spec) for cid, spec in added]
            order = []
            for cid, spec in keyed:
                q = pos.get((cid, id(spec)))
                if q is None:   # schedule built from another plan object: match by value
                    q = next(i for i, (e) in enumerate(
                        [e for r in sorted(schedule.per_rank) for e in schedule.per_rank[r]])
                        if e.child == cid and e.spec == spec)
                order.append(q)
            self._check(self.L.bf_set_round2_order(self.ctx, len(order), native.ints(order)))
        self._finalized = False

    def finalize(self):
        if not self._finalized:
            self._check(self.L.bf_finalize(self.ctx))
            self._finalized = True

    # ------------------------------------------------------------------
    def _check(self, rc, block=None):
        if rc == native.BF_OK:
            return
        if rc == native.BF_ENONPHYSICAL:
            raise bridged(NonPhysicalStateError)(self.error_message())
        msg = native.last_error(self.ctx)
        if rc == native.BF_EINVAL:
            raise bridged(ConfigError)(msg)
        if rc == native.BF_EMETRIC:
            # reformat the index tuple the way the reference prints np.argwhere's row
            import re
            m = re.match(r"block (-?\d+): inverted cell at interior index \((\d+), (\d+), (\d+)\)",
                         msg)
            if m:
                bad = np.array([int(m.group(k)) for k in (2, 3, 4)])
                msg = f"block {int(m.group(1))}: inverted cell at interior index {tuple(bad)}"
            raise bridged(MetricError)(msg)
        raise NativeLibraryError(f"libbfgpu error {rc}: {msg}")

    def error_message(self):
        kind, blk, stage, d = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        idx = (C.c_longlong * 3)()
        self.L.bf_error_info(self.ctx, C.byref(kind), C.byref(blk), C.byref(stage), C.byref(d),
                             idx)
        ix = tuple(np.int64(x) for x in idx)
        if kind.value in (native.ERR_FACE_LEFT, native.ERR_FACE_RIGHT):
            side = "left" if kind.value == native.ERR_FACE_LEFT else "right"
            return (f"block {blk.value}: non-physical {side} face state, "
                    f"direction {d.value}, face index {ix}")
        if kind.value == native.ERR_ROE_A2:
            return f"Roe-averaged state has non-positive sound speed at index {np.array(ix)}"
        if kind.value == native.ERR_UPDATE:
            return (f"block {blk.value}: non-physical update at cell {ix} "
                    f"(CFL {self.config.cfl} may be too high)")
        return native.last_error(self.ctx)

    def upload_initial(self, init="uniform", seed=0):
        """init: "uniform" | "manufactured" (solver.py:258-271) | "perturbed"
        (freestream, interior rho/p x (1 + 0.01 N(0,1)) drawn
        per child in child-id order from default_rng(seed); the draws of
        children owned by other ranks are consumed too, so every rank sees
        the same initial field as a serial run)."""
        self.finalize()
        if init == "perturbed":
            from .cases import perturbed_state
            rng = np.random.default_rng(seed)
            mine = set(self.child_ids)
            for c in sorted(self.plan.children, key=lambda c: c.id):
                if c.id not in mine:
                    # consume the same draws (rho, then p, C order) without the arrays
                    n = int(np.prod(c.dims)) if hasattr(c, "dims") else \
                        self.plan.child_block(c.id).cell_count()
                    for _ in range(2):
                        left = n
                        while left > 0:
                            m = min(left, 1 << 24)
                            rng.standard_normal(m)
                            left -= m
                    continue
                blk = self.setups[c.id].block
                f = perturbed_state(blk, self.fs, self.gas, rng)
                self.upload(c.id, [f[n] for n in FIELD_NAMES])   # Q derived on the device
            return
        for cid in self.child_ids:
            f6, _ = self.setups[cid].initial_state(init)
            self.upload(cid, f6)

    def upload(self, cid, fields6, q5=None):
        """Padded initial fields of a child; q5=None: conserved variables are
        derived on the device (encode_primitive, bitwise)."""
        f6 = [np.asfortranarray(x, dtype=float) for x in fields6]
        q = None if q5 is None else [np.asfortranarray(x, dtype=float) for x in q5]
        self._check(self.L.bf_upload_fields(self.ctx, cid, native.dptrs(f6),
                                            native.dptrs(q) if q is not None else None))

    def update_ghosts(self):
        self._check(self.L.bf_update_ghosts(self.ctx))

    def step(self, step_index):
        out = (C.c_double * 5)()
        n = C.c_longlong()
        self._check(self.L.bf_step(self.ctx, int(step_index), out, C.byref(n)))
        return np.array(out[:], dtype=float), int(n.value)

    def iterate(self, first_step, max_steps, residual_target=None, residual_floor=None,
                divergence_factor=1e6):
        """bf_iterate: up to max_steps steps with the history guards evaluated in C
        after each; returns (norms[steps, 5], status) — status 1 converged, 2
        diverged at the last step, 0 ran max_steps."""
        hist = np.zeros((max(int(max_steps), 1), 5))
        done, status = C.c_int(), C.c_int()
        self._check(self.L.bf_iterate(
            self.ctx, int(first_step), int(max_steps), int(residual_target is not None),
            float(residual_target or 0.0), int(residual_floor is not None),
            float(residual_floor or 0.0), float(divergence_factor), native.dptr(hist),
            C.byref(done), C.byref(status)))
        return hist[:done.value].copy(), status.value

    def download(self, cid, what, out=None):
        """One array of a child (BF_FIELD_* selector or field name); `out`, when
        given, is a preallocated Fortran float64 array of the right shape
        (e.g. in pinned host memory)."""
        blk = self.setups[cid].block
        if isinstance(what, str):
            code = native.FIELD[what]
        else:
            code = int(what)
        if code in (native.FIELD["dtv"], native.FIELD_VOL):
            shape = tuple(blk.dims)
        elif native.FIELD_FACE <= code < native.FIELD_FACE + 12:
            d = (code - native.FIELD_FACE) // 4
            shape = list(blk.dims)
            shape[d] += 1
            shape = tuple(shape)
        elif code >= native.FIELD_PSI:
            r = code - native.FIELD_PSI
            d = r // 10
            shape = list(blk.dims)
            shape[d] += 2
            shape = tuple(shape)
        else:
            shape = blk.shape
        if out is None:
            out = np.empty(shape, order="F")
        elif out.shape != tuple(shape) or out.dtype != np.float64 or not out.flags.f_contiguous:
            raise ValueError(f"download: out must be a Fortran float64 array of shape {shape}")
        self._check(self.L.bf_download(self.ctx, cid, code, native.dptr(out)))
        return out

    def set_stream(self, stream_ptr):
        self._check(self.L.bf_set_stream(self.ctx, C.c_void_p(stream_ptr)))

    def set_profiling(self, on):
        self._check(self.L.bf_set_profiling(self.ctx, int(bool(on))))

    def kernel_stats(self, cls):
        n, ms = C.c_longlong(), C.c_double()
        self._check(self.L.bf_kernel_stats(self.ctx, cls, C.byref(n), C.byref(ms)))
        return int(n.value), float(ms.value)

    def transfer_bytes(self):
        return int(self.L.bf_transfer_bytes(self.ctx, 0)), int(self.L.bf_transfer_bytes(self.ctx, 1))

    COUNTER_NAMES = ("messages", "runs", "bytes", "staging_copies", "waits", "max_pending")

    def transfer_counters(self):
        """The engine's cumulative TransferCounters (bf_transfer_counters,
        exchange.py:83-101 fields) as a dict."""
        out = (C.c_longlong * 6)()
        self._check(self.L.bf_transfer_counters(self.ctx, out))
        return dict(zip(self.COUNTER_NAMES, (int(v) for v in out)))

    def close(self):
        if getattr(self, "ctx", None):
            self.L.bf_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class _LazyFields(dict):
    """fields[name] -> padded Fortran ndarray, downloaded on first access."""

    def __init__(self, view):
        super().__init__()
        self._view = view

    def __missing__(self, name):
        if name not in FIELD_NAMES:
            raise KeyError(name)
        arr = self._view._gpu.download(self._view._cid, name)
        self[name] = arr
        return arr

    def keys(self):
        return FIELD_NAMES

    def __iter__(self):
        return iter(FIELD_NAMES)

    def __len__(self):
        return len(FIELD_NAMES)

    def items(self):
        return [(n, self[n]) for n in FIELD_NAMES]

    def values(self):
        return [self[n] for n in FIELD_NAMES]


class GpuBlockView:
    """Read-side stand-in for a BlockSolver (what callers read after a run,
    SURVEY.md §8b): fields/q are device downloads, geometry is host-side."""

    PRIM_NAMES = PRIM_NAMES

    def __init__(self, gpu, cid):
        s = gpu.setups[cid]
        self._gpu, self._cid = gpu, cid
        self.block = s.block
        self.gas, self.config, self.freestream = gpu.gas, gpu.config, gpu.fs
        self.specs = s.specs
        self.physical_specs = [x for x in s.specs if x.kind == "physical"]
        self.dirs = (0, 1) if s.block.ndim == 2 else (0, 1, 2)
        self._int = s.inner
        self.frozen = False
        self.invalidate()

    @property
    def metrics(self):
        return self._gpu.setups[self._cid].metrics

    @property
    def _vol(self):
        return self._gpu.setups[self._cid].vol

    def invalidate(self):
        self.fields = _LazyFields(self)
        self._q = None
        self._psi = None

    @property
    def q(self):
        if self._q is None:
            self._q = [self._gpu.download(self._cid, native.FIELD_Q0 + e) for e in range(5)]
        return self._q

    @property
    def psi(self):
        """{d: (psi_plus (5, ...), psi_minus (5, ...))} when limiters are kept (freeze runs)."""
        if self._psi is None:
            if not self.config.limiter_freeze_at:
                return {}
            out = {}
            for d in self.dirs:
                pair = []
                for pm in range(2):
                    pair.append(np.stack([self._gpu.download(
                        self._cid, native.FIELD_PSI + 10 * d + 5 * pm + v) for v in range(5)]))
                out[d] = tuple(pair)
            self._psi = out
        return self._psi

    def residual_sumsq(self, R):
        return np.array([float(np.sum(r * r)) for r in R])


class GpuRankStepper:
    """RankStepper (solver.py:763-814) backed by one device context."""

    def __init__(self, gpu: GpuContext, config):
        self.gpu = gpu
        self.config = config
        self.alphas = RK_COEFFS[config.rk_stages]
        self.solvers = {cid: GpuBlockView(gpu, cid) for cid in gpu.child_ids}

    def update_ghosts(self):
        self.gpu.update_ghosts()
        self._invalidate()

    def step(self, step_index):
        fz = self.config.limiter_freeze_at
        try:
            sumsq, ncells = self.gpu.step(step_index)
        finally:
            self._invalidate()
        for v in self.solvers.values():
            v.frozen = fz is not None and step_index > fz
        return sumsq, ncells

    def run(self, first_step, max_steps, residual_target=None, residual_floor=None):
        """Steps first_step .. while the history guards allow, driven from C
        (GpuContext.iterate); returns the norms of the steps taken."""
        fz = self.config.limiter_freeze_at
        try:
            hist, _ = self.gpu.iterate(first_step, max_steps, residual_target, residual_floor)
        finally:
            self._invalidate()
        if len(hist):
            last = first_step + len(hist) - 1
            for v in self.solvers.values():
                v.frozen = fz is not None and last > fz
        return hist

    def _invalidate(self):
        for v in self.solvers.values():
            v.invalidate()


@dataclass
class IterationResult:
    """solver.py:817-829."""
    solvers: dict
    history: np.ndarray
    steps: int
    converged: bool

    def relative_history(self):
        base = self.history[0].copy()
        safe = np.where(base > 0.0, base, 1.0)
        rel = self.history / safe
        rel[:, base == 0.0] = 0.0
        return rel


@dataclass
class DistributedResult:
    """exchange.py:582-596."""
    fields: dict
    history: np.ndarray
    steps: int
    converged: bool
    counters: dict
    solve_seconds: float

    def relative_history(self):
        base = self.history[0].copy()
        safe = np.where(base > 0.0, base, 1.0)
        rel = self.history / safe
        rel[:, base == 0.0] = 0.0
        return rel


def residual_norms(sumsq):
    return np.sqrt(np.asarray(sumsq))


def check_history_guards(history, step, residual_target, divergence_factor=1e6,
                         residual_floor=None):
    """solver.py:836-855 (host-side, per step)."""
    if residual_floor is not None and float(np.max(history[step])) <= residual_floor:
        return True
    base = history[0]
    active = base > 1e-12 * np.max(base)
    if not np.any(active):
        return False
    rel = history[step][active] / base[active]
    if np.any(~np.isfinite(rel)) or np.max(rel) > divergence_factor:
        raise bridged(DivergenceError)(
            f"residual grew by more than {divergence_factor:.0e} at step {step + 1}")
    return residual_target is not None and float(np.max(rel)) <= residual_target


def write_residual_csv(result, path):
    """solver.py:939-945."""
    rel = result.relative_history()
    with open(path, "w") as f:
        f.write("step,r_mass,r_xmom,r_ymom,r_zmom,r_energy\n")
        for i, row in enumerate(rel):
            f.write(f"{i + 1}," + ",".join(f"{v:.16e}" for v in row) + "\n")


def release_cache(device=-1):
    """Hand the block arenas kept for reuse (and the staging pool) back to the
    driver (bf_release_cache).  They are kept only while another context of the
    device is alive, or across contexts when BF_ARENA_CACHE=1."""
    native.lib().bf_release_cache(int(device))


def iterate_gpu(plan, schedule, gas, config, freestream, max_steps, residual_target=None,
                init="uniform", residual_floor=None, device=0, precision="auto",
                metrics_fn=None):
    """solver.iterate on one GPU: every child of the plan in one context, all
    connected boundaries served by device copies (solver.py:914-936).  The
    device memory is returned when the context closes (release_cache)."""
    gpu = GpuContext(plan, [c.id for c in plan.children], gas, config, freestream,
                     device=device, precision=precision, metrics_fn=metrics_fn,
                     schedule=schedule)
    gpu.upload_initial(init)
    stepper = GpuRankStepper(gpu, config)
    # the step loop and its guards run in C (bf_iterate: no return to Python
    # between steps); the guard is re-evaluated here on the last step so a
    # divergence raises exactly as solver.py:836-855 does
    history = list(stepper.run(1, max_steps, residual_target, residual_floor))
    converged = bool(history) and check_history_guards(history, len(history) - 1,
                                                       residual_target,
                                                       residual_floor=residual_floor)
    return IterationResult(solvers=stepper.solvers, history=np.array(history),
                           steps=len(history), converged=converged)


def _gather_parent_fields(plan, views_by_cid):
    names = FIELD_NAMES
    out = {b.id: {n: np.full(b.dims, np.nan) for n in names} for b in plan.grid.blocks}
    for cid, view in views_by_cid.items():
        c = plan.child(cid)
        (i0, i1), (j0, j1), (k0, k1) = c.cell_box()
        for n in names:
            out[c.parent][n][i0:i1, j0:j1, k0:k1] = view.fields[n][view.block.interior()]
    return out


def native_counters(plan, rounds=1, exchanges=1):
    """Predicted transfer counters of the native engine (the analogue of
    exchange.py:166-200 predict_counters) after `exchanges` ghost updates of
    `rounds` rounds each: per round a rank sends ONE message per remote endpoint
    (all fields concatenated, one grouped NCCL send/recv), runs one pack and one
    unpack launch, waits once for the grouped exchange and has every send and
    receive of the group in flight; no staging copies.  bf_transfer_counters
    reports what the engine actually did (tests/test_gpu_loopback.py holds the
    two equal)."""
    from .topology import halo_regions
    ndim = plan.grid.ndim
    nf = 3 + ndim
    out = {r: dict.fromkeys(GpuContext.COUNTER_NAMES, 0) for r in range(plan.np_ranks)}
    for rnd in range(1, rounds + 1):
        per_rank = {r: [0, 0] for r in range(plan.np_ranks)}
        for cid, s in plan.connected_specs():
            rank = plan.child(cid).rank
            if plan.child(s.neighbor_block).rank == rank:
                continue
            blk = plan.child_block(cid)
            send, _ = halo_regions(s, blk.dims, blk.ghost, rnd)
            per_rank[rank][0] += 1
            per_rank[rank][1] += int(np.prod([hi - lo for lo, hi in send])) * nf * 8
        for r, (n, b) in per_rank.items():
            if not n:
                continue
            c = out[r]
            c["messages"] += n * exchanges
            c["bytes"] += b * exchanges
            c["runs"] += 2 * exchanges
            c["waits"] += exchanges
            c["max_pending"] = max(c["max_pending"], 2 * n)
    return out


def run_distributed_gpu(plan, schedule, gas, config, freestream, strategy=None, max_steps=100,
                        residual_target=None, init="uniform", timeout_s=5.0,
                        residual_floor=None, precision="auto", devices=None, metrics_fn=None,
                        transport="loopback"):
    """exchange.run_distributed on GPUs (exchange.py:599-682).

    * torch.distributed initialised with world_size == plan.np_ranks: this
      process runs rank = dist.get_rank() on cuda:LOCAL_RANK, halos over NCCL,
      the residual sum over ranks in rank order; fields are gathered to every
      rank.
    * otherwise every rank lives in this process, rank r on device
      devices[r % len(devices)] (all on device 0 by default):
      - transport="loopback" (default): one host thread per rank, as the
        reference's run_distributed spawns them (exchange.py:647-651), each
        driving its own context through the NCCL code path of the runtime
        (grouped send/recv of the halo messages on the comm stream overlapped
        with the interior tiles, rank-ordered allgather of the residual) with
        the in-process transport of bf_loopback.h bound instead of libnccl;
      - transport="group": all ranks driven in lock step from this thread,
        halos as device-to-device copies (bf_group_*).
    """
    import os
    nr = plan.np_ranks
    dist = None
    try:
        import torch.distributed as tdist
        if tdist.is_available() and tdist.is_initialized() and tdist.get_world_size() == nr:
            dist = tdist
    except Exception:  # noqa: BLE001
        dist = None
    history, converged = [], False
    if dist is not None:
        rank = dist.get_rank()
        device = int(os.environ.get("LOCAL_RANK", rank)) if devices is None else devices[rank]
        gpu = GpuContext(plan, [c.id for c in plan.rank_children(rank)], gas, config, freestream,
                         device=device, rank=rank, nranks=nr, precision=precision,
                         metrics_fn=metrics_fn, schedule=schedule)
        uid = bytearray(128)
        if rank == 0:
            buf = (C.c_char * 128)()
            gpu._check(gpu.L.bf_nccl_unique_id(buf))
            uid = bytearray(buf.raw)
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0)
        idbuf = (C.c_char * 128).from_buffer_copy(box[0])
        gpu._check(gpu.L.bf_nccl_init(gpu.ctx, idbuf))
        gpu.upload_initial(init)
        stepper = GpuRankStepper(gpu, config)
        dist.barrier()
        t0 = time.perf_counter()
        # step loop and guards in C (bf_iterate; the guards see the rank-ordered
        # global norms, so every rank stops at the same step)
        history = list(stepper.run(1, max_steps, residual_target, residual_floor))
        converged = bool(history) and check_history_guards(history, len(history) - 1,
                                                           residual_target,
                                                           residual_floor=residual_floor)
        solve = time.perf_counter() - t0
        from .distributed import assemble_parent_fields, local_interiors
        parts = [None] * nr
        dist.all_gather_object(parts, local_interiors(stepper.solvers))
        fields = assemble_parent_fields(plan, parts)
        counts = [None] * nr
        dist.all_gather_object(counts, gpu.transfer_counters())
        gpu.close()
        return DistributedResult(fields=fields, history=np.array(history), steps=len(history),
                                 converged=converged, counters=dict(enumerate(counts)),
                                 solve_seconds=solve)

    if transport == "loopback":
        return _run_loopback(plan, schedule, gas, config, freestream, max_steps, residual_target,
                             init, residual_floor, precision, devices, metrics_fn)
    if transport != "group":
        raise bridged(ConfigError)(f"unknown transport {transport!r}")
    devs = list(devices) if devices is not None else [0]
    gpus = [GpuContext(plan, [c.id for c in plan.rank_children(r)], gas, config, freestream,
                       device=devs[r % len(devs)], rank=r, nranks=nr, precision=precision,
                       metrics_fn=metrics_fn, schedule=schedule) for r in range(nr)]
    for g in gpus:
        g.upload_initial(init)
    L = native.lib()
    arr = (C.c_void_p * nr)(*[g.ctx for g in gpus])
    grp = L.bf_group_create(arr, nr)
    if not grp:
        raise NativeLibraryError("bf_group_create failed")
    steppers = [GpuRankStepper(g, config) for g in gpus]
    try:
        t0 = time.perf_counter()
        for step in range(max_steps):
            out = (C.c_double * 5)()
            bad = C.c_int(-1)
            rc = L.bf_group_step(grp, step + 1, out, C.byref(bad))
            for st in steppers:
                st._invalidate()
            if rc != native.BF_OK:
                g = gpus[bad.value] if bad.value >= 0 else gpus[0]
                g._check(rc)
            history.append(residual_norms(np.array(out[:])))
            if check_history_guards(history, step, residual_target,
                                    residual_floor=residual_floor):
                converged = True
                break
        solve = time.perf_counter() - t0
        views = {cid: v for st in steppers for cid, v in st.solvers.items()}
        fields = _gather_parent_fields(plan, views)
        counters = {r: g.transfer_counters() for r, g in enumerate(gpus)}
    finally:
        L.bf_group_destroy(grp)
    return DistributedResult(fields=fields, history=np.array(history), steps=len(history),
                             converged=converged, counters=counters,
                             solve_seconds=solve)


def _run_loopback(plan, schedule, gas, config, freestream, max_steps, residual_target, init,
                  residual_floor, precision, devices, metrics_fn):
    """run_distributed_gpu with one host thread per rank over the loopback
    transport (see run_distributed_gpu)."""
    import threading
    nr = plan.np_ranks
    devs = list(devices) if devices is not None else [0]
    L = native.lib()
    world = L.bf_loopback_create(nr)
    if not world:
        raise NativeLibraryError("bf_loopback_create failed")
    gpus = []
    try:
        for r in range(nr):
            g = GpuContext(plan, [c.id for c in plan.rank_children(r)], gas, config, freestream,
                           device=devs[r % len(devs)], rank=r, nranks=nr, precision=precision,
                           metrics_fn=metrics_fn, schedule=schedule)
            gpus.append(g)
            g._check(L.bf_loopback_init(g.ctx, world))
        for g in gpus:
            g.upload_initial(init)
        steppers = [GpuRankStepper(g, config) for g in gpus]
        results, errors = [None] * nr, {}
        # solver time starts once every rank is set up (exchange.py:620-655)
        barrier = threading.Barrier(nr + 1)

        def worker(r):
            try:
                barrier.wait()
                results[r] = steppers[r].run(1, max_steps, residual_target, residual_floor)
            except BaseException as exc:  # noqa: BLE001 — stop the others, re-raise below
                errors[r] = exc
                L.bf_loopback_abort(world)

        threads = [threading.Thread(target=worker, args=(r,), name=f"gpu-rank-{r}")
                   for r in range(nr)]
        for t in threads:
            t.start()
        barrier.wait()
        t0 = time.perf_counter()
        for t in threads:
            t.join()
        solve = time.perf_counter() - t0
        if errors:
            # the first failing rank's own error (the others only saw the abort)
            import re

            def secondary(e):   # a peer's echo of another rank's failure
                return ("loopback transport" in str(e) or
                        re.fullmatch(r"rank \d+: non-physical state", str(e)) is not None)
            raise errors[min(errors, key=lambda r: (secondary(errors[r]), r))]
        history = [np.asarray(h) for h in results[0]]
        for r in range(1, nr):   # every rank saw the same rank-ordered global norms
            if len(results[r]) != len(history) or not np.array_equal(np.asarray(results[r]),
                                                                     np.asarray(results[0])):
                raise NativeLibraryError(f"rank {r} residual history differs from rank 0")
        converged = bool(history) and check_history_guards(history, len(history) - 1,
                                                           residual_target,
                                                           residual_floor=residual_floor)
        views = {cid: v for st in steppers for cid, v in st.solvers.items()}
        fields = _gather_parent_fields(plan, views)
        counters = {r: g.transfer_counters() for r, g in enumerate(gpus)}
        return DistributedResult(fields=fields, history=np.array(history), steps=len(history),
                                 converged=converged, counters=counters,
                                 solve_seconds=solve)
    finally:
        for g in gpus:
            g.close()
        L.bf_loopback_destroy(world)
