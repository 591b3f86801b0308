"""Structured blocks, finite-volume metrics and the built-in case grids.

Host-side setup that feeds the device path (the reference's blockflow/mesh.py
is out of the hot-path scope, but the GPU box has no reference
installed, so the drop-in carries its own).  Every formula below keeps the
reference's floating-point evaluation order, because the device path's
parity tests compare against the reference run on the reference's own
metrics: tests/test_host_mirror.py checks these arrays bitwise.

Storage conventions (mesh.py:1-19): cell arrays are padded by ``ghost_depth``
layers on every stencil axis (k only in 3D) and are i-fastest; face-vector
array ``face_vectors[d]`` has shape (3, N_d+1, padded tangential...) and
points toward increasing index.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import GridFormatError, MetricError
from .topology import BoundarySpec, face_axis, face_side, make_connected_pair

GHOST_DEPTH = 2
CASE_PRESETS = ("inlet_ramp_2d", "c_annulus_2d", "multiblock_box_3d", "cartesian_box")


def _pad_nodes_linear(comp, axis, depth):
    """Linear ghost-node extrapolation, one layer per pass (mesh.py:35-41)."""
    for _ in range(depth):
        first = np.take(comp, [0], axis=axis)
        second = np.take(comp, [1], axis=axis)
        last = np.take(comp, [-1], axis=axis)
        before_last = np.take(comp, [-2], axis=axis)
        comp = np.concatenate([2.0 * first - second, comp, 2.0 * last - before_last], axis=axis)
    return comp


class Block:
    """One structured block (mesh.py:44-119)."""

    def __init__(self, block_id, interior_nodes, ndim, ghost_depth=GHOST_DEPTH):
        if ghost_depth < GHOST_DEPTH:
            raise ValueError(f"ghost_depth must be >= {GHOST_DEPTH}")
        nodes = np.asarray(interior_nodes, dtype=float)
        if nodes.ndim != ndim + 1 or nodes.shape[0] != ndim:
            raise GridFormatError(
                f"block {block_id}: node array must be ({ndim}, ...), got {nodes.shape}")
        if not np.all(np.isfinite(nodes)):
            raise GridFormatError(f"block {block_id}: non-finite node coordinates")
        dims = tuple(n - 1 for n in nodes.shape[1:])
        if any(n <= 0 for n in dims):
            raise GridFormatError(f"block {block_id}: degenerate block, dims {dims}")
        self.id = block_id
        self.ndim = ndim
        self.ghost_depth = ghost_depth
        self.dims = dims if ndim == 3 else (dims[0], dims[1], 1)
        comps = []
        for c in range(ndim):
            comp = nodes[c]
            for axis in range(ndim):
                comp = _pad_nodes_linear(comp, axis, ghost_depth)
            comps.append(comp)
        self.nodes = np.stack(comps)

    @classmethod
    def from_padded_nodes(cls, block_id, padded_nodes, dims, ndim, ghost_depth=GHOST_DEPTH):
        blk = cls.__new__(cls)
        blk.id = block_id
        blk.ndim = ndim
        blk.ghost_depth = ghost_depth
        blk.dims = tuple(dims) if ndim == 3 else (dims[0], dims[1], 1)
        want = tuple(blk.dims[a] + 2 * blk.ghost[a] + 1 for a in range(ndim))
        if padded_nodes.shape != (ndim, *want):
            raise GridFormatError(
                f"block {block_id}: padded nodes shape {padded_nodes.shape} "
                f"does not match dims {dims}")
        blk.nodes = np.asarray(padded_nodes, dtype=float)
        return blk

    @property
    def ghost(self):
        g = self.ghost_depth
        return (g, g, g if self.ndim == 3 else 0)

    @property
    def shape(self):
        return tuple(n + 2 * g for n, g in zip(self.dims, self.ghost))

    def interior(self):
        return tuple(slice(g, g + n) for n, g in zip(self.dims, self.ghost))

    def allocate_field(self, value=0.0):
        out = np.empty(self.shape, dtype=float, order="F")
        out.fill(value)
        return out

    def cell_count(self):
        return int(np.prod(self.dims))


@dataclass
class MultiBlockGrid:
    """Parent blocks plus their boundary patches (mesh.py:122-166)."""
    blocks: list
    boundaries: list = field(default_factory=list)

    def __post_init__(self):
        ids = [b.id for b in self.blocks]
        if len(set(ids)) != len(ids):
            raise GridFormatError(f"duplicate block ids: {ids}")
        self.validate_boundaries()

    @property
    def parent_count(self):
        return len(self.blocks)

    @property
    def ndim(self):
        return self.blocks[0].ndim

    def block(self, block_id):
        for b in self.blocks:
            if b.id == block_id:
                return b
        raise KeyError(f"no block {block_id}")

    def block_boundaries(self, block_id):
        return [s for s in self.boundaries if s.block == block_id]

    def total_cells(self):
        return sum(b.cell_count() for b in self.blocks)

    def validate_boundaries(self):
        links = {}
        for s in self.boundaries:
            self.block(s.block)
            if s.kind == "connected":
                self.block(s.neighbor_block)
                links.setdefault(s.link_id, []).append(s)
        for lid, specs in links.items():
            if len(specs) != 2:
                raise GridFormatError(f"connected link {lid} has {len(specs)} specs, expected 2")
            specs[0].validate_pair(specs[1])


@dataclass
class BlockMetrics:
    """Face area vectors, volumes and centres of one block (mesh.py:173-204)."""
    volume: np.ndarray
    centers: np.ndarray
    face_vectors: list
    ghost: tuple = (0, 0, 0)


def compute_metrics(block):
    """Metrics of a block; raises MetricError on an inverted interior cell."""
    m = _metrics_2d(block) if block.ndim == 2 else _metrics_3d(block)
    inner = m.volume[block.interior()]
    if np.any(inner <= 0.0):
        bad = np.argwhere(inner <= 0.0)[0]
        raise MetricError(f"block {block.id}: inverted cell at interior index {tuple(bad)}")
    return m


def _metrics_2d(block):
    # mesh.py:250-284: shoelace areas, corner-average centres, edge normals.
    x, y = block.nodes[0], block.nodes[1]
    g = block.ghost_depth
    ni, nj, _ = block.dims
    xa, ya = x[:-1, :-1], y[:-1, :-1]      # corner (0,0)
    xb, yb = x[1:, :-1], y[1:, :-1]        # corner (1,0)
    xc, yc = x[1:, 1:], y[1:, 1:]          # corner (1,1)
    xd, yd = x[:-1, 1:], y[:-1, 1:]        # corner (0,1)
    area = 0.5 * ((xa * yb - xb * ya) + (xb * yc - xc * yb)
                  + (xc * yd - xd * yc) + (xd * ya - xa * yd))
    volume = np.asfortranarray(area[..., None])
    cx = 0.25 * (xa + xb + xc + xd)
    cy = 0.25 * (ya + yb + yc + yd)
    centers = np.stack([cx[..., None], cy[..., None], np.zeros_like(cx)[..., None]])

    xi, yi = x[g:g + ni + 1, :], y[g:g + ni + 1, :]
    dx, dy = xi[:, 1:] - xi[:, :-1], yi[:, 1:] - yi[:, :-1]
    fv_i = np.stack([dy, -dx, np.zeros_like(dx)])[..., None]
    xj, yj = x[:, g:g + nj + 1], y[:, g:g + nj + 1]
    dx, dy = xj[1:, :] - xj[:-1, :], yj[1:, :] - yj[:-1, :]
    fv_j = np.stack([-dy, dx, np.zeros_like(dx)])[..., None]
    return BlockMetrics(volume=volume, centers=centers, face_vectors=[fv_i, fv_j, None],
                        ghost=block.ghost)


def _cross0(a, b):
    """Cross product over axis 0 with numpy.cross's operation order."""
    return np.stack([a[1] * b[2] - a[2] * b[1],
                     a[2] * b[0] - a[0] * b[2],
                     a[0] * b[1] - a[1] * b[0]])


def _sum3(v):
    return (v[0] + v[1]) + v[2]


# Corner orderings per face direction; normals point toward +axis (mesh.py:294-298).
_FACE_CORNERS = {
    0: ((0, 0, 0), (0, 1, 0), (0, 1, 1), (0, 0, 1)),
    1: ((0, 0, 0), (0, 0, 1), (1, 0, 1), (1, 0, 0)),
    2: ((0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0)),
}


def _metrics_3d(block):
    # mesh.py:287-331: divergence-theorem volumes over two triangles per quad.
    x, y, z = block.nodes
    g = block.ghost_depth
    dims = block.dims
    cshape = tuple(s - 1 for s in x.shape)

    def corner(off):
        sl = tuple(slice(o, o + n) for o, n in zip(off, cshape))
        return np.stack([x[sl], y[sl], z[sl]])

    def tri_flux(c0, c1, c2, c3):
        t1 = 0.5 * _cross0(c1 - c0, c2 - c0)
        t2 = 0.5 * _cross0(c2 - c0, c3 - c0)
        g1 = (c0 + c1 + c2) / 3.0
        g2 = (c0 + c2 + c3) / 3.0
        return (_sum3(g1 * t1) + _sum3(g2 * t2)) / 3.0

    volume = None
    for d, order in _FACE_CORNERS.items():
        lo = tri_flux(*(corner(c) for c in order))
        hi = tri_flux(*(corner(tuple(c[a] + (a == d) for a in range(3))) for c in order))
        part = hi - lo
        volume = part if volume is None else volume + part
    volume = np.asfortranarray(volume)

    centers = np.zeros((3, *cshape))
    for di in (0, 1):
        for dj in (0, 1):
            for dk in (0, 1):
                centers += corner((di, dj, dk))
    centers /= 8.0

    face_vectors = []
    for d, order in _FACE_CORNERS.items():
        picks = []
        for cidx in order:
            sl = tuple(slice(g, g + dims[a] + 1) if a == d
                       else slice(cidx[a], cidx[a] + dims[a] + 2 * g) for a in range(3))
            picks.append(np.stack([x[sl], y[sl], z[sl]]))
        c0, c1, c2, c3 = picks
        face_vectors.append(0.5 * _cross0(c2 - c0, c3 - c1))
    return BlockMetrics(volume=volume, centers=centers, face_vectors=face_vectors,
                        ghost=block.ghost)


def face_gradient_matrix(block, metrics, d):
    """Laminar NS face matrices of direction d (solver.py:582-642), shape
    (3, 3, N_d+1, interior tangential): out[r, e] = (J^-1)^T where column e
    of J is the centre-to-centre difference across the face (e = d) or the
    mid-edge node difference along the face (e != d).  Same numpy operations
    as the reference (incl. np.linalg.inv), so the device's viscous fluxes are
    computed from bit-identical matrices."""
    g, n, ndim = block.ghost, block.dims, block.ndim
    dirs = tuple(range(ndim))
    cen = metrics.centers
    inner = [slice(g[a], g[a] + n[a]) for a in range(3)]

    def along_d(lo, hi, arr, lead=True):
        cut = list(inner)
        cut[d] = slice(lo, hi)
        return arr[(slice(None), *cut)] if lead else arr[tuple(cut)]

    col = {d: along_d(g[d], g[d] + n[d] + 1, cen) - along_d(g[d] - 1, g[d] + n[d], cen)}
    if ndim == 3:
        xyz = tuple(block.nodes)
    else:
        xyz = (block.nodes[0][..., None], block.nodes[1][..., None])
        xyz = xyz + (np.zeros_like(xyz[0]),)

    def bump(cut, axis):
        out = list(cut)
        out[axis] = slice(cut[axis].start + 1, cut[axis].stop + 1)
        return out

    for e in dirs:
        if e == d:
            continue
        base = [slice(g[a], g[a] + n[a]) for a in range(3)]
        base[d] = slice(g[d], g[d] + n[d] + 1)
        rest = [a for a in dirs if a not in (d, e)]
        up = bump(base, e)
        comps = []
        for x in xyz:
            if rest:
                hi = 0.5 * (x[tuple(up)] + x[tuple(bump(up, rest[0]))])
                lo = 0.5 * (x[tuple(base)] + x[tuple(bump(base, rest[0]))])
            else:
                hi, lo = x[tuple(up)], x[tuple(base)]
            comps.append(hi - lo)
        col[e] = np.stack(comps)
    shape = col[d].shape[1:]
    J = np.zeros((*shape, ndim, ndim))
    for c, e in enumerate(dirs):
        for r in range(ndim):
            J[..., r, c] = col[e][r]
    inv_t = np.linalg.inv(J).swapaxes(-1, -2)
    out = np.zeros((3, 3, *shape))
    for r in range(ndim):
        for c, e in enumerate(dirs):
            out[r, e] = inv_t[..., r, c]
    return out


# ---------------------------------------------------------------------------
# Case grids (mesh.py:433-601) and the multi-parent 2D channel of SURVEY §8d C2
# ---------------------------------------------------------------------------

def make_cartesian_block(block_id, dims, lo, hi, ndim):
    axes = [np.linspace(lo[a], hi[a], dims[a] + 1) for a in range(ndim)]
    return Block(block_id, np.stack(np.meshgrid(*axes, indexing="ij")), ndim)


def full_face_box(dims, face):
    ax, side = face_axis(face), face_side(face)
    box = [(0, dims[a]) for a in range(3)]
    box[ax] = (0, 1) if side == 0 else (dims[ax] - 1, dims[ax])
    return tuple(box)


def physical_patch(block_id, face, dims, bc_type):
    return BoundarySpec(kind="physical", block=block_id, face=face,
                        box=full_face_box(dims, face), bc_type=bc_type)


def generate_case_grid(case, level=0):
    builders = {"inlet_ramp_2d": inlet_ramp_2d, "c_annulus_2d": c_annulus_2d,
                "multiblock_box_3d": multiblock_box_3d, "cartesian_box": cartesian_box_2d}
    if case not in builders:
        raise ValueError(f"unknown case preset {case!r}; choose from {CASE_PRESETS}")
    return builders[case](level)


def _ramp_nodes(ni, nj, x_end=1.8):
    """Channel with a 30-degree compression on the top wall (mesh.py:465-478)."""
    xs = np.linspace(0.0, x_end, ni + 1)
    top = 1.0 - np.tan(np.radians(30.0)) * np.clip(xs - 1.0, 0.0, 0.52)
    eta = np.linspace(0.0, 1.0, nj + 1)
    X = np.repeat(xs[:, None], nj + 1, axis=1)
    Y = eta[None, :] * top[:, None]
    return np.stack([X, Y])


def inlet_ramp_2d(level=0, ni=None, nj=None):
    """Inlet ramp; level L is (52*2^L) x (16*2^L) cells.  `ni, nj` override the
    preset sizes (SURVEY §8d C1 uses 128 x 64 with the same formula)."""
    ni = 52 * 2 ** level if ni is None else ni
    nj = 16 * 2 ** level if nj is None else nj
    blk = Block(0, _ramp_nodes(ni, nj), 2)
    d = blk.dims
    bcs = [physical_patch(0, "i_min", d, "supersonic_inflow"),
           physical_patch(0, "i_max", d, "supersonic_outflow"),
           physical_patch(0, "j_min", d, "slip_wall"),
           physical_patch(0, "j_max", d, "slip_wall")]
    return MultiBlockGrid(blocks=[blk], boundaries=bcs)


def _midpoint_refine(nodes, times):
    """Dyadic midpoint subdivision of a (ncomp, ni+1, nj+1) lattice (mesh.py:489-511)."""
    for _ in range(times):
        for axis in (1, 2):
            n = nodes.shape[axis]
            shape = list(nodes.shape)
            shape[axis] = 2 * n - 1
            out = np.empty(shape)
            ev = [slice(None)] * nodes.ndim
            od = [slice(None)] * nodes.ndim
            lo = [slice(None)] * nodes.ndim
            hi = [slice(None)] * nodes.ndim
            ev[axis], od[axis] = slice(0, None, 2), slice(1, None, 2)
            lo[axis], hi[axis] = slice(0, n - 1), slice(1, n)
            out[tuple(ev)] = nodes
            out[tuple(od)] = 0.5 * (nodes[tuple(lo)] + nodes[tuple(hi)])
            nodes = out
    return nodes


def c_annulus_2d(level=0, wall="slip_wall"):
    """Self-connected annulus (mesh.py:514-534)."""
    theta = np.linspace(0.0, -2.0 * np.pi, 65)
    radius = np.linspace(0.5, 2.0, 17)
    TH, RR = np.meshgrid(theta, radius, indexing="ij")
    nodes = _midpoint_refine(np.stack([RR * np.cos(TH), RR * np.sin(TH)]), level)
    blk = Block(0, nodes, 2)
    d = blk.dims
    a, b = make_connected_pair(0, "i_min", full_face_box(d, "i_min"),
                               0, "i_max", full_face_box(d, "i_max"), link_id=0)
    bcs = [a, b, physical_patch(0, "j_min", d, wall), physical_patch(0, "j_max", d, "farfield")]
    return MultiBlockGrid(blocks=[blk], boundaries=bcs)


def multiblock_box_3d(level=0):
    """Four unequal boxes tiling the unit cube, 4:2:1:1 (mesh.py:537-589).
    Level 15 is 256^3 cells in total."""
    ref = [4, 4, 4]
    for lv in range(level):
        ref[2 - (lv % 3)] *= 2
    rx, ry, rz = ref
    blocks = [
        make_cartesian_block(0, (rx, 2 * ry, 2 * rz), (0.0, 0.0, 0.0), (0.5, 1.0, 1.0), 3),
        make_cartesian_block(1, (rx, ry, 2 * rz), (0.5, 0.0, 0.0), (1.0, 0.5, 1.0), 3),
        make_cartesian_block(2, (rx, ry, rz), (0.5, 0.5, 0.0), (1.0, 1.0, 0.5), 3),
        make_cartesian_block(3, (rx, ry, rz), (0.5, 0.5, 0.5), (1.0, 1.0, 1.0), 3),
    ]
    d0, d1, d2 = blocks[0].dims, blocks[1].dims, blocks[2].dims
    bcs = []

    def connect(ba, fa, boxa, bb, fb, boxb):
        bcs.extend(make_connected_pair(ba, fa, boxa, bb, fb, boxb, link_id=len(bcs) // 2))

    i0 = (d0[0] - 1, d0[0])
    connect(0, "i_max", (i0, (0, ry), (0, 2 * rz)), 1, "i_min", ((0, 1), (0, ry), (0, 2 * rz)))
    connect(0, "i_max", (i0, (ry, 2 * ry), (0, rz)), 2, "i_min", ((0, 1), (0, ry), (0, rz)))
    connect(0, "i_max", (i0, (ry, 2 * ry), (rz, 2 * rz)), 3, "i_min", ((0, 1), (0, ry), (0, rz)))
    j1 = (d1[1] - 1, d1[1])
    connect(1, "j_max", ((0, rx), j1, (0, rz)), 2, "j_min", ((0, rx), (0, 1), (0, rz)))
    connect(1, "j_max", ((0, rx), j1, (rz, 2 * rz)), 3, "j_min", ((0, rx), (0, 1), (0, rz)))
    connect(2, "k_max", ((0, rx), (0, ry), (d2[2] - 1, d2[2])),
            3, "k_min", ((0, rx), (0, ry), (0, 1)))
    covered = {(s.block, s.face) for s in bcs}
    for b in blocks:
        for face in ("i_min", "i_max", "j_min", "j_max", "k_min", "k_max"):
            if (b.id, face) not in covered:
                bcs.append(physical_patch(b.id, face, b.dims, "farfield"))
    return MultiBlockGrid(blocks=blocks, boundaries=bcs)


def cartesian_box_2d(level=0):
    """Unit square with MMS Dirichlet faces (mesh.py:592-601)."""
    ref = [8, 8]
    for lv in range(level):
        ref[1 - (lv % 2)] *= 2
    blk = make_cartesian_block(0, tuple(ref), (0.0, 0.0), (1.0, 1.0), 2)
    d = blk.dims
    return MultiBlockGrid(blocks=[blk], boundaries=[
        physical_patch(0, f, d, "mms_dirichlet") for f in ("i_min", "i_max", "j_min", "j_max")])


def cartesian_box_3d(n, mms=True):
    """Unit cube of n^3 cells, MMS Dirichlet or farfield faces."""
    blk = make_cartesian_block(0, (n, n, n), (0.0, 0.0, 0.0), (1.0, 1.0, 1.0), 3)
    kind = "mms_dirichlet" if mms else "farfield"
    return MultiBlockGrid(blocks=[blk], boundaries=[
        physical_patch(0, f, blk.dims, kind) for f in
        ("i_min", "i_max", "j_min", "j_max", "k_min", "k_max")])


def ramp_channel_2d(parents=4, ni=512, nj=256, subsonic=False):
    """`parents` blocks of ni x nj cells cut along i from one
    (parents*ni) x nj compression-ramp lattice, joined i_max -> i_min.  Walls
    on j; supersonic inflow/outflow ends, or farfield ends when subsonic."""
    nodes = _ramp_nodes(parents * ni, nj)
    blocks, bcs = [], []
    for p in range(parents):
        blocks.append(Block(p, nodes[:, p * ni:(p + 1) * ni + 1, :], 2))
    for p in range(parents - 1):
        d = blocks[p].dims
        bcs.extend(make_connected_pair(p, "i_max", full_face_box(d, "i_max"),
                                       p + 1, "i_min", full_face_box(blocks[p + 1].dims, "i_min"),
                                       link_id=p))
    bcs.append(physical_patch(0, "i_min", blocks[0].dims,
                              "farfield" if subsonic else "supersonic_inflow"))
    bcs.append(physical_patch(parents - 1, "i_max", blocks[-1].dims,
                              "farfield" if subsonic else "supersonic_outflow"))
    for p in range(parents):
        bcs.append(physical_patch(p, "j_min", blocks[p].dims, "slip_wall"))
        bcs.append(physical_patch(p, "j_max", blocks[p].dims, "slip_wall"))
    return MultiBlockGrid(blocks=blocks, boundaries=bcs)
