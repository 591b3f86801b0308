"""The C-ABI library on the CPU: it loads, exports every symbol include/bfgpu.h
declares, fails loudly without a GPU, and its halo lowering is bit-exact.

Ghost indexing: bf_probe_unpack_map returns the affine map the device unpack
applies (recv-box cell -> partner send-box buffer index).  Applied to
index-encoded fields it must reproduce a cell-by-cell brute-force ghost fill
built from the orientation algebra (topology.py:138-161; halo.py:70-106) for
identity, flipped, same-side and cross-axis connections (the cases of the
reference's test_exchange.py:98-162), and the reference's own pack/unpack
when it is installed."""

import ctypes as C
import itertools

import numpy as np
import pytest

from paper_2012_02925_b200 import native
from paper_2012_02925_b200.errors import NativeLibraryError
from paper_2012_02925_b200.topology import FACES, halo_regions, make_connected_pair


def test_library_loads_and_exports_every_declared_symbol():
    L = native.lib()
    declared = native.declared_symbols()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(L, name), f"{name} declared in bfgpu.h but not exported"
    assert L.bf_api_version() == 1
    assert set(declared) == set(native.PROTOTYPES), "ctypes prototypes out of sync with bfgpu.h"


def test_no_silent_cpu_fallback():
    """Without a usable device the context cannot be created and the Python
    layer raises instead of computing anything on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2012_02925_b200 import geometry, planning
    from paper_2012_02925_b200.model import FreestreamState, GasModel, SchemeConfig
    from paper_2012_02925_b200.stepper import iterate_gpu
    gas = GasModel()
    plan = planning.decompose(geometry.inlet_ramp_2d(0), 1, 2)
    fs = FreestreamState.from_mach(gas, 4.0, 12270.0, 217.0, 0.0, 2)
    with pytest.raises(NativeLibraryError):
        iterate_gpu(plan, planning.reorder_boundaries(plan), gas, SchemeConfig(), fs, 1)


def index_fields(dims, ghost, scale=1.0, shift=0.0):
    idx = np.meshgrid(*[np.arange(-g, d + g) for d, g in zip(dims, ghost)], indexing="ij")
    base = idx[0] + 16.0 * idx[1] + 256.0 * idx[2]
    return {n: np.asfortranarray((base + 4096.0 * k) * scale + shift)
            for k, n in enumerate(("rho", "u", "v", "w", "p", "T"))}


def brute_force_fill(own, src, spec, partner, dims, pdims, ghost, pghost):
    """Per ghost cell: tangential coords through the owner->neighbour map,
    ghost depth g <- partner interior layer g counted from its face."""
    ax = spec.axis
    _, recv = halo_regions(spec, dims, ghost, 1)
    out = {k: v.copy() for k, v in own.items()}
    ndim = 2 if ghost[2] == 0 else 3
    names = ("rho", "u", "v", "p", "T") + (("w",) if ndim == 3 else ())
    for idx in itertools.product(*(range(lo, hi) for lo, hi in recv)):
        depth = (ghost[ax] - 1 - idx[ax]) if spec.side == 0 else (idx[ax] - ghost[ax] - dims[ax])
        cell = [idx[a] - ghost[a] for a in range(3)]
        cell[ax] = spec.box[ax][0]
        box = tuple((c, c + 1) for c in cell)
        mapped = [lo for lo, _ in spec.map_box(box)]
        pax = partner.axis
        mapped[pax] = depth if partner.side == 0 else pdims[pax] - 1 - depth
        sidx = tuple(mapped[a] + pghost[a] for a in range(3))
        for n in names:
            out[n][idx] = src[n][sidx]
    return out


def probe_map(spec, partner, dims, ghost, ndim):
    _, recv = halo_regions(spec, dims, ghost, 1)
    count = int(np.prod([hi - lo for lo, hi in recv]))
    out = (C.c_longlong * count)()
    rc = native.lib().bf_probe_unpack_map(
        native.ints(dims), ghost[0], ndim, FACES.index(spec.face),
        native.ints([x for r in spec.box for x in r]),
        native.ints([x for e in spec.axis_map for x in e]), FACES.index(partner.face), out, count)
    assert rc == 0
    return np.array(out[:]), recv


def device_fill(own, src, spec, partner, dims, pdims, ghost, pghost, ndim):
    """What the device does: pack the partner send box i-fastest, unpack with
    the lowered affine map."""
    send, _ = halo_regions(partner, pdims, pghost, 1)
    cut = tuple(slice(lo, hi) for lo, hi in send)
    m, recv = probe_map(spec, partner, dims, ghost, ndim)
    rcut = tuple(slice(lo, hi) for lo, hi in recv)
    shape = tuple(hi - lo for lo, hi in recv)
    out = {k: v.copy() for k, v in own.items()}
    names = ("rho", "u", "v", "p", "T") + (("w",) if ndim == 3 else ())
    for n in names:
        buf = src[n][cut].ravel(order="F")
        out[n][rcut] = buf[m].reshape(shape, order="F")
    return out


CASES = {
    "identity": (("i_max", ((7, 8), (0, 4), (0, 1)), "i_min", ((0, 1), (0, 4), (0, 1))),
                 ((0, 1), (1, 1), (2, 1)), (8, 4, 1), (8, 4, 1), 2),
    "flipped_j": (("i_max", ((7, 8), (0, 4), (0, 1)), "i_min", ((0, 1), (0, 4), (0, 1))),
                  ((0, 1), (1, -1), (2, 1)), (8, 4, 1), (8, 4, 1), 2),
    "same_side_mirror": (("i_min", ((0, 1), (0, 4), (0, 1)), "i_min", ((0, 1), (0, 4), (0, 1))),
                         ((0, 1), (1, -1), (2, 1)), (8, 4, 1), (6, 4, 1), 2),
    "cross_axis_3d": (("i_max", ((3, 4), (0, 5), (0, 6)), "j_min", ((0, 5), (0, 1), (0, 6))),
                      ((1, 1), (0, 1), (2, -1)), (4, 5, 6), (5, 4, 6), 3),
    "partial_patch": (("i_max", ((7, 8), (1, 5), (0, 1)), "i_min", ((0, 1), (1, 5), (0, 1))),
                      ((0, 1), (1, 1), (2, 1)), (8, 6, 1), (8, 6, 1), 2),
    "k_faces_flip_i": (("k_max", ((0, 4), (0, 3), (4, 5)), "k_min", ((0, 4), (0, 3), (0, 1))),
                       ((0, -1), (1, 1), (2, 1)), (4, 3, 5), (4, 3, 2), 3),
    "j_to_k_3d": (("j_max", ((0, 4), (2, 3), (0, 5)), "k_min", ((0, 5), (0, 4), (0, 1))),
                  ((1, -1), (2, 1), (0, 1)), (4, 3, 5), (5, 4, 3), 3),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_device_unpack_map_is_bit_exact(name):
    (fa, ba, fb, bb), amap, da, db, ndim = CASES[name]
    sa, sb = make_connected_pair(0, fa, ba, 1, fb, bb, axis_map=amap, link_id=0)
    ga = gb = (2, 2, 2 if ndim == 3 else 0)
    A = index_fields(da, ga)
    B = index_fields(db, gb, scale=1.5, shift=0.25)
    want = brute_force_fill(A, B, sa, sb, da, db, ga, gb)
    got = device_fill(A, B, sa, sb, da, db, ga, gb, ndim)
    for n in want:
        np.testing.assert_array_equal(got[n], want[n], err_msg=n)
    # and the other direction of the same link
    want2 = brute_force_fill(B, A, sb, sa, db, da, gb, ga)
    got2 = device_fill(B, A, sb, sa, db, da, gb, ga, ndim)
    for n in want2:
        np.testing.assert_array_equal(got2[n], want2[n], err_msg=n)


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_pack_unpack_matches_brute_force(name):
    import oracle
    (fa, ba, fb, bb), amap, da, db, ndim = CASES[name]
    sa, sb = make_connected_pair(0, fa, ba, 1, fb, bb, axis_map=amap, link_id=0)
    ga = gb = (2, 2, 2 if ndim == 3 else 0)
    A = index_fields(da, ga)
    B = index_fields(db, gb, scale=1.5, shift=0.25)
    got = {k: v.copy() for k, v in A.items()}
    oracle.unpack_face(oracle.pack_face(B, sb, db, gb), got, sa, da, ga, sb.side)
    want = brute_force_fill(A, B, sa, sb, da, db, ga, gb)
    for n in want:
        np.testing.assert_array_equal(got[n], want[n], err_msg=n)


@pytest.mark.parametrize("name", sorted(CASES))
def test_reference_pack_unpack_matches_device_map(name, ref):
    (fa, ba, fb, bb), amap, da, db, ndim = CASES[name]
    ra, rb = ref.topology.make_connected_pair(0, fa, ba, 1, fb, bb, axis_map=amap, link_id=0)
    sa, sb = make_connected_pair(0, fa, ba, 1, fb, bb, axis_map=amap, link_id=0)
    ga = gb = (2, 2, 2 if ndim == 3 else 0)
    A = index_fields(da, ga)
    B = index_fields(db, gb, scale=1.5, shift=0.25)
    got = {k: v.copy() for k, v in A.items()}
    ref.halo.unpack_face(ref.halo.pack_face(B, rb, db, gb, 1), got, ra, da, ga, rb.side, 1)
    dev = device_fill(A, B, sa, sb, da, db, ga, gb, ndim)
    for n in got:
        np.testing.assert_array_equal(dev[n], got[n], err_msg=n)
