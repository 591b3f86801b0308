"""ctypes binding of libbfgpu.so (include/bfgpu.h).

The library is the only compute path: if it is missing or fails to load,
:func:`lib` raises :class:`NativeLibraryError`; nothing falls back to the CPU.
"""

from __future__ import annotations

import ctypes as C
import os
import re
from pathlib import Path

from .errors import NativeLibraryError

LIB_PATH = Path(__file__).resolve().parent / "libbfgpu.so"
HEADER = Path(__file__).resolve().parent.parent / "include" / "bfgpu.h"

BF_OK, BF_EINVAL, BF_ECUDA, BF_ENONPHYSICAL, BF_ENCCL, BF_EMETRIC = 0, 1, 2, 3, 4, 5
FLUX = {"roe": 0, "van_leer": 1}
LIMITER = {"none": 0, "van_leer": 1, "van_albada": 2, "minmod": 3}
BC = {"supersonic_inflow": 0, "supersonic_outflow": 1, "slip_wall": 2, "noslip_wall": 3,
      "farfield": 4, "mms_dirichlet": 5}
FACES = ("i_min", "i_max", "j_min", "j_max", "k_min", "k_max")
FIELD = {"rho": 0, "u": 1, "v": 2, "w": 3, "p": 4, "T": 5, "dtv": 11}
FIELD_Q0, FIELD_PSI = 6, 12
FIELD_VOL, FIELD_FACE = 50, 51
ERR_FACE_LEFT, ERR_FACE_RIGHT, ERR_ROE_A2, ERR_UPDATE = 1, 2, 3, 4
PRECISION = {"exact": 0, "fast": 1}


class Gas(C.Structure):
    _fields_ = [("gamma", C.c_double), ("R", C.c_double), ("mu", C.c_double),
                ("prandtl", C.c_double), ("has_sutherland", C.c_int),
                ("sutherland", C.c_double * 3)]


class Freestream(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("rho", "u", "v", "w", "p", "T")]


class Scheme(C.Structure):
    _fields_ = [("flux", C.c_int), ("limiter", C.c_int), ("epsilon", C.c_double),
                ("kappa", C.c_double), ("rk_stages", C.c_int), ("cfl", C.c_double),
                ("limiter_freeze_at", C.c_int), ("entropy_fix_coeff", C.c_double),
                ("has_wall_temperature", C.c_int), ("wall_temperature", C.c_double),
                ("precision", C.c_int), ("viscous", C.c_int)]


_P = C.c_void_p
_I = C.c_int
_PD = C.POINTER(C.c_double)
_PI = C.POINTER(C.c_int)
_PLL = C.POINTER(C.c_longlong)
_PPD = C.POINTER(_PD)

PROTOTYPES = {
    "bf_api_version": (_I, []),
    "bf_create": (_P, [_I, C.POINTER(Gas), C.POINTER(Scheme), C.POINTER(Freestream), _I, _I, _I]),
    "bf_destroy": (None, [_P]),
    "bf_last_error": (_I, [_P, C.c_char_p, C.c_size_t]),
    "bf_add_block": (_I, [_P, _I, _PI, _I, _PPD, _PD, _PPD]),
    "bf_add_block_nodes": (_I, [_P, _I, _PI, _I, _PPD, _PLL, _PPD]),
    "bf_sync_blocks": (_I, [_P]),
    "bf_add_bc_patch": (_I, [_P, _I, _I, _I, _PI, _PD]),
    "bf_add_bc_patch_ext": (_I, [_P, _I, _I, _I, _PI, _PD, _PD]),
    "bf_add_viscous_geometry": (_I, [_P, _I, _PPD]),
    "bf_set_round2_order": (_I, [_P, _I, _PI]),
    "bf_add_link": (_I, [_P, _I, _I, _PI, _PI, _I, _I, _PI, _I, _I]),
    "bf_finalize": (_I, [_P]),
    "bf_upload_fields": (_I, [_P, _I, _PPD, _PPD]),
    "bf_update_ghosts": (_I, [_P]),
    "bf_step": (_I, [_P, _I, _PD, _PLL]),
    "bf_run": (_I, [_P, _I, _I, _PD, _PI]),
    "bf_iterate": (_I, [_P, _I, _I, _I, C.c_double, _I, C.c_double, C.c_double, _PD, _PI, _PI]),
    "bf_download": (_I, [_P, _I, _I, _PD]),
    "bf_error_info": (_I, [_P, _PI, _PI, _PI, _PI, _PLL]),
    "bf_nccl_unique_id": (_I, [_P]),
    "bf_nccl_init": (_I, [_P, _P]),
    "bf_loopback_create": (_P, [_I]),
    "bf_loopback_init": (_I, [_P, _P]),
    "bf_loopback_abort": (None, [_P]),
    "bf_loopback_destroy": (None, [_P]),
    "bf_group_create": (_P, [C.POINTER(_P), _I]),
    "bf_group_destroy": (None, [_P]),
    "bf_group_update_ghosts": (_I, [_P]),
    "bf_group_step": (_I, [_P, _I, _PD, _PI]),
    "bf_set_stream": (_I, [_P, _P]),
    "bf_set_profiling": (_I, [_P, _I]),
    "bf_kernel_stats": (_I, [_P, _I, _PLL, _PD]),
    "bf_transfer_bytes": (C.c_longlong, [_P, _I]),
    "bf_release_cache": (None, [_I]),
    "bf_cache_bytes": (C.c_longlong, [_I]),
    "bf_transfer_counters": (_I, [_P, _PLL]),
    "bf_probe_remote_order": (_I, [_I, _PI, _PI, _PI, _PI]),
    "bf_probe_unpack_map": (_I, [_PI, _I, _I, _I, _PI, _PI, _I, _PLL, C.c_longlong]),
}

_lib = None


def declared_symbols():
    """Function names declared in include/bfgpu.h."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(bf_[a-z0-9_]+)\s*\(", text)))


def lib():
    """The loaded library (raises NativeLibraryError when unavailable)."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("BFGPU_LIB", LIB_PATH))
    if not path.exists():
        raise NativeLibraryError(
            f"{path} is missing: build it with `python -m paper_2012_02925_b200.build` "
            "(there is no CPU fallback)")
    try:
        handle = C.CDLL(str(path))
    except OSError as exc:
        raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    if handle.bf_api_version() != 1:
        raise NativeLibraryError("libbfgpu.so API version mismatch")
    _lib = handle
    return _lib


def ints(values):
    arr = (C.c_int * len(values))(*[int(v) for v in values])
    return arr


def dptr(arr):
    return arr.ctypes.data_as(_PD)


def dptrs(arrays):
    return (_PD * len(arrays))(*[dptr(a) if a is not None else None for a in arrays])


def last_error(ctx):
    buf = C.create_string_buffer(2048)
    lib().bf_last_error(ctx, buf, len(buf))
    return buf.value.decode(errors="replace")
