"""ctypes binding of libdpm_b200.so (the C ABI declared in include/dpm_b200.h).

The library is built in-tree (``make`` / ``__graft_entry__.build()``).  There
is no CPU fallback: if the library or a CUDA device is missing, the product
path raises :class:`DeviceError`.
"""

import ctypes
import os

import numpy as np

from .errors import DeviceError, NumericError, ValidationError

__all__ = ["lib", "check", "PROJ_JOB", "CORR_JOB", "CORR_TILE", "PLACE_JOB", "ASM_JOB", "SMAP_DESC",
           "DETECTION", "PLACE_RANGE", "PRUNE_JOB", "PRUNE_ASM", "COVER_JOB", "MIX_JOB", "LIB_PATH", "MAX_PARTS", "table_ptr"]

LIB_PATH = os.environ.get("DPM_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib",
                                                   "libdpm_b200.so")
MAX_PARTS = 16
ABI_VERSION = 4  # DPM_ABI_VERSION of include/dpm_b200.h

DPM_OK, DPM_ERR_ARG, DPM_ERR_UNSUPPORTED, DPM_ERR_CUDA, DPM_ERR_NUMERIC = 0, -1, -2, -3, -4

# numpy mirrors of the ABI structs (field order and C alignment as in the header)
PROJ_JOB = np.dtype([("x_off", "<i8"), ("p_off", "<i8"), ("H", "<i4"), ("W", "<i4"),
                     ("pitch", "<i4"), ("block0", "<i4")], align=True)
CORR_JOB = np.dtype([("p_off", "<i8"), ("s_off", "<i8"), ("g_off", "<i8"),
                     ("H", "<i4"), ("W", "<i4"), ("pitch", "<i4"), ("chan_off", "<i4"),
                     ("h", "<i4"), ("w", "<i4"), ("R", "<i4"), ("nf", "<i4"),
                     ("nf_pad", "<i4"), ("mode", "<i4"), ("range_idx", "<i4"), ("pad", "<i4")],
                    align=True)
CORR_TILE = np.dtype([("job", "<i4"), ("ty", "<i4"), ("tx", "<i4"), ("pad", "<i4")], align=True)
PLACE_JOB = np.dtype([("s_off", "<i8"), ("x_off", "<i8"), ("Hp", "<i4"), ("Wp", "<i4"),
                      ("ay", "<i4"), ("ax", "<i4"), ("scale", "<i4"), ("radius", "<i4"),
                      ("rx0", "<i4"), ("wr", "<i4"), ("range_idx", "<i4"), ("block0", "<i4"),
                      ("smap", "<i4"), ("smap_z", "<i4"),
                      ("cdx", "<f8"), ("cdy", "<f8"), ("cdxx", "<f8"), ("cdyy", "<f8")],
                     align=True)
ASM_JOB = np.dtype([("root_off", "<i8"), ("total_off", "<i8"), ("pos_off", "<i8"),
                    ("placed_off", "<i8"), ("root_pitch", "<i4"), ("ry0", "<i4"),
                    ("ry1", "<i4"), ("rx0", "<i4"), ("rx1", "<i4"), ("part_job0", "<i4"),
                    ("nparts", "<i4"), ("image", "<i4"), ("level", "<i4"),
                    ("component", "<i4"), ("block0", "<i4"), ("block1", "<i4"),
                    ("bias", "<f8")], align=True)
DETECTION = np.dtype([("image", "<i4"), ("level", "<i4"), ("component", "<i4"), ("ry", "<i4"),
                      ("rx", "<i4"), ("nparts", "<i4"), ("score", "<f8"),
                      ("parts", "<u4", (MAX_PARTS,))], align=True)

PLACE_RANGE = np.dtype([("rx", "<i4"), ("ry", "<i4"), ("E2", "<f4"), ("E2in", "<f4")], align=True)
PRUNE_JOB = np.dtype([("out_off", "<i8"), ("offs0", "<i4"), ("thr0", "<i4"), ("R", "<i4"),
                      ("Hp", "<i4"), ("Wp", "<i4"), ("ry0", "<i4"), ("ry1", "<i4"),
                      ("rx0", "<i4"), ("rx1", "<i4"), ("ay", "<i4"), ("ax", "<i4"),
                      ("scale", "<i4"), ("radius", "<i4"), ("block0", "<i4")], align=True)

PRUNE_ASM = np.dtype([("rank_off", "<i8"), ("lim_off", "<i8"), ("total_off", "<i8"),
                      ("pos_off", "<i8"), ("placed_off", "<i8"), ("root_off", "<i8"),
                      ("root_pitch", "<i4"), ("ry0", "<i4"), ("ry1", "<i4"), ("rx0", "<i4"),
                      ("rx1", "<i4"), ("nparts", "<i4"), ("image", "<i4"), ("level", "<i4"),
                      ("hist_off", "<i4"), ("block0", "<i4"), ("bias", "<f8"),
                      ("part_R", "<i4", (MAX_PARTS,)), ("ay", "<i4", (MAX_PARTS,)),
                      ("ax", "<i4", (MAX_PARTS,))], align=True)
COVER_JOB = np.dtype([("lim_off", "<i8"), ("hr", "<i4"), ("wr", "<i4"), ("y0", "<i4"),
                      ("y1", "<i4"), ("x0", "<i4"), ("x1", "<i4"), ("oy", "<i4"), ("ox", "<i4"),
                      ("radius", "<i4"), ("hist_off", "<i4"), ("block0", "<i4"), ("pad", "<i4")],
                     align=True)

MIX_JOB = np.dtype([("out_off", "<i8"), ("ry0", "<i4"), ("ry1", "<i4"), ("rx0", "<i4"),
                    ("rx1", "<i4"), ("member0", "<i4"), ("nmembers", "<i4"), ("block0", "<i4"),
                    ("pad", "<i4")], align=True)

SMAP_DESC = np.dtype([("s_off", "<i8"), ("Ho", "<i4"), ("Wo", "<i4"), ("nf", "<i4"),
                      ("pad", "<i4")], align=True)
SMAP_BYTES = 128
RESAMPLE_JOB = np.dtype([("img_off", "<i8"), ("out_off", "<i8"), ("H", "<i4"), ("W", "<i4"),
                         ("C", "<i4"), ("Hs", "<i4"), ("Ws", "<i4"), ("block0", "<i4")],
                        align=True)
HOG_JOB = np.dtype([("r_off", "<i8"), ("x_off", "<i8"), ("h_off", "<i8"), ("Hs", "<i4"),
                    ("Ws", "<i4"), ("C", "<i4"), ("block0", "<i4")], align=True)

_SIZES = {"PROJ_JOB": 32, "CORR_JOB": 72, "CORR_TILE": 16, "PLACE_JOB": 96, "ASM_JOB": 88,
          "SMAP_DESC": 24,
          "DETECTION": 96, "PLACE_RANGE": 16, "PRUNE_JOB": 64, "PRUNE_ASM": 288, "COVER_JOB": 56,
          "MIX_JOB": 40, "RESAMPLE_JOB": 40, "HOG_JOB": 40}
for _n, _s in _SIZES.items():
    assert globals()[_n].itemsize == _s, (_n, globals()[_n].itemsize)

_vp = ctypes.c_void_p
_i32 = ctypes.c_int
_i64 = ctypes.c_int64
_dbl = ctypes.c_double

_SIGNATURES = {
    "dpm_abi_version": (_i32, []),
    "dpm_last_error": (ctypes.c_char_p, []),
    "dpm_device_query": (_i32, [_i32, _vp, _vp, _vp]),
    "dpm_project_prepare": (_i64, [_vp, _i32]),
    "dpm_project": (_i32, [_vp, _vp, _vp, _i32, _i32, _vp, _i32, _i64, _vp]),
    "dpm_correlate_tile_shape": (_i32, [_i32, _i32, _vp, _vp]),
    "dpm_correlate": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp]),
    "dpm_ranges_init": (_i32, [_vp, _i32, _vp]),
    "dpm_correlate_prefix_tile": (_i32, [_vp, _vp]),
    "dpm_correlate_prefix_check": (_i32, [_vp, _i32]),
    "dpm_correlate_prefix": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp]),
    "dpm_correlate_tc_smem": (ctypes.c_size_t, [_i32, _i32, _i32, _i32]),
    "dpm_correlate_tc": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp]),
    "dpm_correlate_tc_groups": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32,
                                       _vp, _vp]),
    "dpm_correlate_tc_core_floats": (ctypes.c_size_t, [_i32, _i32, _i32, _i32]),
    "dpm_correlate_tc_stack": (_i32, [_i32, _i32, _i32, _i32]),
    "dpm_place_prepare": (_i64, [_vp, _i32]),
    "dpm_assemble_prepare": (_i64, [_vp, _i32, _vp, _i32, _vp]),
    "dpm_place_ranges": (_i32, [_vp, _i32, _vp, _vp, _vp]),
    "dpm_assemble": (_i32, [_vp, _vp, _vp, _vp, _i32, _i64, _i64, _vp, _vp, _vp, _vp, _dbl, _vp, _i32,
                            _vp, _vp]),
    "dpm_smap_encode": (_i32, [_vp, _vp, _i32, _vp]),
    "dpm_gdt_x_prepare": (_i64, [_vp, _i32]),
    "dpm_gdt_x": (_i32, [_vp, _vp, _vp, _vp, _i32, _i64, _vp, _vp]),
    "dpm_gdt_y_prepare": (_i64, [_vp, _i32, _vp, _i32]),
    "dpm_gdt_y": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, _i64, _vp, _vp, _vp, _vp, _dbl, _vp, _i32,
                         _vp, _vp]),
    "dpm_prune_prepare": (_i64, [_vp, _i32]),
    "dpm_prune_ranks": (_i32, [_vp, _vp, _vp, _vp, _i32, _i64, _vp, _vp]),
    "dpm_prune_compose_prepare": (_i64, [_vp, _i32]),
    "dpm_prune_compose": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i64, _i32, _dbl, _vp, _vp,
                                 _vp, _i32, _vp, _vp]),
    "dpm_prune_cover_prepare": (_i64, [_vp, _i32]),
    "dpm_prune_cover": (_i32, [_vp, _vp, _i32, _i64, _vp, _vp]),
    "dpm_mixture_prepare": (_i64, [_vp, _i32]),
    "dpm_mixture_max": (_i32, [_vp, _vp, _vp, _vp, _i32, _i64, _vp, _vp, _vp]),
    "dpm_ffma_probe": (_i32, [_vp, _i32, _vp, _vp]),
    "dpm_resample_prepare": (_i64, [_vp, _i32]),
    "dpm_resample": (_i32, [_vp, _i32, _vp, _vp, _i32, _i64, _vp]),
    "dpm_hog_prepare": (_i64, [_vp, _i32]),
    "dpm_hog": (_i32, [_vp, _vp, _vp, _vp, _i32, _i64, _vp]),
}

_lib = None


def lib():
    """Load (once) and return the CDLL; raises DeviceError if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
                "the B200 path has no CPU fallback")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.dpm_abi_version() != ABI_VERSION:
            raise DeviceError("libdpm_b200.so ABI version mismatch")
        _lib = handle
    return _lib


def check(status, what=""):
    """Map a dpm_status (or a negative prepare result) onto the error taxonomy."""
    if status >= 0:
        return status
    msg = lib().dpm_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status in (DPM_ERR_ARG, DPM_ERR_UNSUPPORTED):
        raise ValidationError(text)
    if status == DPM_ERR_NUMERIC:
        raise NumericError(text)
    raise DeviceError(text)


def table_ptr(arr):
    """Host pointer of a contiguous numpy structured array (for *_prepare)."""
    assert arr.flags["C_CONTIGUOUS"]
    return arr.ctypes.data_as(ctypes.c_void_p)
