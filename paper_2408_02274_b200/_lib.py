"""ctypes binding of libifgfb200.so (the C ABI in include/ifgfb.h).

The library is built in-tree by ``paper_2408_02274_b200.build.build()``.
Importing this module never falls back to CPU code: if the shared object is
missing or no CUDA device is usable, the compute entry points raise.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

import os

# IFGFB_LIB overrides the in-tree library (used to A/B kernel variants)
LIB_PATH = Path(os.environ.get("IFGFB_LIB") or
                Path(__file__).resolve().parent / "libifgfb200.so")

KERNEL_KINDS = ("leaf", "propagate", "emit", "emit_reduce", "near",
                "pack", "assemble", "other")

IFGFB_OK = 0
IFGFB_ERR_ARG = -1

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)


class TreeDesc(C.Structure):
    _fields_ = [("n_points", C.c_int32), ("depth", C.c_int32),
                ("p_s", C.c_int32), ("p_a", C.c_int32),
                ("points_tree", _dp), ("perm", _ip)]


class LevelDesc(C.Structure):
    _fields_ = [("level", C.c_int32), ("n_boxes", C.c_int32),
                ("n_s", C.c_int32), ("n_a", C.c_int32),
                ("side", C.c_double), ("h", C.c_double),
                ("delta_s", C.c_double), ("delta_a", C.c_double),
                ("centers", _dp), ("pt_start", _ip), ("pt_count", _ip),
                ("n_segments", C.c_int64), ("seg_off", _ip), ("seg_ids", _ip),
                ("s_nodes", _dp), ("sin_t", _dp), ("cos_t", _dp),
                ("sin_p", _dp), ("cos_p", _dp)]


class EmitDesc(C.Structure):
    _fields_ = [("level", C.c_int32), ("n_pairs", C.c_int64),
                ("row", _ip), ("target", _ip), ("geom", _dp),
                ("geom_disp", _dp)]


class AccumDesc(C.Structure):
    _fields_ = [("level", C.c_int32), ("n_types", C.c_int64),
                ("node_geom", _dp), ("node_r", _dp),
                ("n_parent_rows", C.c_int64),
                ("row_order", C.POINTER(C.c_uint8)),
                ("row_cuts", C.POINTER(C.c_uint8)),
                ("inst_off", _ip), ("n_instances", C.c_int64),
                ("inst_type", _ip), ("inst_crow_off", _ip), ("crow", _ip),
                ("tile_off", _ip), ("n_tiles", C.c_int64),
                ("tiles", C.POINTER(C.c_uint8)),
                ("geometry_on_device", C.c_int32),
                ("type_octant", C.POINTER(C.c_uint8)),
                ("group_id", C.POINTER(C.c_uint8))]


class SurfaceDesc(C.Structure):
    _fields_ = [("n_patches", C.c_int32), ("n_c", C.c_int32),
                ("points", _dp), ("normals", _dp), ("weights", _dp),
                ("jacobians", _dp), ("e_u", _dp), ("e_v", _dp),
                ("tangent1", _dp), ("tangent2", _dp),
                ("diff_matrix", _dp), ("coeff_matrix", _dp),
                ("eps_e", _dp), ("mu_e", _dp), ("eps_i", _dp), ("mu_i", _dp),
                ("omega", C.c_double), ("kappas", _dp),
                ("fd_step", C.c_double)]


class NearDesc(C.Structure):
    _fields_ = [("n_mom", C.c_int64), ("mom_off", _ip), ("mom_patch", _ip),
                ("moments", _dp), ("n_direct", C.c_int64), ("dir_off", _ip),
                ("dir_src", _ip)]


class LevelPart(C.Structure):
    _fields_ = [("level", C.c_int32), ("seg_lo", C.c_int64),
                ("seg_hi", C.c_int64), ("pair_lo", C.c_int64),
                ("pair_hi", C.c_int64)]


class PartitionDesc(C.Structure):
    _fields_ = [("n_levels", C.c_int32), ("levels", C.POINTER(LevelPart)),
                ("target_lo", C.c_int64), ("target_hi", C.c_int64)]


class RankDesc(C.Structure):
    _fields_ = [("target_lo", C.c_int64), ("target_hi", C.c_int64),
                ("chunk", C.c_int64), ("rank", C.c_int32), ("n_ranks", C.c_int32)]


class ConeLevelDesc(C.Structure):
    _fields_ = [("n_s", C.c_int32), ("n_a", C.c_int32), ("delta_s", C.c_double),
                ("delta_a", C.c_double), ("s_num", C.c_double), ("n_boxes", C.c_int64),
                ("amb_capacity", C.c_int64)]


class ConeParentDesc(C.Structure):
    _fields_ = [("n_boxes", C.c_int64), ("inst_off", _ip), ("row0", _ip),
                ("parent_box", C.POINTER(C.c_int32)), ("n_parent_rows", C.c_int64),
                ("parent_seg_ids", C.POINTER(C.c_int32)), ("n_parent_boxes", C.c_int64),
                ("parent_centers", _dp), ("centers", _dp), ("pn_s", C.c_int32),
                ("pn_a", C.c_int32), ("ph", C.c_double), ("parent_tabs", _dp)]


class AccumTypesDesc(C.Structure):
    _fields_ = [("n_types", C.c_int64), ("gamma", C.POINTER(C.c_int32)),
                ("octant", C.POINTER(C.c_uint8)), ("pn_s", C.c_int32), ("pn_a", C.c_int32),
                ("ph", C.c_double), ("parent_tabs", _dp), ("n_s", C.c_int32),
                ("n_a", C.c_int32), ("delta_s", C.c_double), ("delta_a", C.c_double),
                ("s_num", C.c_double), ("half", C.c_double)]


class MomentDesc(C.Structure):
    _fields_ = [("n_pairs", C.c_int64), ("target_xyz", _dp), ("target_nrm", _dp),
                ("patch", C.POINTER(C.c_int32)), ("uv", _dp),
                ("n_patches", C.c_int32), ("n_p", C.c_int32),
                ("patch_coeffs", _dp), ("n_c", C.c_int32),
                ("n_beta", C.c_int32), ("grading", C.c_int32),
                ("base", _dp), ("weights", _dp), ("kappas", _dp),
                ("nodes", _dp), ("gemm_tail_u", C.c_int32), ("gemm_tail_v", C.c_int32)]


EXPORTS = {
    "ifgfb_abi_version": ([], C.c_int),
    "ifgfb_last_error": ([], C.c_char_p),
    "ifgfb_device_info": ([C.c_char_p, C.c_size_t], C.c_int),
    "ifgfb_singular_moments": ([C.POINTER(MomentDesc), _dp], C.c_int),
    "ifgfb_plan_create": ([C.POINTER(TreeDesc), C.POINTER(C.c_void_p)], C.c_int),
    "ifgfb_plan_add_level": ([C.c_void_p, C.POINTER(LevelDesc)], C.c_int),
    "ifgfb_plan_add_accum": ([C.c_void_p, C.POINTER(AccumDesc)], C.c_int),
    "ifgfb_plan_set_emission": ([C.c_void_p, C.POINTER(EmitDesc)], C.c_int),
    "ifgfb_plan_set_surface": ([C.c_void_p, C.POINTER(SurfaceDesc)], C.c_int),
    "ifgfb_plan_set_near": ([C.c_void_p, C.POINTER(NearDesc)], C.c_int),
    "ifgfb_plan_finalize": ([C.c_void_p], C.c_int),
    "ifgfb_plan_destroy": ([C.c_void_p], C.c_int),
    "ifgfb_plan_device_bytes": ([C.c_void_p], C.c_int64),
    "ifgfb_plan_last_launches": ([C.c_void_p], C.c_int64),
    "ifgfb_plan_set_timing": ([C.c_void_p, C.c_int], C.c_int),
    "ifgfb_plan_kernel_times": ([C.c_void_p, _dp, _ip], C.c_int),
    "ifgfb_plan_level_times": ([C.c_void_p, C.c_int, _dp, _ip], C.c_int),
    "ifgfb_far_apply": ([C.c_void_p, C.c_void_p, C.c_int, _dp, C.c_int,
                         C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "ifgfb_potentials": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                          C.c_void_p], C.c_int),
    "ifgfb_muller_apply": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p],
                           C.c_int),
    "ifgfb_muller_apply_host": ([C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p], C.c_int),
    "ifgfb_zdotc": ([C.c_void_p, C.c_void_p, C.c_int64, _dp, C.c_void_p],
                    C.c_int),
    "ifgfb_dznrm2": ([C.c_void_p, C.c_int64, _dp, C.c_void_p], C.c_int),
    "ifgfb_zaxpy": ([_dp, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p],
                    C.c_int),
    "ifgfb_arnoldi_mgs": ([C.c_void_p, C.c_int64, C.c_int, C.c_int64,
                           C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "ifgfb_basis_combine": ([C.c_void_p, C.c_int64, C.c_int, C.c_int64,
                             C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "ifgfb_arnoldi_mgs_rows": ([C.c_void_p, C.c_int, C.c_int64, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "ifgfb_basis_combine_rows": ([C.c_void_p, C.c_int, C.c_int64, C.c_void_p,
                                  C.c_void_p, C.c_void_p], C.c_int),
    "ifgfb_plan_set_streaming": ([C.c_void_p, C.POINTER(PartitionDesc),
                                  C.c_int], C.c_int),
    "ifgfb_muller_far_phase": ([C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "ifgfb_muller_near_phase": ([C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p], C.c_int),
    "ifgfb_cones_begin": ([C.POINTER(ConeLevelDesc), C.POINTER(C.c_void_p)], C.c_int),
    "ifgfb_cones_mark_points": ([C.c_void_p, C.c_int64, C.POINTER(C.c_int32),
                                 C.POINTER(C.c_int32), C.c_int64, _dp, _dp], C.c_int),
    "ifgfb_cones_mark_parents": ([C.c_void_p, C.POINTER(ConeParentDesc)], C.c_int),
    "ifgfb_cones_ambiguous": ([C.c_void_p, C.POINTER(C.c_int64), _ip, _dp], C.c_int),
    "ifgfb_cones_set": ([C.c_void_p, C.c_int64, _ip, _ip], C.c_int),
    "ifgfb_cones_finish": ([C.c_void_p, _ip, C.c_void_p, C.POINTER(C.c_int64)], C.c_int),
    "ifgfb_cones_ids": ([C.c_void_p, _ip, _ip], C.c_int),
    "ifgfb_cones_free": ([C.c_void_p], C.c_int),
    "ifgfb_accum_types": ([C.POINTER(AccumTypesDesc), _u8p, C.POINTER(C.c_int32), _u8p,
                           _u8p, _dp, _dp], C.c_int),
    "ifgfb_plan_set_rank": ([C.c_void_p, C.POINTER(RankDesc)], C.c_int),
    "ifgfb_plan_rank_buffers": ([C.c_void_p] + [C.POINTER(C.c_void_p)] * 4
                                + [C.POINTER(C.c_int64)], C.c_int),
    "ifgfb_rank_unpack": ([C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "ifgfb_row_tiles_plan": ([C.c_int64, _ip, _ip, C.c_int64, _u8p, _u8p, _u8p,
                              _ip, C.c_int32, C.c_int32], C.c_int),
    "ifgfb_row_cuts_wide": ([C.c_int64, _ip, _ip, C.c_int64, _u8p, _u8p, _u8p,
                             C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32], C.c_int),
    "ifgfb_wide_warps": ([], C.c_int),
    "ifgfb_row_tiles_fill": ([C.c_int64, _ip, _ip, C.c_int64, _u8p, _u8p, _u8p,
                              _ip, _u8p, C.c_int32], C.c_int),
    "ifgfb_layer_fields": ([C.c_int64, _dp, C.c_int64, _dp, _dp, _dp, _dp],
                           C.c_int),
    "ifgfb_zscal_div": ([C.c_void_p, C.c_void_p, C.c_double, C.c_int64,
                         C.c_void_p], C.c_int),
}

ABI_VERSION = 8
_lib = None


def load():
    """Load the shared library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} missing: run paper_2408_02274_b200.build.build() "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    for name, (args, res) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.ifgfb_abi_version() != ABI_VERSION:
        raise RuntimeError("libifgfb200 ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc == IFGFB_OK:
        return
    msg = load().ifgfb_last_error().decode(errors="replace")
    if rc == IFGFB_ERR_ARG:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg} (code {rc})")


def dptr(a: np.ndarray):
    """double* of a C-contiguous float64/complex128 host array (or NULL)."""
    if a is None:
        return None
    assert a.flags.c_contiguous and a.dtype in (np.float64, np.complex128)
    return a.ctypes.data_as(_dp)


def u8ptr(a: np.ndarray):
    if a is None:
        return None
    assert a.flags.c_contiguous and a.dtype == np.uint8
    return a.ctypes.data_as(_u8p)


def iptr(a: np.ndarray):
    if a is None:
        return None
    assert a.flags.c_contiguous and a.dtype == np.int64
    return a.ctypes.data_as(_ip)
