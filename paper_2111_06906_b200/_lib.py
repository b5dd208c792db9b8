"""ctypes view of the C ABI in include/prx.h (the product's only compute path).

Loading fails loudly when the in-tree library ``_prx.so`` is missing: there is no CPU
fallback.  Struct layouts mirror prx.h field for field.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_prx.so")

MAX_LIGHTS = 16

PRX_OK = 0
PRX_E_INVALID_ARGUMENT = 1
PRX_E_OUT_OF_RANGE = 2
PRX_E_LOGIC = 3
PRX_E_SCENE = 4
PRX_E_RUNTIME = 5
PRX_E_CUDA = 6

MODES = {"baseline": 0, "naive": 1, "error": 2, "error_based": 2, "error-based": 2}
MODE_NAMES = {0: "baseline", 1: "naive", 2: "error"}

LIGHT_KINDS = {"point": 0, "spot": 1, "disc_area": 2, "rect_area": 3}
MATERIAL_KINDS = {"diffuse": 0, "glossy": 1}

FIELD = {
    "photons": 0, "aux": 1, "pos_obj": 2, "energy": 3, "in_dir": 4, "out_dir": 5,
    "origin": 6, "emission_dir": 7, "canonical": 8, "cell": 9, "epoch": 10,
    "path_info": 11, "meta": 12, "retrace_start": 13, "segment_flags": 14,
    "dm_target": 15, "dm_current": 16, "pruned": 17,
}

STAGE = {"update_origins": 0, "occlusions": 1, "compute_dm": 2, "prune": 3, "fill": 4,
         "trace": 5, "release_all": 6}


class Vec3(C.Structure):
    _fields_ = [("x", C.c_float), ("y", C.c_float), ("z", C.c_float)]


class Quat(C.Structure):
    _fields_ = [("x", C.c_float), ("y", C.c_float), ("z", C.c_float), ("w", C.c_float)]


class Triangle(C.Structure):
    _fields_ = [("a", Vec3), ("b", Vec3), ("c", Vec3)]


class Keyframe(C.Structure):
    _fields_ = [("frame", C.c_int32), ("rotation", Quat), ("translation", Vec3),
                ("scale", C.c_float)]


class Material(C.Structure):
    _fields_ = [("kind", C.c_int32), ("albedo", Vec3), ("glossy_exponent", C.c_float)]


class ObjectDesc(C.Structure):
    _fields_ = [("name", C.c_char_p), ("mesh", C.POINTER(Triangle)), ("n_triangles", C.c_uint32),
                ("material", Material), ("keyframes", C.POINTER(Keyframe)),
                ("n_keyframes", C.c_uint32)]


class LightDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("flux", Vec3), ("cone_angle_deg", C.c_float),
                ("radius", C.c_float), ("half_x", C.c_float), ("half_y", C.c_float),
                ("keyframes", C.POINTER(Keyframe)), ("n_keyframes", C.c_uint32)]


class Camera(C.Structure):
    _fields_ = [("position", Vec3), ("look_at", Vec3), ("fov_deg", C.c_float),
                ("width", C.c_uint32), ("height", C.c_uint32)]


class SceneDesc(C.Structure):
    _fields_ = [("objects", C.POINTER(ObjectDesc)), ("n_objects", C.c_uint32),
                ("lights", C.POINTER(LightDesc)), ("n_lights", C.c_uint32),
                ("camera", Camera), ("frames", C.c_int32)]


class Config(C.Structure):
    _fields_ = [("mode", C.c_int32), ("n_paths", C.c_uint32), ("max_bounces", C.c_uint32),
                ("dm_dims", C.c_uint32 * 4), ("threshold", C.c_float), ("seed", C.c_uint64),
                ("gather_radius", C.c_float), ("workers", C.c_uint32),
                ("record_flags", C.c_int32), ("device", C.c_int32),
                ("shard_begin", C.c_uint32), ("shard_end", C.c_uint32),
                ("exact_trig", C.c_int32), ("dfs_traversal", C.c_int32)]


class FrameStats(C.Structure):
    _fields_ = [("frame", C.c_int32), ("mode", C.c_int32),
                ("rays_traced", C.c_uint64), ("rays_reused", C.c_uint64),
                ("paths_replaced", C.c_uint64), ("paths_pruned", C.c_uint64),
                ("paths_filled", C.c_uint64), ("visibility_rays", C.c_uint64),
                ("t_update", C.c_double), ("t_occlusion", C.c_double), ("t_dm", C.c_double),
                ("t_prune", C.c_double), ("t_fill", C.c_double), ("t_trace", C.c_double),
                ("t_gather", C.c_double),
                ("ms_frame_update", C.c_double), ("ms_verify", C.c_double),
                ("ms_retrace", C.c_double), ("ms_splat", C.c_double),
                ("live_segments_before", C.c_uint64), ("paths_retraced", C.c_uint64)]

    COUNTS = ("rays_traced", "rays_reused", "paths_replaced", "paths_pruned", "paths_filled",
              "visibility_rays")

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class EngineInfo(C.Structure):
    _fields_ = [("n_paths", C.c_uint32), ("max_bounces", C.c_uint32), ("n_lights", C.c_uint32),
                ("shard_begin", C.c_uint32), ("shard_end", C.c_uint32),
                ("eps_world", C.c_float), ("diagonal", C.c_float), ("frames_run", C.c_int32),
                ("n_pruned", C.c_uint32),
                ("light_path_begin", C.c_uint32 * MAX_LIGHTS),
                ("light_path_end", C.c_uint32 * MAX_LIGHTS),
                ("dm_ndims", C.c_uint32 * MAX_LIGHTS),
                ("dm_dims", (C.c_uint32 * 4) * MAX_LIGHTS),
                ("dm_cells", C.c_uint32 * MAX_LIGHTS),
                ("flux_per_path", (C.c_float * 3) * MAX_LIGHTS),
                ("device_bytes", C.c_uint64)]


class Collectives(C.Structure):
    """prx_collectives (include/prx.h): the function pointers stay opaque to Python."""
    _fields_ = [("ctx", C.c_void_p), ("rank", C.c_int32), ("world", C.c_int32),
                ("all_reduce_sum_u32", C.c_void_p), ("all_reduce_sum_u64", C.c_void_p),
                ("all_reduce_sum_f32", C.c_void_p), ("all_gather_u32", C.c_void_p)]


# Every symbol include/prx.h declares: (name, restype, argtypes)
P = C.c_void_p
SIGNATURES = [
    ("prx_prune_probability", C.c_double, [C.c_uint32, C.c_uint32]),
    ("prx_energies_close", C.c_int, [C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_float]),
    ("prx_encode_path_info", C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_int,
                                       C.POINTER(C.c_uint32)]),
    ("prx_decode_path_info", None, [C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                    C.POINTER(C.c_uint32), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("prx_memory_footprint", None, [C.c_uint64, C.c_uint32, C.POINTER(C.c_uint32), C.c_uint32,
                                    C.c_int, C.POINTER(C.c_double)]),
    ("prx_select_paths_to_prune", C.c_int, [C.POINTER(C.c_uint32), C.c_size_t, C.c_uint32, C.c_uint32,
                                            C.c_uint64, C.c_uint32, C.POINTER(C.c_uint32),
                                            C.POINTER(C.c_size_t)]),
    ("prx_scene_create", C.c_int, [C.POINTER(SceneDesc), C.POINTER(P)]),
    ("prx_scene_builtin", C.c_int, [C.c_char_p, C.POINTER(P)]),
    ("prx_scene_load", C.c_int, [C.c_char_p, C.POINTER(P)]),
    ("prx_scene_load_text", C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(P)]),
    ("prx_scene_synthetic", C.c_int, [C.c_char_p, C.c_uint32, C.c_float, C.POINTER(P)]),
    ("prx_scene_describe", C.c_int, [P, C.POINTER(SceneDesc)]),
    ("prx_scene_bvh_permutation", C.c_int, [P, C.POINTER(C.c_uint32), C.c_size_t,
                                            C.POINTER(C.c_size_t)]),
    ("prx_scene_counts", C.c_int, [P, C.POINTER(C.c_uint64)]),
    ("prx_scene_diagonal", C.c_float, [P]),
    ("prx_scene_state_at", C.c_int, [P, C.c_int32, P, C.c_size_t, C.POINTER(C.c_size_t), P, C.c_size_t,
                                     C.POINTER(C.c_size_t)]),
    ("prx_scene_destroy", None, [P]),
    ("prx_engine_create", C.c_int, [P, C.POINTER(Config), C.POINTER(P)]),
    ("prx_engine_destroy", None, [P]),
    ("prx_engine_get_info", C.c_int, [P, C.POINTER(EngineInfo)]),
    ("prx_run_frame", C.c_int, [P, C.POINTER(FrameStats)]),
    ("prx_frame_update", C.c_int, [P, C.POINTER(FrameStats)]),
    ("prx_verify_paths", C.c_int, [P, C.POINTER(FrameStats)]),
    ("prx_retrace_invalid", C.c_int, [P, C.POINTER(FrameStats)]),
    ("prx_run_stage", C.c_int, [P, C.c_int, C.POINTER(FrameStats)]),
    ("prx_engine_dm_current", C.c_int, [P, C.c_uint32, C.POINTER(P), C.POINTER(C.c_uint32)]),
    ("prx_prune_count", C.c_int, [P, C.POINTER(C.POINTER(C.c_uint32))]),
    ("prx_prune_apply", C.c_int, [P, C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.POINTER(C.c_uint32)),
                                  C.POINTER(FrameStats)]),
    ("prx_fill_count", C.c_int, [P, C.POINTER(C.c_uint32)]),
    ("prx_fill_apply", C.c_int, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(FrameStats)]),
    ("prx_engine_set_collectives", C.c_int, [P, C.POINTER(Collectives)]),
    ("prx_group_create", C.c_int, [P, C.POINTER(Config), C.POINTER(C.c_int32), C.c_int32, C.POINTER(P)]),
    ("prx_group_run_frame", C.c_int, [P, C.POINTER(FrameStats)]),
    ("prx_group_splat", C.c_int, [P, C.POINTER(Camera), C.c_float, C.c_int, P]),
    ("prx_group_engine", P, [P, C.c_int32]),
    ("prx_group_size", C.c_int32, [P]),
    ("prx_group_destroy", None, [P]),
    ("prx_comm_nccl_unique_id", C.c_int, [C.POINTER(C.c_uint8)]),
    ("prx_comm_nccl_create", C.c_int, [C.POINTER(C.c_uint8), C.c_int32, C.c_int32, C.c_int32, C.POINTER(P)]),
    ("prx_comm_local_create", C.c_int, [C.c_int32, C.POINTER(P)]),
    ("prx_comm_collectives", C.c_int, [P, C.POINTER(Collectives)]),
    ("prx_comm_destroy", None, [P]),
    ("prx_engine_set_stream", C.c_int, [P, P]),
    ("prx_engine_synchronize", C.c_int, [P]),
    ("prx_engine_set_splat_overlap", C.c_int, [P, C.c_int32]),
    ("prx_splat", C.c_int, [P, C.POINTER(Camera), C.c_float, C.c_int, P, P,
                            C.POINTER(FrameStats)]),
    ("prx_gather_photons", C.c_int, [P, P, P, C.c_uint32, C.c_uint32, C.c_int32, C.POINTER(Camera),
                                     C.c_float, C.c_int, P]),
    ("prx_field_bytes", C.c_size_t, [P, C.c_int, C.c_uint32]),
    ("prx_engine_download", C.c_int, [P, C.c_int, C.c_uint32, P, C.c_size_t]),
    ("prx_engine_upload", C.c_int, [P, C.c_int, C.c_uint32, P, C.c_size_t]),
    ("prx_engine_set_frame_counter", C.c_int, [P, C.c_int32]),
    ("prx_intersect_batch", C.c_int, [P, C.POINTER(C.c_float), C.c_size_t, C.c_int, C.POINTER(C.c_float)]),
    ("prx_photon_dump_write", C.c_int, [C.c_char_p, C.c_uint32, C.c_uint32, P, C.c_size_t]),
    ("prx_photon_dump_read", C.c_int, [C.c_char_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), P,
                                       C.c_size_t]),
    ("prx_engine_write_photon_dump", C.c_int, [P, C.c_char_p]),
    ("prx_image_write_ppm", C.c_int, [C.c_char_p, C.POINTER(C.c_float), C.c_uint32, C.c_uint32]),
    ("prx_frame_image_name", C.c_size_t, [C.c_int32, C.c_char_p, C.c_size_t]),
    ("prx_stats_csv_write", C.c_int, [C.c_char_p, C.POINTER(FrameStats), C.c_size_t]),
    ("prx_stats_csv_read", C.c_int, [C.c_char_p, C.POINTER(FrameStats), C.c_size_t, C.POINTER(C.c_size_t)]),
    ("prx_reuse_report", C.c_int, [C.POINTER(FrameStats), C.c_size_t, C.c_char_p, C.c_size_t,
                                   C.POINTER(C.c_size_t)]),
    ("prx_engine_launch_count", C.c_uint64, [P]),
    ("prx_engine_transfer_bytes", C.c_int, [P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("prx_last_error", C.c_char_p, []),
    ("prx_abi_version", C.c_int, []),
]


class PrxError(RuntimeError):
    """Base of errors raised from C-ABI status codes."""


class SceneError(PrxError):
    """pathreuse::SceneError (scene.hpp:76)."""


class CudaError(PrxError):
    """A CUDA runtime failure inside the engine."""


def _exception_for(code: int, msg: str) -> Exception:
    if code == PRX_E_INVALID_ARGUMENT:
        return ValueError(msg)
    if code == PRX_E_OUT_OF_RANGE:
        return IndexError(msg)
    if code == PRX_E_SCENE:
        return SceneError(msg)
    if code == PRX_E_CUDA:
        return CudaError(msg)
    return PrxError(msg)


_lib = None


def lib() -> C.CDLL:
    """Load the engine library (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"B200 engine library missing: {LIB_PATH}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (make -C paper_2111_06906_b200)")
        handle = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(code: int) -> None:
    if code != PRX_OK:
        raise _exception_for(code, lib().prx_last_error().decode(errors="replace"))
