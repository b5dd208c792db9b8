"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes wrapper over oracle/_ref/libpathreuse_ref.so -- the unmodified reference engine
(/root/reference/proj/src, compiled by oracle/Makefile) plus ref_shim.cpp.  Used by tests/,
``__graft_entry__.smoke()`` and bench.py's reference arm as the checker / CPU baseline;
never by the product.  Data crosses in the product's C-ABI layouts (include/prx.h), whose
ctypes structs are reused from paper_2111_06906_b200._lib (definitions only).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2111_06906_b200 import _lib as L
from paper_2111_06906_b200.pathreuse import AUX_DTYPE, PHOTON_DTYPE

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libpathreuse_ref.so")
ACCEPTANCE_BIN = os.path.join(HERE, "_ref", "acceptance")

_P = C.c_void_p
_SIGS = [
    ("prxref_last_error", C.c_char_p, []),
    ("prxref_scene_create", C.c_int, [C.POINTER(L.SceneDesc), C.POINTER(_P)]),
    ("prxref_scene_builtin", C.c_int, [C.c_char_p, C.POINTER(_P)]),
    ("prxref_scene_describe", C.c_int, [_P, C.POINTER(L.SceneDesc)]),
    ("prxref_scene_diagonal", C.c_float, [_P]),
    ("prxref_scene_bvh_permutation", C.c_int, [_P, C.POINTER(C.c_uint32), C.c_size_t,
                                               C.POINTER(C.c_size_t)]),
    ("prxref_scene_dynamic_flags", C.c_int, [_P, C.POINTER(C.c_uint8), C.c_size_t]),
    ("prxref_scene_destroy", None, [_P]),
    ("prxref_engine_create", C.c_int, [_P, C.POINTER(L.Config), C.POINTER(_P)]),
    ("prxref_engine_destroy", None, [_P]),
    ("prxref_engine_set_workers", None, [_P, C.c_uint]),
    ("prxref_engine_get_info", C.c_int, [_P, C.POINTER(L.EngineInfo)]),
    ("prxref_run_frame", C.c_int, [_P, C.POINTER(L.FrameStats)]),
    ("prxref_frame_update", C.c_int, [_P, C.POINTER(L.FrameStats)]),
    ("prxref_run_stage", C.c_int, [_P, C.c_int, C.POINTER(L.FrameStats)]),
    ("prxref_field_bytes", C.c_size_t, [_P, C.c_int, C.c_uint32]),
    ("prxref_download", C.c_int, [_P, C.c_int, C.c_uint32, _P, C.c_size_t]),
    ("prxref_upload", C.c_int, [_P, C.c_int, C.c_uint32, _P, C.c_size_t]),
    ("prxref_set_frame_counter", C.c_int, [_P, C.c_int]),
    ("prxref_gather", C.c_int, [_P, C.POINTER(L.Camera), C.c_float, C.c_uint, C.POINTER(C.c_float),
                                C.POINTER(C.c_double)]),
    ("prxref_select_paths_to_prune", C.c_int, [C.POINTER(C.c_uint32), C.c_size_t, C.c_uint32,
                                               C.c_uint32, C.c_uint64, C.c_uint32,
                                               C.POINTER(C.c_uint32), C.POINTER(C.c_size_t)]),
    ("prxref_intersect_batch", C.c_int, [_P, C.c_int, C.POINTER(C.c_float), C.c_size_t,
                                         C.POINTER(C.c_float)]),
    ("prxref_occluded_batch", C.c_int, [_P, C.c_int, C.POINTER(C.c_float), C.c_size_t, C.POINTER(C.c_float)]),
    ("prxref_gen_last_error", C.c_char_p, []),
    ("prxref_synthetic_desc", C.c_int, [C.c_char_p, C.c_uint32, C.c_float, C.POINTER(_P),
                                        C.POINTER(L.SceneDesc)]),
    ("prxref_synthetic_free", None, [_P]),
    ("prxref_scene_load_text", C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(_P)]),
    ("prxref_write_photon_dump", C.c_int, [_P, C.c_char_p]),
    ("prxref_write_image", C.c_int, [C.c_char_p, C.POINTER(C.c_float), C.c_uint32, C.c_uint32]),
    ("prxref_write_stats_csv", C.c_int, [C.c_char_p, C.POINTER(L.FrameStats), C.c_size_t]),
    ("prxref_reuse_report", C.c_int, [C.POINTER(L.FrameStats), C.c_size_t, C.c_char_p, C.c_size_t,
                                      C.POINTER(C.c_size_t)]),
]

_lib = None


def available() -> bool:
    return os.path.exists(REF_LIB)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not available():
            raise ImportError(f"reference oracle not built: {REF_LIB} (make -C oracle ref)")
        h = C.CDLL(REF_LIB)
        for name, res, args in _SIGS:
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(code: int) -> None:
    if code != 0:
        raise L._exception_for(code, lib().prxref_last_error().decode(errors="replace"))


class RefScene:
    def __init__(self, handle):
        self._h = C.c_void_p(handle)

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().prxref_scene_destroy(self._h)
            self._h = None

    @classmethod
    def builtin(cls, name: str) -> "RefScene":
        h = C.c_void_p()
        check(lib().prxref_scene_builtin(name.encode(), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_text(cls, text: str, base_dir: str = "") -> "RefScene":
        """load_scene_text (scene.cpp:272-379) of the reference."""
        h = C.c_void_p()
        check(lib().prxref_scene_load_text(text.encode(), base_dir.encode(), C.byref(h)))
        return cls(h.value)

    @classmethod
    def synthetic(cls, name: str, n_dynamic: int = 0, tri_scale: float = 0.0) -> "RefScene":
        """The BASELINE workload scenes C1-C5 from the generators compiled into the oracle
        library (oracle/scene_gen.cpp) -- same description as pathreuse.Scene.synthetic,
        without loading the product library."""
        holder, desc = C.c_void_p(), L.SceneDesc()
        if lib().prxref_synthetic_desc(name.encode(), int(n_dynamic), float(tri_scale), C.byref(holder),
                                       C.byref(desc)) != 0:
            raise L.SceneError(lib().prxref_gen_last_error().decode(errors="replace"))
        try:
            return cls.from_desc(desc)
        finally:
            lib().prxref_synthetic_free(holder)

    @classmethod
    def from_desc(cls, desc: L.SceneDesc) -> "RefScene":
        h = C.c_void_p()
        check(lib().prxref_scene_create(C.byref(desc), C.byref(h)))
        return cls(h.value)

    def describe(self) -> L.SceneDesc:
        d = L.SceneDesc()
        check(lib().prxref_scene_describe(self._h, C.byref(d)))
        return d

    @property
    def diagonal(self) -> float:
        return float(lib().prxref_scene_diagonal(self._h))

    def bvh_permutation(self) -> np.ndarray:
        n = C.c_size_t()
        check(lib().prxref_scene_bvh_permutation(self._h, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.uint32)
        check(lib().prxref_scene_bvh_permutation(
            self._h, out.ctypes.data_as(C.POINTER(C.c_uint32)), n.value, C.byref(n)))
        return out

    def intersect(self, frame: int, rays: np.ndarray) -> np.ndarray:
        rays = np.ascontiguousarray(rays, dtype=np.float32).reshape(-1, 8)
        hits = np.zeros((rays.shape[0], 9), dtype=np.float32)
        check(lib().prxref_intersect_batch(self._h, int(frame),
                                           rays.ctypes.data_as(C.POINTER(C.c_float)),
                                           rays.shape[0], hits.ctypes.data_as(C.POINTER(C.c_float))))
        return hits

    def occluded(self, frame: int, rays: np.ndarray) -> np.ndarray:
        rays = np.ascontiguousarray(rays, dtype=np.float32).reshape(-1, 8)
        out = np.zeros(rays.shape[0], dtype=np.float32)
        check(lib().prxref_occluded_batch(self._h, int(frame), rays.ctypes.data_as(C.POINTER(C.c_float)),
                                          rays.shape[0], out.ctypes.data_as(C.POINTER(C.c_float))))
        return out


_DT = {
    "photons": PHOTON_DTYPE, "aux": AUX_DTYPE, "pos_obj": np.dtype("<f4"),
    "energy": np.dtype("<f4"), "in_dir": np.dtype("<f4"), "out_dir": np.dtype("<f4"),
    "origin": np.dtype("<f4"), "emission_dir": np.dtype("<f4"), "canonical": np.dtype("<f4"),
    "cell": np.dtype("<u4"), "epoch": np.dtype("<u4"), "path_info": np.dtype("<u4"),
    "meta": np.dtype("u1"), "retrace_start": np.dtype("u1"), "segment_flags": np.dtype("<u4"),
    "dm_target": np.dtype("<u4"), "dm_current": np.dtype("<u4"), "pruned": np.dtype("<u4"),
}
_VEC4 = {"pos_obj", "energy", "in_dir", "out_dir", "origin", "emission_dir", "canonical", "meta"}


class RefEngine:
    """pathreuse::Engine (engine.hpp:69-179), the CPU reference, behind the shim."""

    def __init__(self, scene: RefScene, config: L.Config):
        self.scene = scene
        self.config = config
        h = C.c_void_p()
        check(lib().prxref_engine_create(scene._h, C.byref(config), C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().prxref_engine_destroy(self._h)
            self._h = None

    def write_photon_dump(self, path: str) -> None:
        check(lib().prxref_write_photon_dump(self._h, path.encode()))

    def set_workers(self, n: int) -> None:
        lib().prxref_engine_set_workers(self._h, int(n))

    def run_frame(self) -> L.FrameStats:
        st = L.FrameStats()
        check(lib().prxref_run_frame(self._h, C.byref(st)))
        return st

    def frame_update(self) -> L.FrameStats:
        st = L.FrameStats()
        check(lib().prxref_frame_update(self._h, C.byref(st)))
        return st

    def run_stage(self, stage: str, st: L.FrameStats | None = None) -> L.FrameStats:
        st = st if st is not None else L.FrameStats()
        check(lib().prxref_run_stage(self._h, L.STAGE[stage], C.byref(st)))
        return st

    def info(self) -> L.EngineInfo:
        inf = L.EngineInfo()
        check(lib().prxref_engine_get_info(self._h, C.byref(inf)))
        return inf

    def download(self, field: str, index: int = 0) -> np.ndarray:
        fid = L.FIELD[field]
        n = lib().prxref_field_bytes(self._h, fid, int(index))
        dt = _DT[field]
        out = np.empty(n // dt.itemsize, dtype=dt)
        if n:
            check(lib().prxref_download(self._h, fid, int(index), out.ctypes.data_as(C.c_void_p), n))
        return out.reshape(-1, 4) if field in _VEC4 else out

    def upload(self, field: str, data: np.ndarray, index: int = 0) -> None:
        arr = np.ascontiguousarray(data)
        check(lib().prxref_upload(self._h, L.FIELD[field], int(index),
                                  arr.ctypes.data_as(C.c_void_p), arr.nbytes))

    def set_frame_counter(self, frames_run: int) -> None:
        check(lib().prxref_set_frame_counter(self._h, int(frames_run)))

    def gather(self, camera: L.Camera | None = None, radius: float = 0.25,
               workers: int = 0) -> tuple:
        cam = camera if camera is not None else self.scene.describe().camera
        out = np.zeros((cam.height, cam.width, 3), dtype=np.float32)
        secs = C.c_double()
        check(lib().prxref_gather(self._h, C.byref(cam), float(radius), int(workers),
                                  out.ctypes.data_as(C.POINTER(C.c_float)), C.byref(secs)))
        return out, secs.value


def select_paths_to_prune(paths, dm_c: int, dm_t: int, seed: int, frame: int) -> np.ndarray:
    arr = np.ascontiguousarray(paths, dtype=np.uint32)
    out = np.zeros(max(1, arr.size), dtype=np.uint32)
    n = C.c_size_t()
    check(lib().prxref_select_paths_to_prune(arr.ctypes.data_as(C.POINTER(C.c_uint32)), arr.size,
                                             int(dm_c), int(dm_t), int(seed), int(frame),
                                             out.ctypes.data_as(C.POINTER(C.c_uint32)),
                                             C.byref(n)))
    return out[: n.value]


STATE_FIELDS = ("pos_obj", "energy", "in_dir", "out_dir", "origin", "emission_dir", "canonical",
                "cell", "epoch", "path_info", "meta", "retrace_start")


def copy_state(src, dst, n_lights: int) -> None:
    """Copy the full per-path/per-vertex state + DMs from one engine to another."""
    for f in STATE_FIELDS:
        dst.upload(f, src.download(f))
    for li in range(n_lights):
        dst.upload("dm_target", src.download("dm_target", li), li)
        dst.upload("dm_current", src.download("dm_current", li), li)


# ---- the reference's own writers (offline artefacts) ----
def write_image(image: np.ndarray, path: str) -> None:
    img = np.ascontiguousarray(image, dtype=np.float32)
    check(lib().prxref_write_image(path.encode(), img.ctypes.data_as(C.POINTER(C.c_float)),
                                   img.shape[1], img.shape[0]))


def write_stats_csv(rows, path: str) -> None:
    arr = (L.FrameStats * len(rows))(*rows)
    check(lib().prxref_write_stats_csv(path.encode(), arr, len(rows)))


def reuse_report(rows) -> str:
    arr = (L.FrameStats * len(rows))(*rows)
    n = C.c_size_t(0)
    check(lib().prxref_reuse_report(arr, len(rows), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(lib().prxref_reuse_report(arr, len(rows), buf, len(buf), C.byref(n)))
    return buf.value.decode()
