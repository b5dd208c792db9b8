"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes wrapper of oracle/_build/liboracle.so, the plain-C restatement of the reference hot
path (oracle/pathreuse_oracle.c).  Same method names as oracle/ref.py's RefEngine so the
tests can run either checker.  Used by tests/ and smoke() only.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2111_06906_b200 import _lib as L
from oracle.ref import _DT, _VEC4

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "_build", "liboracle.so")
_P = C.c_void_p
_SIGS = [
    ("po_last_error", C.c_char_p, []),
    ("po_prune_probability", C.c_double, [C.c_uint32, C.c_uint32]),
    ("po_energies_close", C.c_int, [C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_float]),
    ("po_encode_path_info", C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_int,
                                      C.POINTER(C.c_uint32)]),
    ("po_decode_path_info", None, [C.c_uint32, C.POINTER(C.c_uint32)]),
    ("po_memory_footprint", None, [C.c_uint64, C.c_uint32, C.POINTER(C.c_uint32), C.c_uint32, C.c_int,
                                   C.POINTER(C.c_double)]),
    ("po_select_paths_to_prune", C.c_int, [C.POINTER(C.c_uint32), C.c_size_t, C.c_uint32, C.c_uint32,
                                           C.c_uint64, C.c_uint32, C.POINTER(C.c_uint32),
                                           C.POINTER(C.c_size_t)]),
    ("po_scene_create", C.c_int, [C.POINTER(L.SceneDesc), C.POINTER(_P)]),
    ("po_scene_destroy", None, [_P]),
    ("po_scene_diagonal", C.c_float, [_P]),
    ("po_scene_bvh_permutation", C.c_int, [_P, C.POINTER(C.c_uint32), C.c_size_t, C.POINTER(C.c_size_t)]),
    ("po_engine_create", C.c_int, [_P, C.POINTER(L.Config), C.POINTER(_P)]),
    ("po_engine_destroy", None, [_P]),
    ("po_run_frame", C.c_int, [_P, C.POINTER(L.FrameStats)]),
    ("po_frame_update", C.c_int, [_P, C.POINTER(L.FrameStats)]),
    ("po_run_stage", C.c_int, [_P, C.c_int, C.POINTER(L.FrameStats)]),
    ("po_field_bytes", C.c_size_t, [_P, C.c_int, C.c_uint32]),
    ("po_download", C.c_int, [_P, C.c_int, C.c_uint32, _P, C.c_size_t]),
    ("po_upload", C.c_int, [_P, C.c_int, C.c_uint32, _P, C.c_size_t]),
    ("po_set_frame_counter", C.c_int, [_P, C.c_int]),
    ("po_gather", C.c_int, [_P, C.POINTER(L.Camera), C.c_float, C.POINTER(C.c_float)]),
    ("po_intersect_batch", C.c_int, [_P, C.c_int, C.POINTER(C.c_float), C.c_size_t, C.POINTER(C.c_float)]),
]
_lib = None


def available() -> bool:
    return os.path.exists(PORT_LIB)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not available():
            raise ImportError(f"C oracle not built: {PORT_LIB} (make -C oracle port)")
        h = C.CDLL(PORT_LIB)
        for name, res, args in _SIGS:
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(code: int) -> None:
    if code != 0:
        raise L._exception_for(code, lib().po_last_error().decode(errors="replace"))


class PortScene:
    def __init__(self, desc: L.SceneDesc):
        self.desc = desc
        h = C.c_void_p()
        check(lib().po_scene_create(C.byref(desc), C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().po_scene_destroy(self._h)
            self._h = None

    def describe(self) -> L.SceneDesc:
        return self.desc

    @property
    def diagonal(self) -> float:
        return float(lib().po_scene_diagonal(self._h))

    def bvh_permutation(self) -> np.ndarray:
        n = C.c_size_t()
        check(lib().po_scene_bvh_permutation(self._h, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.uint32)
        check(lib().po_scene_bvh_permutation(self._h, out.ctypes.data_as(C.POINTER(C.c_uint32)), n.value,
                                             C.byref(n)))
        return out

    def intersect(self, frame: int, rays: np.ndarray) -> np.ndarray:
        rays = np.ascontiguousarray(rays, dtype=np.float32).reshape(-1, 8)
        hits = np.zeros((rays.shape[0], 9), dtype=np.float32)
        check(lib().po_intersect_batch(self._h, int(frame), rays.ctypes.data_as(C.POINTER(C.c_float)),
                                       rays.shape[0], hits.ctypes.data_as(C.POINTER(C.c_float))))
        return hits


class PortEngine:
    def __init__(self, scene: PortScene, config: L.Config):
        self.scene = scene
        self.config = config
        h = C.c_void_p()
        check(lib().po_engine_create(scene._h, C.byref(config), C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().po_engine_destroy(self._h)
            self._h = None

    def set_workers(self, n: int) -> None:  # single-threaded restatement
        pass

    def run_frame(self) -> L.FrameStats:
        st = L.FrameStats()
        check(lib().po_run_frame(self._h, C.byref(st)))
        return st

    def frame_update(self) -> L.FrameStats:
        st = L.FrameStats()
        check(lib().po_frame_update(self._h, C.byref(st)))
        return st

    def run_stage(self, stage: str, st: L.FrameStats | None = None) -> L.FrameStats:
        st = st if st is not None else L.FrameStats()
        check(lib().po_run_stage(self._h, L.STAGE[stage], C.byref(st)))
        return st

    def download(self, field: str, index: int = 0) -> np.ndarray:
        fid = L.FIELD[field]
        n = lib().po_field_bytes(self._h, fid, int(index))
        dt = _DT[field]
        out = np.empty(n // dt.itemsize, dtype=dt)
        if n:
            check(lib().po_download(self._h, fid, int(index), out.ctypes.data_as(C.c_void_p), n))
        return out.reshape(-1, 4) if field in _VEC4 else out

    def upload(self, field: str, data: np.ndarray, index: int = 0) -> None:
        arr = np.ascontiguousarray(data)
        check(lib().po_upload(self._h, L.FIELD[field], int(index), arr.ctypes.data_as(C.c_void_p), arr.nbytes))

    def set_frame_counter(self, frames_run: int) -> None:
        check(lib().po_set_frame_counter(self._h, int(frames_run)))

    def gather(self, camera: L.Camera | None = None, radius: float = 0.25, workers: int = 0) -> tuple:
        cam = camera if camera is not None else self.scene.describe().camera
        out = np.zeros((cam.height, cam.width, 3), dtype=np.float32)
        check(lib().po_gather(self._h, C.byref(cam), float(radius), out.ctypes.data_as(C.POINTER(C.c_float))))
        return out, 0.0
