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


_SHARD_SIGS = [
    ("po_prune_count", C.c_int, [_P, C.POINTER(C.POINTER(C.c_uint32))]),
    ("po_prune_apply", C.c_int, [_P, C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.POINTER(C.c_uint32)),
                                 C.POINTER(L.FrameStats)]),
    ("po_fill_count", C.c_int, [_P, C.POINTER(C.c_uint32)]),
    ("po_fill_apply", C.c_int, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(L.FrameStats)]),
]


def _shard_lib():
    h = lib()
    for name, res, args in _SHARD_SIGS:
        fn = getattr(h, name)
        fn.restype = res
        fn.argtypes = args
    return h


class PortShardExecutor:
    """One path shard of the C oracle behind the executor interface of
    paper_2111_06906_b200.distributed (CPU torch tensors, for gloo tests)."""

    def __init__(self, scene: PortScene, config: L.Config):
        import torch

        self.torch = torch
        self.engine = PortEngine(scene, config)
        self.sb, self.se = config.shard_begin, config.shard_end
        self.mode = config.mode
        self.n_lights = scene.describe().n_lights
        self.cells = [self.engine.download("dm_target", li).size for li in range(self.n_lights)]
        self.st = L.FrameStats()
        self.lib = _shard_lib()

    def _meta(self):
        return self.engine.download("meta")[self.sb:self.se]

    def frame_update(self):
        m = self._meta()
        live = m[:, 2] == 1
        self.live_segments = int((m[live, 0].astype(np.int64) + m[live, 1]).sum())
        self.st = self.engine.frame_update()

    def verify(self):
        for s in ("update_origins", "occlusions", "compute_dm"):
            self.engine.run_stage(s, self.st)

    def dm_buffers(self):
        return [self.torch.from_numpy(self.engine.download("dm_current", li).view(np.int32).copy())
                for li in range(self.n_lights)]

    def dm_commit(self, bufs):
        for li, t in enumerate(bufs):
            self.engine.upload("dm_current", t.numpy().view(np.uint32), li)

    def prune_count(self):
        outs = [np.zeros(c, dtype=np.uint32) for c in self.cells]
        arr = (C.POINTER(C.c_uint32) * self.n_lights)(*[o.ctypes.data_as(C.POINTER(C.c_uint32)) for o in outs])
        check(self.lib.po_prune_count(self.engine._h, arr))
        return [self.torch.from_numpy(o.view(np.int32)) for o in outs]

    def prune_apply(self, prefix, total):
        pn = [np.ascontiguousarray(p.numpy()).view(np.uint32) for p in prefix]
        tn = [np.ascontiguousarray(t.numpy()).view(np.uint32) for t in total]
        pa = (C.POINTER(C.c_uint32) * self.n_lights)(*[a.ctypes.data_as(C.POINTER(C.c_uint32)) for a in pn])
        ta = (C.POINTER(C.c_uint32) * self.n_lights)(*[a.ctypes.data_as(C.POINTER(C.c_uint32)) for a in tn])
        check(self.lib.po_prune_apply(self.engine._h, pa, ta, C.byref(self.st)))

    def fill_count(self):
        out = (C.c_uint32 * self.n_lights)()
        check(self.lib.po_fill_count(self.engine._h, out))
        return list(out)

    def fill_apply(self, prefix, total):
        pa = (C.c_uint64 * self.n_lights)(*prefix)
        ta = (C.c_uint64 * self.n_lights)(*total)
        check(self.lib.po_fill_apply(self.engine._h, pa, ta, C.byref(self.st)))

    def trace(self):
        m = self._meta()
        rs = self.engine.download("retrace_start")[self.sb:self.se]
        retraced = int(((m[:, 2] == 1) & (rs != 0xFF)).sum())
        self.engine.run_stage("trace", self.st)
        st = self.st
        return {"rays_traced": st.rays_traced, "paths_replaced": st.paths_replaced,
                "paths_pruned": st.paths_pruned, "paths_filled": st.paths_filled,
                "visibility_rays": st.visibility_rays, "live_segments_before": self.live_segments,
                "paths_retraced": retraced, "segments": st.rays_traced + st.rays_reused}

    def new_tensor(self, values, dtype="int64"):
        return self.torch.tensor(values, dtype=getattr(self.torch, dtype))
