"""Drop-in mirror of the reference's Python module ``pathreuse``
(/root/reference/proj/python/pathreuse/__init__.py:3-12, bindings/module.cpp:44-135),
executed by the B200 engine through the C ABI (include/prx.h).

The eight reference functions keep their names, argument names, defaults, return shapes
and error types.  ``Scene`` / ``Engine`` additionally expose the engine the C++ API
(engine.hpp:69-179) offers: the north_star stages ``frame_update`` / ``verify_paths`` /
``retrace_invalid`` / ``splat`` and lazy host mirrors of the device state.
"""
from __future__ import annotations

import ctypes as C
from typing import Iterable, Sequence

import numpy as np

from . import _lib as L

PHOTON_DTYPE = np.dtype([("incoming_dir", "<f4", (3,)), ("object_id", "<u4"),
                         ("energy", "<f4", (3,)), ("radius", "<f4")])   # photon_store.hpp:13-21
AUX_DTYPE = np.dtype([("position", "<f4", (3,)), ("outgoing", "<f4", (3,))])  # :75-78

_BUILTINS = ["static-box", "moving-cube", "parallel-spot", "merry-go-round-analog",
             "armadillo-analog", "villa-analog"]


# --------------------------------------------------------------------------- pure helpers
def prune_probability(dm_current: int, dm_target: int) -> float:
    """Eq. 1 (light.hpp:132-135)."""
    return float(L.lib().prx_prune_probability(int(dm_current), int(dm_target)))


def energies_close(e_old: Sequence[float], e_new: Sequence[float], threshold: float) -> bool:
    """Eq. 2 (engine.hpp:34-41)."""
    a = (C.c_float * 3)(*[float(v) for v in e_old])
    b = (C.c_float * 3)(*[float(v) for v in e_new])
    return bool(L.lib().prx_energies_close(a, b, float(threshold)))


def encode_path_info(cell: int, seg_count: int, retrace_start: int = 0, replace: bool = False,
                     reuse_light: bool = False) -> int:
    """photon_store.cpp:9-20; IndexError on a field overflow (std::out_of_range)."""
    out = C.c_uint32()
    for v in (cell, seg_count, retrace_start):
        if int(v) < 0 or int(v) > 0xFFFFFFFF:
            raise TypeError("path info fields are unsigned 32-bit integers")
    L.check(L.lib().prx_encode_path_info(int(cell), int(seg_count), int(retrace_start),
                                         int(bool(replace)), int(bool(reuse_light)),
                                         C.byref(out)))
    return int(out.value)


def decode_path_info(word: int) -> dict:
    """photon_store.cpp:22-30."""
    cell, seg, start = C.c_uint32(), C.c_uint32(), C.c_uint32()
    rep, reuse = C.c_int(), C.c_int()
    L.lib().prx_decode_path_info(int(word) & 0xFFFFFFFF, C.byref(cell), C.byref(seg),
                                 C.byref(start), C.byref(rep), C.byref(reuse))
    return {"cell": cell.value, "seg_count": seg.value, "retrace_start": start.value,
            "replace": bool(rep.value), "reuse_light": bool(reuse.value)}


def memory_footprint(n_paths: int, max_bounces: int, dm_dims: Sequence[int],
                     area_light: bool) -> dict:
    """Table 1 of the paper (photon_store.cpp:38-54), MiB."""
    dims = (C.c_uint32 * max(1, len(dm_dims)))(*[int(d) for d in dm_dims])
    out = (C.c_double * 7)()
    L.lib().prx_memory_footprint(int(n_paths), int(max_bounces), dims, len(dm_dims),
                                 int(bool(area_light)), out)
    keys = ("path_info", "origin_positions", "distribution_maps", "pruned_array",
            "photon_map", "subtotal_reuse", "total")
    return {k: float(v) for k, v in zip(keys, out)}


def builtin_scenes() -> list:
    """module.cpp:57-61."""
    return list(_BUILTINS)


# --------------------------------------------------------------------------- scenes
class Scene:
    """A finalized scene (finalize_scene, scene.cpp:63-113) owned by the C ABI."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and L is not None:  # (module globals may be gone at exit)
            L.lib().prx_scene_destroy(h)
            self._h = None

    @classmethod
    def builtin(cls, name: str) -> "Scene":
        h = C.c_void_p()
        L.check(L.lib().prx_scene_builtin(name.encode(), C.byref(h)))
        return cls(h.value)

    @classmethod
    def synthetic(cls, name: str, n_dynamic: int = 0, tri_scale: float = 0.0) -> "Scene":
        """Procedural BASELINE configurations "C1".."C5"."""
        h = C.c_void_p()
        L.check(L.lib().prx_scene_synthetic(name.encode(), int(n_dynamic), float(tri_scale),
                                            C.byref(h)))
        return cls(h.value)

    @classmethod
    def load(cls, source: str) -> "Scene":
        """load_scene_source (scene.cpp:392-398): "builtin:NAME", a builtin name, or a JSON
        scene file whose OBJ meshes are resolved relative to the file."""
        h = C.c_void_p()
        L.check(L.lib().prx_scene_load(str(source).encode(), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_text(cls, json_text: str, base_dir: str = "") -> "Scene":
        """load_scene_text (scene.cpp:272-379)."""
        h = C.c_void_p()
        L.check(L.lib().prx_scene_load_text(json_text.encode(), str(base_dir).encode(), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_desc(cls, desc: L.SceneDesc) -> "Scene":
        h = C.c_void_p()
        L.check(L.lib().prx_scene_create(C.byref(desc), C.byref(h)))
        return cls(h.value)

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def describe(self) -> L.SceneDesc:
        """Borrowed C description (valid while this Scene lives)."""
        d = L.SceneDesc()
        L.check(L.lib().prx_scene_describe(self._h, C.byref(d)))
        return d

    def counts(self) -> dict:
        c = (C.c_uint64 * 4)()
        L.check(L.lib().prx_scene_counts(self._h, c))
        return {"static_triangles": c[0], "dynamic_triangles": c[1], "bvh_nodes": c[2],
                "objects": c[3]}

    def bvh_permutation(self) -> np.ndarray:
        n = C.c_size_t()
        L.check(L.lib().prx_scene_bvh_permutation(self._h, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.uint32)
        L.check(L.lib().prx_scene_bvh_permutation(
            self._h, out.ctypes.data_as(C.POINTER(C.c_uint32)), n.value, C.byref(n)))
        return out

    @property
    def diagonal(self) -> float:
        return float(L.lib().prx_scene_diagonal(self._h))


def make_config(mode: str = "naive", paths: int = 10000, bounces: int = 7,
                dm: Sequence[int] = (8, 8, 64, 64), threshold: float = 0.001, seed: int = 1,
                radius: float = 0.25, workers: int = 1, record_flags: bool = False,
                device: int = 0, shard: tuple = (0, 0), exact_trig: bool = True,
                dfs_traversal: bool = False) -> L.Config:
    """EngineConfig (engine.hpp:43-53) + make_config (module.cpp:15-27)."""
    if mode not in L.MODES:
        raise ValueError("unknown engine mode: " + str(mode))
    dm = list(dm)
    if len(dm) != 4:
        raise ValueError("engine: dm_dims needs 4 axis counts")
    cfg = L.Config()
    cfg.mode = L.MODES[mode]
    cfg.n_paths = int(paths)
    cfg.max_bounces = int(bounces)
    for i, v in enumerate(dm):
        cfg.dm_dims[i] = int(v)
    cfg.threshold = float(threshold)
    cfg.seed = int(seed)
    cfg.gather_radius = float(radius)
    cfg.workers = int(workers)
    cfg.record_flags = int(bool(record_flags))
    cfg.device = int(device)
    cfg.shard_begin, cfg.shard_end = int(shard[0]), int(shard[1])
    cfg.exact_trig = 0 if exact_trig else -1
    cfg.dfs_traversal = int(bool(dfs_traversal))
    return cfg


_FIELD_DTYPES = {
    "photons": PHOTON_DTYPE, "aux": AUX_DTYPE,
    "pos_obj": np.dtype("<f4"), "energy": np.dtype("<f4"), "in_dir": np.dtype("<f4"),
    "out_dir": np.dtype("<f4"), "origin": np.dtype("<f4"), "emission_dir": np.dtype("<f4"),
    "canonical": np.dtype("<f4"), "cell": np.dtype("<u4"), "epoch": np.dtype("<u4"),
    "path_info": np.dtype("<u4"), "meta": np.dtype("u1"), "retrace_start": np.dtype("u1"),
    "segment_flags": np.dtype("<u4"), "dm_target": np.dtype("<u4"),
    "dm_current": np.dtype("<u4"), "pruned": np.dtype("<u4"),
}
_VEC4 = {"pos_obj", "energy", "in_dir", "out_dir", "origin", "emission_dir", "canonical", "meta"}


class Engine:
    """pathreuse::Engine (engine.hpp:69-179) on one B200 (optionally one path shard)."""

    _overlap = False  # set_splat_overlap

    def __init__(self, scene: Scene, config: L.Config | None = None, **kwargs):
        self.scene = scene  # keeps the scene alive
        self.config = config if config is not None else make_config(**kwargs)
        h = C.c_void_p()
        L.check(L.lib().prx_engine_create(scene.handle, C.byref(self.config), C.byref(h)))
        self._h = h

    @classmethod
    def _borrowed(cls, handle: int, scene: Scene, config: L.Config, owner) -> "Engine":
        """A view of an engine owned by someone else (a prx_group shard): never destroyed here."""
        e = cls.__new__(cls)
        e.scene, e.config, e._h, e._owner = scene, config, C.c_void_p(handle), owner
        return e

    def close(self):
        h = getattr(self, "_h", None)
        if getattr(self, "_owner", None) is None and h is not None and h.value and L is not None:
            L.lib().prx_engine_destroy(h)  # (module globals may be gone at exit)
        self._h = None

    def __del__(self):
        self.close()

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    # -- frame stages
    def run_frame(self) -> L.FrameStats:
        st = L.FrameStats()
        L.check(L.lib().prx_run_frame(self._h, C.byref(st)))
        return st

    def frame_update(self, st: L.FrameStats | None = None) -> L.FrameStats:
        st = st if st is not None else L.FrameStats()
        L.check(L.lib().prx_frame_update(self._h, C.byref(st)))
        return st

    def verify_paths(self, st: L.FrameStats) -> L.FrameStats:
        L.check(L.lib().prx_verify_paths(self._h, C.byref(st)))
        return st

    def retrace_invalid(self, st: L.FrameStats) -> L.FrameStats:
        L.check(L.lib().prx_retrace_invalid(self._h, C.byref(st)))
        return st

    def run_stage(self, stage: str) -> L.FrameStats:
        st = L.FrameStats()
        L.check(L.lib().prx_run_stage(self._h, L.STAGE[stage], C.byref(st)))
        return st

    def splat(self, camera: L.Camera | None = None, radius: float | None = None, mode: int = 1,
              st: L.FrameStats | None = None) -> np.ndarray:
        """gather_image (gather.cpp:35-75) as a GPU splat -> float32 [h, w, 3]."""
        info = self.info()
        cam = camera if camera is not None else self.scene.describe().camera
        w, h = int(cam.width), int(cam.height)
        out = np.zeros((h, w, 3), dtype=np.float32)
        r = self.config.gather_radius if radius is None else radius
        L.check(L.lib().prx_splat(self._h, C.byref(cam), float(r), int(mode),
                                  out.ctypes.data_as(C.c_void_p), None,
                                  C.byref(st) if st is not None else None))
        if self._overlap:  # (an overlapped splat fills `out` at the next engine call)
            self.synchronize()
        del info
        return out

    # -- introspection
    def info(self) -> L.EngineInfo:
        inf = L.EngineInfo()
        L.check(L.lib().prx_engine_get_info(self._h, C.byref(inf)))
        return inf

    def launch_count(self) -> int:
        return int(L.lib().prx_engine_launch_count(self._h))

    def transfer_bytes(self) -> tuple:
        """(host->device, device->host) bytes this engine has copied since creation."""
        h2d, d2h = C.c_uint64(0), C.c_uint64(0)
        L.check(L.lib().prx_engine_transfer_bytes(self._h, C.byref(h2d), C.byref(d2h)))
        return int(h2d.value), int(d2h.value)

    def download(self, field: str, index: int = 0) -> np.ndarray:
        fid = L.FIELD[field]
        nbytes = L.lib().prx_field_bytes(self._h, fid, int(index))
        dt = _FIELD_DTYPES[field]
        out = np.empty(nbytes // dt.itemsize, dtype=dt)
        if nbytes:
            L.check(L.lib().prx_engine_download(self._h, fid, int(index),
                                                out.ctypes.data_as(C.c_void_p), nbytes))
        if field in _VEC4:
            out = out.reshape(-1, 4)
        return out

    def upload(self, field: str, data: np.ndarray, index: int = 0) -> None:
        fid = L.FIELD[field]
        arr = np.ascontiguousarray(data)
        L.check(L.lib().prx_engine_upload(self._h, fid, int(index),
                                          arr.ctypes.data_as(C.c_void_p), arr.nbytes))

    def set_frame_counter(self, frames_run: int) -> None:
        L.check(L.lib().prx_engine_set_frame_counter(self._h, int(frames_run)))

    def set_stream(self, cuda_stream: int | None) -> None:
        L.check(L.lib().prx_engine_set_stream(self._h, C.c_void_p(cuda_stream or 0)))

    def synchronize(self) -> None:
        L.check(L.lib().prx_engine_synchronize(self._h))

    def set_splat_overlap(self, on: bool) -> None:
        """Device-output splats of the scene camera run on a side stream, overlapping the next
        frame's scene update and occlusion flags (prx_engine_set_splat_overlap)."""
        L.check(L.lib().prx_engine_set_splat_overlap(self._h, 1 if on else 0))
        self._overlap = bool(on)

    def splat_into(self, out: np.ndarray, camera: L.Camera | None = None, radius: float | None = None,
                   mode: int = 1) -> np.ndarray:
        """splat into a host float32 [h, w, 3] array.  With the overlap on (scene camera at the
        prefix radius), the call returns at once and `out` is filled when the next engine call
        (run_frame, synchronize, ...) returns."""
        cam = camera if camera is not None else self.scene.describe().camera
        if out.dtype != np.float32 or not out.flags.c_contiguous or out.size != 3 * cam.width * cam.height:
            raise ValueError("splat_into: out must be a C-contiguous float32 [h, w, 3] array of the camera's size")
        r = self.config.gather_radius if radius is None else radius
        L.check(L.lib().prx_splat(self._h, C.byref(cam), float(r), int(mode), out.ctypes.data_as(C.c_void_p), None,
                                  None))
        return out

    def splat_device(self, rgb_dev_ptr: int, camera: L.Camera | None = None, radius: float | None = None,
                     mode: int = 1) -> None:
        """splat into a device float[3*w*h] buffer (asynchronous when the overlap is on)."""
        cam = camera if camera is not None else self.scene.describe().camera
        r = self.config.gather_radius if radius is None else radius
        L.check(L.lib().prx_splat(self._h, C.byref(cam), float(r), int(mode), None, C.c_void_p(int(rgb_dev_ptr)),
                                  None))

    def photon_map(self) -> np.ndarray:
        return self.download("photons")

    def intersect(self, rays: np.ndarray, any_hit: bool = False) -> np.ndarray:
        """intersect_scene / occluded (scene.cpp:136-177) at the current frame for rays
        [n, 8] = {origin, dir, t_min, t_max}: [n, 9] hits (see prx_intersect_batch) or [n]."""
        r = np.ascontiguousarray(rays, dtype=np.float32).reshape(-1, 8)
        out = np.zeros((r.shape[0],) if any_hit else (r.shape[0], 9), dtype=np.float32)
        L.check(L.lib().prx_intersect_batch(self._h, r.ctypes.data_as(C.POINTER(C.c_float)), r.shape[0],
                                            int(bool(any_hit)), out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def write_photon_dump(self, path: str) -> None:
        """write_photon_dump(engine.photon_map(), path) (photon_store.cpp:76-86)."""
        L.check(L.lib().prx_engine_write_photon_dump(self._h, str(path).encode()))

    def vertex_aux(self) -> np.ndarray:
        return self.download("aux")


def _stats_dict(st: L.FrameStats) -> dict:
    """stats_dict (module.cpp:29-40)."""
    return {"frame": st.frame, "mode": L.MODE_NAMES[st.mode], "rays_traced": st.rays_traced,
            "rays_reused": st.rays_reused, "paths_replaced": st.paths_replaced,
            "paths_pruned": st.paths_pruned, "paths_filled": st.paths_filled,
            "visibility_rays": st.visibility_rays}


def run_builtin(scene: str, mode: str = "naive", paths: int = 10000, bounces: int = 7,
                frames: int = 1, seed: int = 1, dm: Iterable[int] = (8, 8, 64, 64),
                threshold: float = 0.001, radius: float = 0.25, workers: int = 1) -> list:
    """module.cpp:100-115."""
    cfg = make_config(mode, paths, bounces, list(dm), threshold, seed, radius, workers)
    eng = Engine(Scene.builtin(scene), cfg)
    out = [_stats_dict(eng.run_frame()) for _ in range(int(frames))]
    eng.close()
    return out


def render_builtin(scene: str, mode: str = "naive", paths: int = 10000, bounces: int = 7,
                   frames: int = 1, seed: int = 1, dm: Iterable[int] = (8, 8, 64, 64),
                   threshold: float = 0.001, radius: float = 0.25, workers: int = 1) -> tuple:
    """module.cpp:117-134: (width, height, bytes of float32 RGB rows)."""
    cfg = make_config(mode, paths, bounces, list(dm), threshold, seed, radius, workers)
    sc = Scene.builtin(scene)
    eng = Engine(sc, cfg)
    for _ in range(int(frames)):
        eng.run_frame()
    img = eng.splat(radius=radius)
    eng.close()
    return int(img.shape[1]), int(img.shape[0]), img.astype("<f4").tobytes()


# --------------------------------------------------------------------------- offline artefacts
def write_photon_dump(photons: np.ndarray, n_paths: int, max_bounces: int, path: str) -> None:
    """PHM1 photon dump (photon_store.cpp:76-86) of a [max_bounces * n_paths] Photon array."""
    rec = np.ascontiguousarray(photons, dtype=PHOTON_DTYPE)
    L.check(L.lib().prx_photon_dump_write(str(path).encode(), int(n_paths), int(max_bounces),
                                          rec.ctypes.data_as(C.c_void_p), rec.nbytes))


def read_photon_dump(path: str) -> tuple:
    """read_photon_dump (photon_store.cpp:88-102) -> (n_paths, max_bounces, photons)."""
    n, b = C.c_uint32(0), C.c_uint32(0)
    L.check(L.lib().prx_photon_dump_read(str(path).encode(), C.byref(n), C.byref(b), None, 0))
    rec = np.zeros(n.value * b.value, dtype=PHOTON_DTYPE)
    L.check(L.lib().prx_photon_dump_read(str(path).encode(), C.byref(n), C.byref(b),
                                         rec.ctypes.data_as(C.c_void_p), rec.nbytes))
    return int(n.value), int(b.value), rec


def write_image(image: np.ndarray, path: str) -> None:
    """write_image (gather.cpp:77-92): [H, W, 3] float32 -> binary PPM, gamma 1/2.2."""
    img = np.ascontiguousarray(image, dtype=np.float32)
    if img.ndim != 3 or img.shape[2] != 3:
        raise ValueError("image must be [height, width, 3]")
    L.check(L.lib().prx_image_write_ppm(str(path).encode(), img.ctypes.data_as(C.POINTER(C.c_float)),
                                        int(img.shape[1]), int(img.shape[0])))


def frame_image_name(frame: int) -> str:
    """frame_image_name (gather.cpp:94-98)."""
    buf = C.create_string_buffer(64)
    L.lib().prx_frame_image_name(int(frame), buf, len(buf))
    return buf.value.decode()


def _stats_array(rows) -> C.Array:
    arr = (L.FrameStats * len(rows))()
    for i, r in enumerate(rows):
        if isinstance(r, L.FrameStats):
            C.memmove(C.byref(arr[i]), C.byref(r), C.sizeof(L.FrameStats))
            continue
        arr[i].frame = int(r["frame"])
        arr[i].mode = L.MODES[r["mode"]] if isinstance(r["mode"], str) else int(r["mode"])
        for k in L.FrameStats.COUNTS:
            setattr(arr[i], k, int(r.get(k, 0)))
        for k in ("t_update", "t_occlusion", "t_dm", "t_prune", "t_fill", "t_trace", "t_gather"):
            setattr(arr[i], k, float(r.get(k, 0.0)))
    return arr


def write_stats_csv(rows, path: str) -> None:
    """write_stats_csv (stats.cpp:14-33); rows are FrameStats or run_builtin-style dicts."""
    arr = _stats_array(list(rows))
    L.check(L.lib().prx_stats_csv_write(str(path).encode(), arr, len(arr)))


def read_stats_csv(path: str) -> list:
    """read_stats_csv (stats.cpp:35-70) -> list of FrameStats."""
    n = C.c_size_t(0)
    L.check(L.lib().prx_stats_csv_read(str(path).encode(), None, 0, C.byref(n)))
    arr = (L.FrameStats * n.value)()
    L.check(L.lib().prx_stats_csv_read(str(path).encode(), arr, n.value, C.byref(n)))
    return list(arr)


def reuse_report(rows) -> str:
    """reuse_report (stats.cpp:72-107)."""
    arr = _stats_array(list(rows))
    n = C.c_size_t(0)
    L.check(L.lib().prx_reuse_report(arr, len(arr), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    L.check(L.lib().prx_reuse_report(arr, len(arr), buf, len(buf), C.byref(n)))
    return buf.value.decode()
