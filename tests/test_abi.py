"""The C-ABI library (paper_2111_06906_b200/_prx.so) on the CPU: it loads, exports every
symbol include/prx.h declares, its host-side functions reproduce the reference's
known answers, scenes/BVHs equal the reference's, and errors map to the reference's
exception types.  No kernel runs here (no GPU in this container)."""
import json
import os
import re

import numpy as np
import pytest

from paper_2111_06906_b200 import _lib as L
from paper_2111_06906_b200 import pathreuse as pr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_runs.json")))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "prx.h")).read()
    return sorted(set(re.findall(r"\b(prx_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    names = declared_symbols()
    assert len(names) >= 30
    for name in names:
        assert hasattr(lib, name), name
    assert {n for n, _, _ in L.SIGNATURES} == set(names)
    assert lib.prx_abi_version() == 1


def test_pure_functions_kat():
    assert pr.encode_path_info(cell=5, seg_count=7, retrace_start=0, replace=False, reuse_light=True) == 0x81800005
    d = pr.decode_path_info(0x81800005)
    assert d == {"cell": 5, "seg_count": 7, "retrace_start": 0, "replace": False, "reuse_light": True}
    for c, t, want in GOLD["kat"]["prune_probability"]:
        assert pr.prune_probability(c, t) == want
    for a, b, th, want in GOLD["kat"]["energies_close"]:
        assert pr.energies_close(a, b, th) == want
    fp = pr.memory_footprint(5_000_000, 7, [32, 32, 32, 32], True)
    for k, v in GOLD["kat"]["table1_mib"].items():
        assert abs(fp[k] - v) <= 0.005 * v
    assert pr.memory_footprint(5_000_000, 7, [32, 32, 32, 32], False)["origin_positions"] == 0.0


def test_path_info_round_trip_exhaustive_sample():
    rng = np.random.default_rng(17)  # acceptance.cpp:436-457 (criterion 12), sampled
    for cell in rng.integers(0, 1 << 22, 64):
        for seg in range(1, 17):
            for start in (0, 7, 15):
                for flags in range(4):
                    w = pr.encode_path_info(int(cell), seg, start, bool(flags & 1), bool(flags & 2))
                    assert pr.decode_path_info(w) == {"cell": int(cell), "seg_count": seg, "retrace_start": start,
                                                      "replace": bool(flags & 1), "reuse_light": bool(flags & 2)}


def test_error_mapping():
    with pytest.raises(IndexError):
        pr.encode_path_info(1 << 22, 1)
    with pytest.raises(IndexError):
        pr.encode_path_info(0, 17)
    with pytest.raises(IndexError):
        pr.encode_path_info(0, 1, 16)
    with pytest.raises(L.SceneError):
        pr.Scene.builtin("no-such-scene")
    with pytest.raises(ValueError):
        pr.make_config(mode="nope")
    with pytest.raises(ValueError):
        pr.make_config(dm=[8, 8])
    assert pr.builtin_scenes() == ["static-box", "moving-cube", "parallel-spot", "merry-go-round-analog",
                                   "armadillo-analog", "villa-analog"]


def test_scene_validation_errors():
    # finalize_scene errors (scene.cpp:63-113) through the C ABI
    tri = L.Triangle(L.Vec3(0, 0, 0), L.Vec3(1, 0, 0), L.Vec3(0, 1, 0))
    degenerate = L.Triangle(L.Vec3(0, 0, 0), L.Vec3(1, 0, 0), L.Vec3(2, 0, 0))
    mesh = (L.Triangle * 1)(tri)
    bad_mesh = (L.Triangle * 1)(degenerate)
    kf = (L.Keyframe * 1)(L.Keyframe(0, L.Quat(0, 0, 0, 1), L.Vec3(0, 2, 0), 1.0))
    light = (L.LightDesc * 1)(L.LightDesc(0, L.Vec3(1, 1, 1), 60.0, 1.0, 1.0, 1.0, kf, 1))
    cam = L.Camera(L.Vec3(0, 1, 4), L.Vec3(0, 1, 0), 60.0, 32, 24)

    def scene(m, albedo=(0.5, 0.5, 0.5), lights=light, n_lights=1):
        obj = (L.ObjectDesc * 1)(L.ObjectDesc(b"floor", m, 1, L.Material(0, L.Vec3(*albedo), 1.0), None, 0))
        return L.SceneDesc(obj, 1, lights, n_lights, cam, 4)

    pr.Scene.from_desc(scene(mesh))
    with pytest.raises(L.SceneError):
        pr.Scene.from_desc(scene(bad_mesh))
    with pytest.raises(L.SceneError):
        pr.Scene.from_desc(scene(mesh, albedo=(1.5, 0.5, 0.5)))
    with pytest.raises(L.SceneError):
        pr.Scene.from_desc(scene(mesh, n_lights=0))
    spot = (L.LightDesc * 1)(L.LightDesc(1, L.Vec3(1, 1, 1), 190.0, 1.0, 1.0, 1.0, kf, 1))
    with pytest.raises(ValueError):  # validate_light -> std::invalid_argument
        pr.Scene.from_desc(scene(mesh, lights=spot))


@pytest.mark.parametrize("name", ["static-box", "moving-cube", "villa-analog"])
def test_builtin_scene_bvh_matches_reference(name):
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built")
    a, b = pr.Scene.builtin(name), ref.RefScene.builtin(name)
    assert np.array_equal(a.bvh_permutation(), b.bvh_permutation())
    assert a.diagonal == b.diagonal


def test_synthetic_scene_sizes():
    c = pr.Scene.synthetic("C1").counts()
    assert c["dynamic_triangles"] == 992 and 900 <= c["static_triangles"] <= 1100
    c3 = pr.Scene.synthetic("C3").counts()
    assert c3["dynamic_triangles"] == 4 * 20000 and 250_000 <= c3["static_triangles"] <= 320_000


def test_engine_fails_loudly_without_gpu():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises((L.CudaError, L.PrxError)):
        pr.Engine(pr.Scene.builtin("static-box"), pr.make_config(paths=100))


def test_select_paths_to_prune_matches_reference():
    """select_paths_to_prune (engine.cpp:443-471) behind the C ABI == the reference's."""
    import ctypes as C

    import numpy as np

    from oracle import ref

    if not ref.available():
        import pytest

        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(3)
    for n, dm_c, dm_t, seed, frame in ((1000, 1000, 600, 5, 3), (600, 600, 600, 5, 3), (37, 80, 12, 9, 0),
                                       (500, 300, 0, 1, 7), (0, 0, 5, 1, 1), (2000, 5000, 4999, 11, 2)):
        paths = rng.permutation(np.arange(100, 100 + 3 * n, 3, dtype=np.uint32))[:n]
        out = np.zeros(max(n, 1), dtype=np.uint32)
        k = C.c_size_t()
        L.check(L.lib().prx_select_paths_to_prune(paths.ctypes.data_as(C.POINTER(C.c_uint32)), n, dm_c, dm_t,
                                                   seed, frame, out.ctypes.data_as(C.POINTER(C.c_uint32)),
                                                   C.byref(k)))
        assert np.array_equal(out[: k.value], ref.select_paths_to_prune(paths, dm_c, dm_t, seed, frame))
