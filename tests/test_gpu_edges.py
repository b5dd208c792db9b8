"""Edge cases of the engine configuration and scenes, bit-exact against the reference
(the cases test_engine.cpp / acceptance.cpp exercise around the hot path): fewer paths than
lights, one and sixteen bounces, a single DM cell, the 2^22-cell limit, thresholds 0 and
huge, several light kinds in one scene."""
import pytest

from paper_2111_06906_b200 import pathreuse as pr
from tests.helpers import compare_state, counts
from tests.test_io import DOC, OBJ_TEXT

CASES = [
    # (scene, mode, paths, bounces, dm, threshold)
    ("doc", "naive", 4, 3, [2, 2, 4, 4], 0.001),        # one path per light (4 lights)
    ("doc", "error", 7, 6, [2, 2, 4, 4], 0.01),         # uneven light blocks
    ("doc", "error", 1000, 1, [2, 2, 8, 8], 0.01),      # one bounce
    ("moving-cube", "error", 2000, 16, [2, 2, 8, 8], 0.001),  # sixteen bounces
    ("moving-cube", "naive", 3000, 5, [1, 1, 1, 1], 0.001),   # a single DM cell
    ("doc", "naive", 6000, 4, [32, 32, 64, 64], 0.001),       # 2^22 cells for the area lights
    ("doc", "error", 3000, 5, [2, 2, 8, 8], 0.0),       # threshold 0: any energy change retraces
    ("moving-cube", "error", 3000, 5, [2, 2, 8, 8], 1e9),  # threshold huge: positions only
    ("doc", "baseline", 2000, 5, [2, 2, 8, 8], 0.001),
]


@pytest.mark.gpu
@pytest.mark.parametrize("scene,mode,paths,bounces,dm,threshold", CASES)
def test_edge_configs_bit_exact(tmp_path, scene, mode, paths, bounces, dm, threshold):
    from oracle import ref

    if scene == "doc":
        (tmp_path / "part.obj").write_text(OBJ_TEXT)
        gscene = pr.Scene.from_text(DOC, str(tmp_path))
        rscene = ref.RefScene.from_text(DOC, str(tmp_path))
    else:
        gscene = pr.Scene.builtin(scene)
        rscene = ref.RefScene.builtin(scene)
    cfg = dict(mode=mode, paths=paths, bounces=bounces, dm=dm, threshold=threshold, seed=13)
    gpu = pr.Engine(gscene, pr.make_config(**cfg))
    cpu = ref.RefEngine(rscene, pr.make_config(**cfg))
    cpu.set_workers(0)
    n_lights = gpu.info().n_lights
    for f in range(3):
        sg, sc = gpu.run_frame(), cpu.run_frame()
        assert counts(sg) == counts(sc), f"frame {f}: gpu {counts(sg)} ref {counts(sc)}"
        bad = compare_state(gpu, cpu, n_lights)
        assert all(v == 0 for v in bad.values()), f"frame {f}: mismatches {bad}"


@pytest.mark.gpu
def test_fewer_paths_than_lights_rejected(tmp_path):
    from oracle import ref

    (tmp_path / "part.obj").write_text(OBJ_TEXT)
    with pytest.raises(ValueError):  # engine.cpp:84
        pr.Engine(pr.Scene.from_text(DOC, str(tmp_path)), pr.make_config(paths=3))
    with pytest.raises(ValueError):
        ref.RefEngine(ref.RefScene.from_text(DOC, str(tmp_path)), pr.make_config(paths=3))


@pytest.mark.gpu
@pytest.mark.parametrize("bounces", [0, 17])
def test_bounce_limits_rejected(bounces):
    from oracle import ref

    with pytest.raises(ValueError):
        pr.Engine(pr.Scene.builtin("static-box"), pr.make_config(paths=100, bounces=bounces))
    with pytest.raises(ValueError):
        ref.RefEngine(ref.RefScene.builtin("static-box"), pr.make_config(paths=100, bounces=bounces))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["naive", "error", "baseline"])
def test_odd_sizes_bit_exact(mode):
    """Odd path and vertex counts through every stage and the image."""
    from oracle import ref

    cfg = dict(mode=mode, paths=7777, bounces=5, dm=[3, 5, 7, 9], threshold=0.001, seed=29)
    gpu = pr.Engine(pr.Scene.builtin("merry-go-round-analog"), pr.make_config(**cfg))
    cpu = ref.RefEngine(ref.RefScene.builtin("merry-go-round-analog"), pr.make_config(**cfg))
    cpu.set_workers(0)
    for f in range(3):
        sg, sc = gpu.run_frame(), cpu.run_frame()
        assert counts(sg) == counts(sc), f
        bad = compare_state(gpu, cpu, gpu.info().n_lights)
        assert all(v == 0 for v in bad.values()), (f, bad)
    assert gpu.splat(radius=0.25).tobytes() == cpu.gather(radius=0.25)[0].tobytes()


ROOM = {"name": "room", "material": {"kind": "diffuse", "albedo": [0.7, 0.7, 0.7]},
        "mesh": {"vertices": [[-3, 0, -3], [3, 0, -3], [3, 0, 3], [-3, 0, 3], [-3, 3, -3], [3, 3, -3]],
                 "faces": [[0, 1, 2], [0, 2, 3], [0, 4, 5], [0, 5, 1]]}}
TRI_MOVER = {"name": "tri", "material": {"kind": "glossy", "albedo": [0.9, 0.8, 0.7], "glossy_exponent": 9},
             "mesh": {"vertices": [[-0.5, 0, 0], [0.5, 0, 0], [0, 0.8, 0]], "faces": [[0, 1, 2]]},
             "keyframes": [{"frame": 0, "translation": [0, 0.5, 0]},
                           {"frame": 10, "translation": [0.5, 1.0, -0.5], "rotation": [0, 0.3826834, 0, 0.9238795]}]}
CAM = {"position": [0, 1.5, 4], "look_at": [0, 1, 0], "fov": 60, "resolution": [40, 30]}


def _doc(objects, lights):
    import json

    return json.dumps({"camera": CAM, "objects": objects, "lights": lights, "frames": 20})


@pytest.mark.gpu
@pytest.mark.parametrize("name,doc", [
    ("dynamic-only", _doc([TRI_MOVER], [{"kind": "point", "flux": [5, 5, 5],
                                         "keyframes": [{"frame": 0, "translation": [0, 2, 1]}]}])),
    ("one-dynamic-triangle", _doc([ROOM, TRI_MOVER], [{"kind": "disc_area", "flux": [5, 5, 5], "radius": 0.2,
                                                        "keyframes": [{"frame": 0, "translation": [0, 2.9, 0]}]}])),
    ("light-facing-away", _doc([ROOM], [{"kind": "spot", "flux": [5, 5, 5], "cone_angle": 20,
                                         "keyframes": [{"frame": 0, "translation": [0, 1, 3.5],
                                                        "rotation": [1, 0, 0, 0]}]}])),
])
def test_degenerate_scenes_bit_exact(name, doc):
    from oracle import ref

    cfg = dict(mode="error", paths=3001, bounces=4, dm=[2, 2, 8, 8], threshold=0.001, seed=31)
    gpu = pr.Engine(pr.Scene.from_text(doc), pr.make_config(**cfg))
    cpu = ref.RefEngine(ref.RefScene.from_text(doc), pr.make_config(**cfg))
    cpu.set_workers(0)
    for f in range(4):
        sg, sc = gpu.run_frame(), cpu.run_frame()
        assert counts(sg) == counts(sc), (name, f)
        bad = compare_state(gpu, cpu, gpu.info().n_lights)
        assert all(v == 0 for v in bad.values()), (name, f, bad)
    assert gpu.splat(radius=0.25).tobytes() == cpu.gather(radius=0.25)[0].tobytes()
