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
