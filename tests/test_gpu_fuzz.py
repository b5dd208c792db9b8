"""Randomised configurations, bit-exact against the reference: scene, mode, path count,
bounce limit, DM layout, threshold and seed drawn per case from a fixed generator, three
frames each, then the image. Complements the hand-picked cases of test_gpu_parity.py and
test_gpu_edges.py with combinations nobody chose."""
import numpy as np
import pytest

from paper_2111_06906_b200 import pathreuse as pr
from tests.helpers import compare_state, counts

SCENES = ["static-box", "moving-cube", "parallel-spot", "merry-go-round-analog", "armadillo-analog",
          "villa-analog"]


def draw(case):
    rng = np.random.default_rng(1000 + case)
    scene = SCENES[int(rng.integers(len(SCENES)))]
    mode = ["naive", "error", "baseline"][int(rng.integers(3))]
    bounces = int(rng.integers(1, 17))
    paths = int(rng.integers(50, 6000))
    dm = [int(rng.integers(1, 9)), int(rng.integers(1, 9)), int(rng.integers(1, 33)), int(rng.integers(1, 33))]
    threshold = float([0.0, 1e-4, 1e-3, 1e-2, 0.1, 1e9][int(rng.integers(6))])
    seed = int(rng.integers(1, 2**31))
    frames = int(rng.integers(2, 5))
    return dict(scene=scene, mode=mode, paths=paths, bounces=bounces, dm=dm, threshold=threshold, seed=seed,
                frames=frames)


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(96))
def test_random_configs_bit_exact(case):
    from oracle import ref

    c = draw(case)
    cfg = dict(mode=c["mode"], paths=c["paths"], bounces=c["bounces"], dm=c["dm"], threshold=c["threshold"],
               seed=c["seed"])
    gpu = pr.Engine(pr.Scene.builtin(c["scene"]), pr.make_config(**cfg))
    cpu = ref.RefEngine(ref.RefScene.builtin(c["scene"]), pr.make_config(**cfg))
    cpu.set_workers(0)
    n_lights = gpu.info().n_lights
    for f in range(c["frames"]):
        sg, sc = gpu.run_frame(), cpu.run_frame()
        assert counts(sg) == counts(sc), (c, f)
        bad = compare_state(gpu, cpu, n_lights)
        assert all(v == 0 for v in bad.values()), (c, f, bad)
    assert gpu.splat(radius=0.25).tobytes() == cpu.gather(radius=0.25)[0].tobytes(), c


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(6))
def test_random_configs_synthetic_bit_exact(case):
    """The same on the synthetic C1/C3 scenes (282K static triangles and movers for C3)."""
    from oracle import ref

    c = draw(500 + case)
    name = ["C1", "C3"][case % 2]
    cfg = dict(mode=c["mode"], paths=min(c["paths"], 3000), bounces=c["bounces"], dm=c["dm"],
               threshold=c["threshold"], seed=c["seed"])
    scene = pr.Scene.synthetic(name)
    gpu = pr.Engine(scene, pr.make_config(**cfg))
    cpu = ref.RefEngine(ref.RefScene.from_desc(scene.describe()), pr.make_config(**cfg))
    cpu.set_workers(0)
    for f in range(c["frames"]):
        sg, sc = gpu.run_frame(), cpu.run_frame()
        assert counts(sg) == counts(sc), (name, c, f)
        bad = compare_state(gpu, cpu, gpu.info().n_lights)
        assert all(v == 0 for v in bad.values()), (name, c, f, bad)
    assert gpu.splat(radius=0.25).tobytes() == cpu.gather(radius=0.25)[0].tobytes(), (name, c)
