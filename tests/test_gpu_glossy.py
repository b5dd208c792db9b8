"""Glossy materials: phong_lobe_sample (engine.cpp:34-42) and the
forced retrace of glossy hits (engine.cpp:373-384), bit-exact against the reference.

The engine tabulates the host libm's powf(k * 2^-24, 1 / (exponent + 1)) per distinct
glossy exponent, so glossy bounce directions match the reference bit for bit, like the
cosine lobe does through the sincosf table.
"""
import pytest

from paper_2111_06906_b200 import _lib as L
from paper_2111_06906_b200 import pathreuse as pr
from tests.helpers import compare_state, counts

GLOSSY = 1  # PRX_MATERIAL_GLOSSY (prx.h, scene.hpp:16)


def glossy_variant(name, exponents):
    """Builtin scene `name` with objects i (of `exponents`) turned glossy."""
    base = pr.Scene.builtin(name)
    d = base.describe()
    objs = (L.ObjectDesc * d.n_objects)(*[d.objects[i] for i in range(d.n_objects)])
    for i, e in exponents.items():
        objs[i].material.kind = GLOSSY
        objs[i].material.glossy_exponent = e
    desc = L.SceneDesc(objects=objs, n_objects=d.n_objects, lights=d.lights, n_lights=d.n_lights,
                       camera=d.camera, frames=d.frames)
    return base, objs, desc


@pytest.mark.gpu
@pytest.mark.parametrize("scene,mode,exps", [
    ("moving-cube", "error", {0: 20.0, 2: 20.0}),
    ("moving-cube", "naive", {0: 8.0}),
    ("villa-analog", "error", {0: 50.0, 2: 3.0}),
])
def test_glossy_bit_exact(scene, mode, exps):
    from oracle import ref

    base, objs, desc = glossy_variant(scene, exps)
    gscene = pr.Scene.from_desc(desc)
    rscene = ref.RefScene.from_desc(desc)
    cfg = dict(mode=mode, paths=4000, bounces=6, dm=[2, 2, 8, 8], threshold=0.001, seed=5)
    gpu = pr.Engine(gscene, pr.make_config(**cfg))
    cpu = ref.RefEngine(rscene, pr.make_config(**cfg))
    cpu.set_workers(0)
    n_lights = gpu.info().n_lights
    for f in range(4):
        sg, sc = gpu.run_frame(), cpu.run_frame()
        assert counts(sg) == counts(sc), f"frame {f}: gpu {counts(sg)} ref {counts(sc)}"
        bad = compare_state(gpu, cpu, n_lights)
        assert all(v == 0 for v in bad.values()), f"frame {f}: mismatches {bad}"
