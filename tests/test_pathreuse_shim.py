"""The `pathreuse` import shim (pathreuse/__init__.py): the reference's Python module surface
(python/pathreuse/__init__.py:3-12) served by the B200 engine.

* Here (CPU): the reference's own tests/python/test_smoke.py, unmodified, is run against the
  shim when /root/reference is present -- its four pure-function tests must pass (the two
  engine tests need a GPU and are deselected).
* On the GPU: the same six checks restated (the reference tree is not on the GPU box), so
  the engine-backed run_builtin / render_builtin are exercised through `import pathreuse`.
"""
import math
import os
import struct
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SMOKE = "/root/reference/proj/tests/python/test_smoke.py"


def test_shim_exports_the_reference_surface():
    import pathreuse

    assert sorted(pathreuse.__all__) == sorted(["builtin_scenes", "decode_path_info", "encode_path_info",
                                                "energies_close", "memory_footprint", "prune_probability",
                                                "render_builtin", "run_builtin"])
    assert "villa-analog" in pathreuse.builtin_scenes()


@pytest.mark.skipif(not os.path.exists(REF_SMOKE), reason="reference tree not present")
def test_reference_python_smoke_pure_functions():
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", REF_SMOKE,
                          "-k", "not run_builtin and not render_builtin", "--rootdir", "/tmp"],
                         capture_output=True, text=True, env=env, cwd="/tmp")
    assert out.returncode == 0, out.stdout + out.stderr
    assert "4 passed" in out.stdout


def test_pure_functions_through_the_shim():
    import pathreuse

    assert pathreuse.prune_probability(10, 4) == pytest.approx(0.6)
    assert pathreuse.prune_probability(4, 10) == 0.0 and pathreuse.prune_probability(0, 5) == 0.0
    assert pathreuse.energies_close([1.0, 1.0, 1.0], [1.0005, 1.0, 0.9995], 0.001)
    assert not pathreuse.energies_close([1.0, 1.0, 1.0], [1.1, 1.0, 1.0], 0.001)
    word = pathreuse.encode_path_info(cell=5, seg_count=7, retrace_start=0, replace=False, reuse_light=True)
    assert word == 0x81800005
    f = pathreuse.decode_path_info(word)
    assert (f["cell"], f["seg_count"], f["reuse_light"]) == (5, 7, True)
    fp = pathreuse.memory_footprint(5_000_000, 7, [32, 32, 32, 32], True)
    assert fp["photon_map"] == pytest.approx(1068.12, rel=5e-3)
    assert fp["subtotal_reuse"] == pytest.approx(103.36, rel=5e-3)


@pytest.mark.gpu
def test_run_builtin_static_scene_reuses_everything():
    import pathreuse

    rows = pathreuse.run_builtin("static-box", mode="naive", paths=2000, frames=3, dm=[1, 1, 8, 8])
    assert rows[0]["rays_traced"] > 0
    assert rows[1]["rays_traced"] == 0 and rows[2]["rays_traced"] == 0


@pytest.mark.gpu
def test_render_builtin_returns_image():
    import pathreuse

    w, h, raw = pathreuse.render_builtin("static-box", paths=2000, frames=1, dm=[1, 1, 8, 8])
    assert w > 0 and h > 0
    px = struct.unpack(f"<{3 * w * h}f", raw)
    assert all(math.isfinite(v) and v >= 0.0 for v in px)
    assert any(v > 0.0 for v in px)
