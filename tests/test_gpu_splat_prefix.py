"""The splat prefix (G-buffer + cell-key table of the scene camera) that run_frame computes on a
side stream during verify/retrace (engine.cpp: Engine::splat_prefix_fork) must give the same
image as gather_image (gather.cpp:35-75) through every sequence that can invalidate it:
moving dynamics, a new radius, another camera in between, the scene camera passed explicitly,
frames run through the stage API, and graph-replayed frames.
"""
import numpy as np
import pytest

from paper_2111_06906_b200 import _lib as L
from tests.helpers import pair


def _splat_launches(gpu, **kw):
    l0 = gpu.launch_count()
    img = gpu.splat(**kw)
    return img, gpu.launch_count() - l0


@pytest.mark.gpu
@pytest.mark.parametrize("scene,synthetic,mode", [("moving-cube", False, "error"), ("C4", True, "error"),
                                                  ("merry-go-round-analog", False, "naive")])
def test_prefix_images_bit_exact(scene, synthetic, mode):
    gpu, cpu = pair(scene, synthetic=synthetic, mode=mode, paths=40000, bounces=5, dm=[2, 2, 8, 8], seed=5)
    cam = gpu.scene.describe().camera
    same = L.Camera(cam.position, cam.look_at, cam.fov_deg, cam.width, cam.height)
    other = L.Camera(cam.position, cam.look_at, cam.fov_deg + 5.0, 160, 100)
    launches = {}
    for f in range(7):
        gpu.run_frame()
        cpu.run_frame()
        radius = 0.3 if f == 4 else 0.25  # frame 4: a new radius (the prefix is recomputed inline)
        for label, kw in (("scene", dict(radius=radius)), ("explicit", dict(camera=same, radius=radius)),
                          ("other", dict(camera=other, radius=radius))):
            img, n = _splat_launches(gpu, mode=1, **kw)
            ref_kw = dict(kw)
            img_c = cpu.gather(**ref_kw)[0]
            assert np.array_equal(img, img_c), (f, label, int(np.any(img != img_c, axis=-1).sum()))
            launches.setdefault(label, []).append(n)
        # atomic splat on the same prefix
        img0 = gpu.splat(radius=radius, mode=0)
        img1 = gpu.splat(radius=radius, mode=1)
        assert np.array_equal(img0 == 0, img1 == 0)
    # frames 1-3, 6 reuse the prefix (scene camera, same radius): fewer launches than the
    # other camera (no G-buffer / cell table, and a sort over the dense cell ids' bits);
    # frame 0 (no radius yet) and frame 5 (radius changed back) do not
    sc, ot = launches["scene"], launches["other"]
    for f in (1, 2, 3, 6):
        assert sc[f] < ot[f], (f, sc, ot)
        assert launches["explicit"][f] == sc[f]
    assert sc[0] == ot[0] and sc[5] == ot[5], (sc, ot)


@pytest.mark.gpu
def test_prefix_after_stage_api_frame():
    """frames run stage by stage move the dynamics without the side stream: the splat must not
    reuse the previous frame's prefix."""
    gpu, cpu = pair("C4", synthetic=True, mode="error", paths=30000, bounces=5, dm=[2, 2, 8, 8], seed=7)
    for _ in range(3):
        gpu.run_frame()
        cpu.run_frame()
        assert np.array_equal(gpu.splat(radius=0.25), cpu.gather(radius=0.25)[0])
    for _ in range(2):
        st = gpu.frame_update()
        gpu.verify_paths(st)
        gpu.retrace_invalid(st)
        cpu.run_frame()
        img, n = _splat_launches(gpu, radius=0.25)
        assert np.array_equal(img, cpu.gather(radius=0.25)[0])
    gpu.run_frame()
    cpu.run_frame()
    assert np.array_equal(gpu.splat(radius=0.25), cpu.gather(radius=0.25)[0])
