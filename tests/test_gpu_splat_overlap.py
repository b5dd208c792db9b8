"""Overlapped splat (prx_engine_set_splat_overlap): the splat of frame N runs on the engine's
side stream while frame N+1 updates the scene and computes its occlusion flags; frame N+1
waits for it before its first photon-map write (the verify walk / compute_dm / baseline
release) and before recomputing the splat prefix.  Every frame's state and every image must
still equal the reference's (engine.cpp:201-242, gather.cpp:35-75), through graph-replayed
frames, mixed with synchronous splats and downloads.
"""
import numpy as np
import pytest

from tests.helpers import compare_state, pair


def _img(buf, cam):
    return buf.cpu().numpy().reshape(cam.height, cam.width, 3)


@pytest.mark.gpu
@pytest.mark.parametrize("scene,synthetic,mode,graphs", [("C4", True, "error", "1"), ("C4", True, "error", "0"),
                                                         ("moving-cube", False, "naive", "1"),
                                                         ("merry-go-round-analog", False, "baseline", "1")])
def test_overlapped_splat_bit_exact(monkeypatch, scene, synthetic, mode, graphs):
    """graphs "0": plain stream launches (PRX_GRAPHS=0) instead of replayed frame graphs."""
    import torch

    monkeypatch.setenv("PRX_GRAPHS", graphs)
    gpu, cpu = pair(scene, synthetic=synthetic, mode=mode, paths=30000, bounces=5, dm=[2, 2, 8, 8], seed=11)
    gpu.set_splat_overlap(True)
    cam = gpu.scene.describe().camera
    buf = torch.zeros(cam.height * cam.width * 3, dtype=torch.float32, device="cuda")
    pending = None  # reference image of the splat in flight
    n_lights = gpu.info().n_lights
    for f in range(8):
        gpu.run_frame()  # waits for the previous frame's splat before touching the photon map
        if pending is not None:
            assert np.array_equal(_img(buf, cam), pending), f
        cpu.run_frame()
        if f in (3, 6):  # downloads and a synchronous splat in between (both join the side stream)
            bad = compare_state(gpu, cpu, n_lights)
            assert not any(bad.values()), (f, bad)
            assert np.array_equal(gpu.splat(radius=0.25), cpu.gather(radius=0.25)[0]), f
        pending = cpu.gather(radius=0.25)[0]
        gpu.splat_device(buf.data_ptr(), radius=0.25)  # asynchronous
    gpu.synchronize()
    assert np.array_equal(_img(buf, cam), pending)
    bad = compare_state(gpu, cpu, n_lights)
    assert not any(bad.values()), bad


@pytest.mark.gpu
def test_overlap_toggle_and_other_camera():
    """Switching the overlap off and on again, and splats that cannot overlap (another camera,
    host output), stay exact."""
    import torch
    from paper_2111_06906_b200 import _lib as L

    gpu, cpu = pair("C4", synthetic=True, mode="error", paths=20000, bounces=5, dm=[2, 2, 8, 8], seed=4)
    cam = gpu.scene.describe().camera
    other = L.Camera(cam.position, cam.look_at, cam.fov_deg + 3.0, 64, 48)
    buf = torch.zeros(cam.height * cam.width * 3, dtype=torch.float32, device="cuda")
    obuf = torch.zeros(64 * 48 * 3, dtype=torch.float32, device="cuda")
    for f in range(6):
        gpu.set_splat_overlap(f % 3 != 2)
        gpu.run_frame()
        cpu.run_frame()
        gpu.splat_device(buf.data_ptr(), radius=0.25)
        gpu.splat_device(obuf.data_ptr(), camera=other, radius=0.25)  # synchronous (not the scene camera)
        assert np.array_equal(obuf.cpu().numpy().reshape(48, 64, 3), cpu.gather(camera=other, radius=0.25)[0]), f
        gpu.synchronize()
        assert np.array_equal(_img(buf, cam), cpu.gather(radius=0.25)[0]), f


@pytest.mark.gpu
def test_overlapped_host_splat():
    """splat_into a host array with the overlap on: filled by the next engine call, equal to
    gather_image of its frame (the bench's pipelined e2e loop)."""
    gpu, cpu = pair("C4", synthetic=True, mode="error", paths=30000, bounces=5, dm=[2, 2, 8, 8], seed=8)
    gpu.set_splat_overlap(True)
    cam = gpu.scene.describe().camera
    out = np.zeros((cam.height, cam.width, 3), dtype=np.float32)
    pending = None
    for f in range(7):
        gpu.run_frame()
        if pending is not None:
            assert np.array_equal(out, pending), f
        cpu.run_frame()
        pending = cpu.gather(radius=0.25)[0]
        out[...] = -1.0
        gpu.splat_into(out, radius=0.25)
    gpu.synchronize()
    assert np.array_equal(out, pending)
