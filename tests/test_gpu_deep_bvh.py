"""Adversarial BVH depth: log-spaced triangle centroids make a binned SAH peel
off a few triangles per level, so an unbounded build would exceed the traversal's 64-entry
stack (device_scene.cuh fast_closest / joint_closest).  The builder caps the depth
(fast_bvh.cpp kMaxDepth, centroid-median splits below it); these scenes must still match the
reference's intersect_scene (scene.cpp:136-177) and a full frame bit for bit."""
import json

import numpy as np
import pytest

from paper_2111_06906_b200 import pathreuse as pr
from tests.helpers import compare_state, counts
from tests.test_gpu_intersect import make_rays


def staircase(n=200, ratio=1.5, size=1e-3):
    """Three chains of equal small triangles with centroids at ratio^k along x, y and z (the
    tests/cpp/bvh_depth.cpp chains: 86 levels deep without the cap)."""
    verts, faces = [], []
    for axis in range(3):
        for k in range(n):
            c = float(np.float32(ratio) ** np.float32(k - n // 2))
            base = len(verts)
            for du, dv in ((-size, -size), (size, -size), (0.0, size)):
                p = [0.0, 0.0, 0.0]
                p[axis] = c
                p[(axis + 1) % 3] += du
                p[(axis + 2) % 3] += dv
                verts.append([float(np.float32(x)) for x in p])
            faces.append([base, base + 1, base + 2])
    return {"vertices": verts, "faces": faces}


def doc():
    return json.dumps({
        "frames": 8,
        "camera": {"position": [-6, 0, 0], "look_at": [0, 0, 0], "fov": 50, "resolution": [32, 24]},
        "objects": [
            {"name": "stairs", "material": {"kind": "diffuse", "albedo": [0.7, 0.7, 0.7]}, "mesh": staircase()},
            {"name": "floor", "material": {"kind": "diffuse", "albedo": [0.5, 0.5, 0.5]},
             "mesh": {"vertices": [[-4, -2, -4], [4, -2, -4], [4, -2, 4], [-4, -2, 4]], "faces": [[0, 1, 2], [0, 2, 3]]}},
            {"name": "mover", "material": {"kind": "diffuse", "albedo": [0.6, 0.5, 0.4]}, "mesh": staircase(),
             "keyframes": [{"frame": 0, "translation": [0.0, 0.5, 0.3]}, {"frame": 7, "translation": [0.2, 0.0, -0.3]}]},
        ],
        "lights": [{"kind": "point", "flux": [10, 10, 10], "keyframes": [{"frame": 0, "translation": [-3, 0.5, 0.2]}]}],
    })


@pytest.mark.gpu
def test_deep_staircase_bit_exact():
    from oracle import ref

    text = doc()
    sc, rs = pr.Scene.from_text(text), ref.RefScene.from_text(text)
    cfg = dict(mode="naive", paths=4000, bounces=4, dm=[2, 2, 8, 8], seed=3)
    gpu = pr.Engine(sc, pr.make_config(**cfg))
    cpu = ref.RefEngine(rs, pr.make_config(**cfg))
    for f in range(3):
        assert counts(gpu.run_frame()) == counts(cpu.run_frame()), f
    bad = compare_state(gpu, cpu, 1)
    assert all(v == 0 for v in bad.values()), bad
    rng = np.random.default_rng(5)
    rays = make_rays(sc.describe(), 30000, rng, sc.diagonal)
    # plus rays straight down the staircase axis (every triangle's box is entered)
    m = 3000
    ax = np.zeros((m, 8), dtype=np.float32)
    ax[:, 0] = -2.0
    ax[:, 1:3] = rng.uniform(-1e-3, 1e-3, (m, 2)).astype(np.float32)
    d = np.column_stack([np.ones(m), rng.normal(0, 1e-3, (m, 2))]).astype(np.float32)
    ax[:, 3:6] = d / np.linalg.norm(d, axis=1, keepdims=True).astype(np.float32)
    ax[:, 7] = np.float32(3.4028235e38)
    rays = np.concatenate([rays, ax])
    frame = gpu.info().frames_run - 1
    got, want = gpu.intersect(rays), rs.intersect(frame, rays)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
