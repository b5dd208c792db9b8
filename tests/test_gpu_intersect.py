"""intersect_scene / occluded (scene.cpp:136-177) as GPU batch queries vs the reference, on
random and adversarial rays: axis-parallel and zero-component directions, origins on
vertices, rays aimed at shared edges and vertices (exact-t ties between triangles, resolved
by the reference's DFS / index order), finite t_max windows, camera rays.

This stresses the certified fast traversal directly: every hit must match the reference's
(t, object, triangle, position, normal) bit for bit.
"""
import numpy as np
import pytest

from paper_2111_06906_b200 import pathreuse as pr

FLT_MAX = np.float32(3.4028235e38)


def scene_triangles(desc):
    tris = []
    for i in range(desc.n_objects):
        o = desc.objects[i]
        for t in range(o.n_triangles):
            m = o.mesh[t]
            tris.append([[m.a.x, m.a.y, m.a.z], [m.b.x, m.b.y, m.b.z], [m.c.x, m.c.y, m.c.z]])
    return np.array(tris, dtype=np.float32)


def unit(v):
    v = v.astype(np.float32)
    n = np.sqrt((v * v).sum(axis=1, dtype=np.float32)).astype(np.float32)
    n[n == 0] = 1
    return (v / n[:, None]).astype(np.float32)


def make_rays(desc, n, rng, diag):
    tris = scene_triangles(desc)
    lo, hi = tris.reshape(-1, 3).min(0), tris.reshape(-1, 3).max(0)
    rays = []
    k = n // 6
    # 1. random origins / directions
    o = lo + (hi - lo) * rng.random((k, 3), dtype=np.float32)
    d = unit(rng.normal(size=(k, 3)))
    rays.append((o, d))
    # 2. axis-parallel and one-zero-component directions
    o = lo + (hi - lo) * rng.random((k, 3), dtype=np.float32)
    d = np.zeros((k, 3), dtype=np.float32)
    axis = rng.integers(0, 3, k)
    d[np.arange(k), axis] = rng.choice([-1.0, 1.0], k)
    half = k // 2
    d2 = unit(rng.normal(size=(half, 3)))
    d2[np.arange(half), rng.integers(0, 3, half)] = 0
    d[:half] = unit(d2)
    rays.append((o, d))
    # 3. origins on vertices towards other triangles' centroids
    ia, ib = rng.integers(0, len(tris), k), rng.integers(0, len(tris), k)
    o = tris[ia, rng.integers(0, 3, k)]
    d = unit(tris[ib].mean(axis=1) - o)
    rays.append((o, d))
    # 4. aimed at shared edges (edge midpoints) and vertices from random points
    o = lo + (hi - lo) * rng.random((k, 3), dtype=np.float32)
    e = rng.integers(0, 3, k)
    tgt = ((tris[ia, e] + tris[ia, (e + 1) % 3]) * np.float32(0.5)).astype(np.float32)
    tgt[: k // 3] = tris[ia[: k // 3], e[: k // 3]]
    d = unit(tgt - o)
    rays.append((o, d))
    # 5. grazing: origin on a triangle, direction in its plane
    t = tris[ia]
    o = t[:, 0]
    d = unit(t[:, 1] - t[:, 0] + (t[:, 2] - t[:, 0]) * rng.random((k, 1), dtype=np.float32))
    rays.append((o, d))
    # 6. random with finite windows
    o = lo + (hi - lo) * rng.random((n - 5 * k, 3), dtype=np.float32)
    d = unit(rng.normal(size=(n - 5 * k, 3)))
    rays.append((o, d))
    o = np.concatenate([r[0] for r in rays]).astype(np.float32)
    d = np.concatenate([r[1] for r in rays]).astype(np.float32)
    out = np.zeros((len(o), 8), dtype=np.float32)
    out[:, :3], out[:, 3:6] = o, d
    out[:, 6] = np.where(rng.random(len(o)) < 0.5, np.float32(0), np.float32(1e-4) * np.float32(diag))
    out[:, 7] = FLT_MAX
    last = len(o) - (n - 5 * k)
    out[last:, 7] = (rng.random(n - 5 * k) * diag * 0.5).astype(np.float32)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("scene,synthetic,frames", [("moving-cube", False, 3), ("villa-analog", False, 2),
                                                     ("armadillo-analog", False, 2), ("C3", True, 2),
                                                     ("C1", True, 4), ("C4", True, 2)])
def test_intersect_and_occluded_bit_exact(scene, synthetic, frames):
    from oracle import ref

    sc = pr.Scene.synthetic(scene) if synthetic else pr.Scene.builtin(scene)
    rs = ref.RefScene.from_desc(sc.describe()) if synthetic else ref.RefScene.builtin(scene)
    eng = pr.Engine(sc, pr.make_config("naive", paths=1000, bounces=2, dm=[2, 2, 4, 4]))
    for _ in range(frames):
        eng.run_frame()
    frame = eng.info().frames_run - 1
    rng = np.random.default_rng(17)
    rays = make_rays(sc.describe(), 60000, rng, sc.diagonal)
    got = eng.intersect(rays)
    want = rs.intersect(frame, rays)
    bad = np.any(got.view(np.uint32) != want.view(np.uint32), axis=1)
    assert not bad.any(), f"{bad.sum()} of {len(rays)} rays differ, first {np.nonzero(bad)[0][:5]}"
    hits = got[:, 1].view(np.uint32) != 0xFFFFFFFF
    assert hits.mean() > 0.3
    occ = eng.intersect(rays, any_hit=True)
    assert np.array_equal(occ, rs.occluded(frame, rays))


@pytest.mark.gpu
@pytest.mark.parametrize("tree", ["sah", "karras"])
@pytest.mark.parametrize("scene", ["merry-go-round-analog", "C4"])
def test_dynamic_tree_variants_bit_exact(monkeypatch, tree, scene):
    """The combined dynamic tree is either per-object SAH topologies refit every frame (the
    default) or a per-frame Karras rebuild (PRX_DYN_TREE=karras); the query result must not
    depend on it."""
    from oracle import ref

    monkeypatch.setenv("PRX_DYN_TREE", tree)
    synthetic = scene.startswith("C")
    sc = pr.Scene.synthetic(scene) if synthetic else pr.Scene.builtin(scene)
    rs = ref.RefScene.from_desc(sc.describe()) if synthetic else ref.RefScene.builtin(scene)
    eng = pr.Engine(sc, pr.make_config("naive", paths=1000, bounces=2, dm=[2, 2, 4, 4]))
    for _ in range(3):
        eng.run_frame()
    frame = eng.info().frames_run - 1
    rays = make_rays(sc.describe(), 40000, np.random.default_rng(23), sc.diagonal)
    assert np.array_equal(eng.intersect(rays).view(np.uint32), rs.intersect(frame, rays).view(np.uint32))
    assert np.array_equal(eng.intersect(rays, any_hit=True), rs.occluded(frame, rays))


@pytest.mark.gpu
@pytest.mark.parametrize("scene", ["merry-go-round-analog", "C3"])
def test_exact_fallbacks_bit_exact(monkeypatch, scene):
    """PRX_CERT_OFF=1 fails every certificate, so each query takes the exact fallback the
    fast path relies on in its rare certificate failures (reference-order static DFS, the
    sequential gated dynamic phase over per-object subtrees); engine state and queries must
    still match the reference."""
    from oracle import ref
    from tests.helpers import compare_state, counts

    monkeypatch.setenv("PRX_CERT_OFF", "1")
    synthetic = scene.startswith("C")
    sc = pr.Scene.synthetic(scene) if synthetic else pr.Scene.builtin(scene)
    rs = ref.RefScene.from_desc(sc.describe()) if synthetic else ref.RefScene.builtin(scene)
    cfg = dict(mode="error", paths=3000, bounces=4, dm=[2, 2, 8, 8], threshold=0.001, seed=41)
    eng = pr.Engine(sc, pr.make_config(**cfg))
    cpu = ref.RefEngine(rs, pr.make_config(**cfg))
    cpu.set_workers(0)
    for f in range(3):
        sg, scs = eng.run_frame(), cpu.run_frame()
        assert counts(sg) == counts(scs), f
        bad = compare_state(eng, cpu, eng.info().n_lights)
        assert all(v == 0 for v in bad.values()), (f, bad)
    frame = eng.info().frames_run - 1
    rays = make_rays(sc.describe(), 12000, np.random.default_rng(29), sc.diagonal)
    assert np.array_equal(eng.intersect(rays).view(np.uint32), rs.intersect(frame, rays).view(np.uint32))
    assert np.array_equal(eng.intersect(rays, any_hit=True), rs.occluded(frame, rays))


def _offset_doc(offset):
    """test_io's document with every object and light moved far from the origin."""
    import json

    from tests.test_io import DOC

    d = json.loads(DOC)
    ox, oy, oz = offset
    for node in d["objects"] + d["lights"]:
        kfs = node.get("keyframes") or [{"frame": 0}]
        for kf in kfs:
            t = kf.get("translation", [0, 0, 0])
            kf["translation"] = [t[0] + ox, t[1] + oy, t[2] + oz]
        node["keyframes"] = kfs
    c = d["camera"]
    c["position"] = [c["position"][0] + ox, c["position"][1] + oy, c["position"][2] + oz]
    c["look_at"] = [c["look_at"][0] + ox, c["look_at"][1] + oy, c["look_at"][2] + oz]
    return json.dumps(d)


@pytest.mark.gpu
@pytest.mark.parametrize("offset", [(12345.0, -6789.0, 4321.5), (-3.0e5, 2.5e5, 1.0e5)])
def test_far_from_origin_bit_exact(tmp_path, offset):
    """Coordinates far from the origin stress the float filters' margins (slab quotients,
    box inflation relative to the scene diagonal, fma culling error bounds)."""
    from oracle import ref
    from tests.helpers import compare_state, counts
    from tests.test_io import OBJ_TEXT

    (tmp_path / "part.obj").write_text(OBJ_TEXT)
    doc = _offset_doc(offset)
    sc = pr.Scene.from_text(doc, str(tmp_path))
    rs = ref.RefScene.from_text(doc, str(tmp_path))
    cfg = dict(mode="error", paths=4000, bounces=5, dm=[2, 2, 8, 8], threshold=0.001, seed=3)
    eng = pr.Engine(sc, pr.make_config(**cfg))
    cpu = ref.RefEngine(rs, pr.make_config(**cfg))
    cpu.set_workers(0)
    for f in range(3):
        sg, scs = eng.run_frame(), cpu.run_frame()
        assert counts(sg) == counts(scs), f"frame {f}"
        bad = compare_state(eng, cpu, eng.info().n_lights)
        assert all(v == 0 for v in bad.values()), f"frame {f}: {bad}"
    rays = make_rays(sc.describe(), 30000, np.random.default_rng(5), sc.diagonal)
    frame = eng.info().frames_run - 1
    got, want = eng.intersect(rays), rs.intersect(frame, rays)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert np.array_equal(eng.intersect(rays, any_hit=True), rs.occluded(frame, rays))


@pytest.mark.gpu
@pytest.mark.parametrize("scene,synthetic", [("villa-analog", False), ("C4", True)])
def test_negative_t_min_bit_exact(scene, synthetic):
    """Rays with t_min < 0 (hits behind the origin count) take the careful culling slabs (the
    fast slabs' one-product acceptance assumes t_min >= 0); results stay bit-exact."""
    from oracle import ref

    sc = pr.Scene.synthetic(scene) if synthetic else pr.Scene.builtin(scene)
    rs = ref.RefScene.from_desc(sc.describe()) if synthetic else ref.RefScene.builtin(scene)
    eng = pr.Engine(sc, pr.make_config("naive", paths=1000, bounces=2, dm=[2, 2, 4, 4]))
    eng.run_frame()
    frame = eng.info().frames_run - 1
    rng = np.random.default_rng(23)
    rays = make_rays(sc.describe(), 30000, rng, sc.diagonal)
    neg = rng.random(len(rays)) < 0.5
    rays[neg, 6] = -(rng.random(int(neg.sum())) * sc.diagonal * 0.5).astype(np.float32)
    got = eng.intersect(rays)
    want = rs.intersect(frame, rays)
    bad = np.any(got.view(np.uint32) != want.view(np.uint32), axis=1)
    assert not bad.any(), f"{bad.sum()} of {len(rays)} rays differ"
    assert np.array_equal(eng.intersect(rays, any_hit=True), rs.occluded(frame, rays))


@pytest.mark.gpu
def test_degenerate_query_rays_bit_exact():
    """Scene-query rays the engine itself never casts: zero direction, negative zero
    components, inverted windows (t_max < t_min), infinite t_max, origins far outside the
    scene -- all against the reference's intersect_scene / occluded."""
    from oracle import ref

    sc = pr.Scene.synthetic("C4")
    rs = ref.RefScene.from_desc(sc.describe())
    eng = pr.Engine(sc, pr.make_config("naive", paths=1000, bounces=2, dm=[2, 2, 4, 4]))
    eng.run_frame()
    frame = eng.info().frames_run - 1
    rng = np.random.default_rng(29)
    rays = make_rays(sc.describe(), 6000, rng, sc.diagonal)
    n = len(rays)
    q = n // 6
    rays[:q, 3:6] = 0.0                                   # zero direction
    rays[q:2 * q, 3] = np.float32(-0.0)                   # a negative-zero component
    rays[2 * q:3 * q, 6], rays[2 * q:3 * q, 7] = 1.0, 0.5  # inverted window
    rays[3 * q:4 * q, 7] = np.inf                          # infinite t_max
    rays[4 * q:5 * q, :3] *= np.float32(1e3)               # far outside the scene
    got = eng.intersect(rays)
    want = rs.intersect(frame, rays)
    bad = np.any(got.view(np.uint32) != want.view(np.uint32), axis=1)
    assert not bad.any(), f"{bad.sum()} of {n} rays differ, first {np.nonzero(bad)[0][:5]}"
    assert np.array_equal(eng.intersect(rays, any_hit=True), rs.occluded(frame, rays))
