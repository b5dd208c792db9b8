"""Scene documents and offline artefacts, against the reference's
own loader and writers (oracle/_ref): same scenes bit for bit, byte-identical files.

CPU only: the loader and writers are host code behind the C ABI (csrc/scene_io.cpp,
csrc/wire.cpp); the engine-level photon dump is covered in test_gpu_io.py.
"""
import struct

import numpy as np
import pytest

from paper_2111_06906_b200 import _lib as L
from paper_2111_06906_b200 import pathreuse as pr

ref = pytest.importorskip("oracle.ref")
pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def f32(x):
    return struct.pack("<f", x)


def digest(desc: L.SceneDesc):
    """Every field of a scene description, floats as raw bytes."""
    v3 = lambda v: f32(v.x) + f32(v.y) + f32(v.z)
    kfs = lambda p, n: [(p[i].frame, v3(p[i].translation), f32(p[i].rotation.x) + f32(p[i].rotation.y)
                         + f32(p[i].rotation.z) + f32(p[i].rotation.w), f32(p[i].scale)) for i in range(n)]
    objs = []
    for i in range(desc.n_objects):
        o = desc.objects[i]
        mesh = b"".join(v3(o.mesh[t].a) + v3(o.mesh[t].b) + v3(o.mesh[t].c) for t in range(o.n_triangles))
        objs.append((o.name, mesh, o.material.kind, v3(o.material.albedo), f32(o.material.glossy_exponent),
                     kfs(o.keyframes, o.n_keyframes)))
    lights = []
    for i in range(desc.n_lights):
        li = desc.lights[i]
        lights.append((li.kind, v3(li.flux), f32(li.cone_angle_deg), f32(li.radius), f32(li.half_x),
                       f32(li.half_y), kfs(li.keyframes, li.n_keyframes)))
    c = desc.camera
    return objs, lights, (v3(c.position), v3(c.look_at), f32(c.fov_deg), c.width, c.height), desc.frames


def both(text, base_dir=""):
    ours = pr.Scene.from_text(text, base_dir)
    theirs = ref.RefScene.from_text(text, base_dir)
    return ours, theirs


OBJ_TEXT = """# a quad, a fan and negative indices
v 0 0 0
v 1.0000001 0 0
v 1 1 0
v 0 1e0 0
v 0.5 0.5 -0.3333333333
f 1 2 3 4
f 1/1 3/3/3 5//5
f -1 -2 -3
"""

DOC = """{
  "frames": 12,
  "camera": {"position": [0, 1.5, 4.25], "look_at": [0, 0.9, 0], "fov": 55, "resolution": [64, 48]},
  "objects": [
    {"name": "room", "material": {"kind": "diffuse", "albedo": [0.8, 0.75, 0.7]},
     "mesh": {"vertices": [[-3,0,-3],[3,0,-3],[3,0,3],[-3,0,3],[-3,3,-3],[3,3,-3]],
              "faces": [[0,1,2],[0,2,3],[0,4,5],[0,5,1]]}},
    {"name": "mesh-from-obj", "material": {"kind": "glossy", "albedo": [0.9, 0.9, 0.9], "glossy_exponent": 35.5},
     "mesh": {"obj": "part.obj"},
     "keyframes": [{"frame": 0, "translation": [0.1, 0.2, 0.3]},
                   {"frame": 6, "translation": [0.7, 0.2, -0.3], "rotation": [0, 0.3826834, 0, 0.9238795], "scale": 1.25},
                   {"frame": 11, "translation": [1.3, 0.2, -0.9]}]},
    {"material": {"kind": "diffuse", "albedo": [0.2, 0.4, 0.6]},
     "mesh": {"vertices": [[0,0.1,0],[0.3,0.1,0],[0,0.1,0.3]], "faces": [[0,1,2]]}}
  ],
  "lights": [
    {"kind": "point", "flux": [10, 10, 10], "keyframes": [{"frame": 0, "translation": [0, 2.5, 0]}]},
    {"kind": "spot", "flux": [5, 4, 3], "cone_angle": 40,
     "keyframes": [{"frame": 0, "translation": [1, 2.5, 0], "rotation": [0.7071068, 0, 0, 0.7071068]}]},
    {"kind": "disc_area", "flux": [3, 3, 3], "radius": 0.3,
     "keyframes": [{"frame": 0, "translation": [-1, 2.9, 0]}, {"frame": 10, "translation": [1, 2.9, 0]}]},
    {"kind": "rect_area", "flux": [2, 2, 2], "half_extents": [0.4, 0.2],
     "keyframes": [{"frame": 0, "translation": [0, 2.95, 1]}]}
  ]
}"""


def test_scene_document_bit_identical(tmp_path):
    (tmp_path / "part.obj").write_text(OBJ_TEXT)
    ours, theirs = both(DOC, str(tmp_path))
    assert digest(ours.describe()) == digest(theirs.describe())
    assert np.array_equal(ours.bvh_permutation(), theirs.bvh_permutation())
    assert struct.pack("<f", ours.diagonal) == struct.pack("<f", theirs.diagonal)
    # the file path variant resolves the OBJ relative to the document
    (tmp_path / "scene.json").write_text(DOC)
    loaded = pr.Scene.load(str(tmp_path / "scene.json"))
    assert digest(loaded.describe()) == digest(theirs.describe())


def test_builtin_sources():
    for name in pr.builtin_scenes():
        a = pr.Scene.load("builtin:" + name)
        b = pr.Scene.load(name)
        r = ref.RefScene.builtin(name)
        assert digest(a.describe()) == digest(r.describe()) == digest(b.describe())


BAD_DOCS = [
    '{"objects": [], "lights": [], "camera": {"position": [0,0,0], "look_at": [0,0,1], "fov": 60, "resolution": [8,8]}, "extra": 1}',
    '{"objects": [{"material": {"kind": "metal", "albedo": [1,1,1]}, "mesh": {"vertices": [], "faces": []}}], "lights": [], "camera": {"position": [0,0,0], "look_at": [0,0,1], "fov": 60, "resolution": [8,8]}}',
    '{"objects": [{"material": {"kind": "diffuse", "albedo": [1,1]}, "mesh": {"vertices": [], "faces": []}}], "lights": [], "camera": {"position": [0,0,0], "look_at": [0,0,1], "fov": 60, "resolution": [8,8]}}',
    '{"objects": [{"material": {"kind": "diffuse", "albedo": [1,1,1]}, "mesh": {"vertices": [[0,0,0]], "faces": [[0,0,5]]}}], "lights": [], "camera": {"position": [0,0,0], "look_at": [0,0,1], "fov": 60, "resolution": [8,8]}}',
    '{"objects": [], "lights": [{"kind": "laser", "flux": [1,1,1]}], "camera": {"position": [0,0,0], "look_at": [0,0,1], "fov": 60, "resolution": [8,8]}}',
    '{"objects": [], "lights": [], "camera": {"position": [0,0,0], "look_at": [0,0,1], "fov": 60, "resolution": [8]}}',
    '{"objects": [', '[1, 2', '{"a": tru}',
    # finalize_scene rejections (no objects / no lights)
    '{"objects": [], "lights": [], "camera": {"position": [0,0,0], "look_at": [0,0,1], "fov": 60, "resolution": [8,8]}}',
]


@pytest.mark.parametrize("doc", BAD_DOCS)
def test_scene_document_errors_match(doc):
    with pytest.raises(L.SceneError):
        ref.RefScene.from_text(doc)
    with pytest.raises(L.SceneError):
        pr.Scene.from_text(doc)


def test_obj_errors_match(tmp_path):
    cases = {"comment.obj": "#nospace\nv 0 0 0\n", "vn.obj": "v 0 0 0\nvn 0 1 0\n",
             "short.obj": "v 0 0 0\nv 1 0 0\nf 1 2\n", "range.obj": "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 9\n",
             "empty.obj": "v 0 0 0\n", "badv.obj": "v 0 x 0\n"}
    for name, text in cases.items():
        (tmp_path / name).write_text(text)
        doc = DOC.replace("part.obj", name)
        with pytest.raises(L.SceneError):
            ref.RefScene.from_text(doc, str(tmp_path))
        with pytest.raises(L.SceneError):
            pr.Scene.from_text(doc, str(tmp_path))
    with pytest.raises(L.SceneError):  # missing mesh file
        pr.Scene.from_text(DOC, str(tmp_path / "nowhere"))


def _rows():
    rng = np.random.default_rng(3)
    rows = []
    for mode in (0, 1, 2):
        for f in range(3):
            s = L.FrameStats()
            s.frame, s.mode = f, mode
            for k in L.FrameStats.COUNTS:
                setattr(s, k, int(rng.integers(0, 10**7)))
            for k in ("t_update", "t_occlusion", "t_dm", "t_prune", "t_fill", "t_trace", "t_gather"):
                setattr(s, k, float(rng.random() * 10.0 ** float(rng.integers(-9, 2))))
            rows.append(s)
    return rows


def test_stats_csv_and_report_byte_identical(tmp_path):
    rows = _rows()
    pr.write_stats_csv(rows, str(tmp_path / "ours.csv"))
    ref.write_stats_csv(rows, str(tmp_path / "ref.csv"))
    assert (tmp_path / "ours.csv").read_bytes() == (tmp_path / "ref.csv").read_bytes()
    back = pr.read_stats_csv(str(tmp_path / "ref.csv"))
    assert [(r.frame, r.mode, r.rays_traced) for r in back] == [(r.frame, r.mode, r.rays_traced) for r in rows]
    assert pr.reuse_report(rows) == ref.reuse_report(rows)
    with pytest.raises(L.PrxError):  # no baseline rows
        pr.reuse_report([r for r in rows if r.mode != 0])
    (tmp_path / "bad.csv").write_text("frame,mode\n")
    with pytest.raises(L.PrxError):
        pr.read_stats_csv(str(tmp_path / "bad.csv"))


def test_ppm_byte_identical(tmp_path):
    rng = np.random.default_rng(7)
    img = (rng.random((9, 13, 3)) * 1.4 - 0.2).astype(np.float32)
    img[0, 0] = [np.nan, np.inf, -np.inf]
    pr.write_image(img, str(tmp_path / "ours.ppm"))
    ref.write_image(img, str(tmp_path / "ref.ppm"))
    assert (tmp_path / "ours.ppm").read_bytes() == (tmp_path / "ref.ppm").read_bytes()
    assert pr.frame_image_name(3) == "frame_0003.ppm"


def test_photon_dump_byte_identical(tmp_path):
    scene = ref.RefScene.builtin("moving-cube")
    eng = ref.RefEngine(scene, pr.make_config("naive", paths=500, bounces=4, dm=[2, 2, 4, 4]))
    eng.run_frame()
    eng.write_photon_dump(str(tmp_path / "ref.phm"))
    photons = eng.download("photons")
    pr.write_photon_dump(photons, 500, 4, str(tmp_path / "ours.phm"))
    assert (tmp_path / "ours.phm").read_bytes() == (tmp_path / "ref.phm").read_bytes()
    n, b, back = pr.read_photon_dump(str(tmp_path / "ref.phm"))
    assert (n, b) == (500, 4) and back.tobytes() == photons.tobytes()
    (tmp_path / "trunc.phm").write_bytes((tmp_path / "ref.phm").read_bytes()[:100])
    with pytest.raises(L.PrxError):
        pr.read_photon_dump(str(tmp_path / "trunc.phm"))
    (tmp_path / "magic.phm").write_bytes(b"XXXX" + bytes(12))
    with pytest.raises(L.PrxError):
        pr.read_photon_dump(str(tmp_path / "magic.phm"))


def test_oracle_synthetic_scenes_identical():
    """The reference arm builds C1-C4 from the generators compiled into the oracle library
    (oracle/scene_gen.cpp): the same description bit for bit as the product's."""
    for name in ("C1", "C2", "C3", "C4"):
        a, b = ref.RefScene.synthetic(name), pr.Scene.synthetic(name)
        assert digest(a.describe()) == digest(b.describe()), name
        assert np.array_equal(a.bvh_permutation(), b.bvh_permutation()), name


def test_reference_arm_loads_only_the_oracle():
    """bench.py --impl reference runs without loading the product library."""
    import subprocess
    import sys

    code = ("import sys, json; sys.argv=['bench.py']; import bench; "
            "v, d = bench.run_reference(None, 'C1', 2000, 1, 0); "
            "maps = open('/proc/self/maps').read(); "
            "print(json.dumps({'prx': '_prx.so' in maps, 'ref': 'libpathreuse_ref.so' in maps, 'v': v}))")
    import json
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, check=True)
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["ref"] and not res["prx"] and res["v"] > 0
