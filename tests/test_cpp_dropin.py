"""The source-compatible C++ surface (include/pathreuse_b200.hpp): a reference-style program
compiles against it (CPU) and, on the GPU, reproduces the reference engine's per-frame
counters while the reference's own engine invariants hold (test_engine.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_example.cpp")
LIBDIR = os.path.join(ROOT, "paper_2111_06906_b200")


def build(tmp_path):
    exe = os.path.join(str(tmp_path), "dropin_example")
    subprocess.check_call(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", SRC, f"-L{LIBDIR}", "-l:_prx.so",
                           f"-Wl,-rpath,{LIBDIR}", "-o", exe])
    return exe


def test_dropin_header_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
@pytest.mark.parametrize("scene,mode", [("moving-cube", "error"), ("parallel-spot", "naive")])
def test_dropin_program_matches_reference(tmp_path, scene, mode):
    from oracle import ref
    from paper_2111_06906_b200 import pathreuse as pr

    out = subprocess.run([build(tmp_path), scene, mode, "--check"], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    rows = [list(map(int, line.split())) for line in out.stdout.strip().splitlines()]
    eng = ref.RefEngine(ref.RefScene.builtin(scene),
                        pr.make_config(mode=mode, paths=5000, bounces=7, dm=[1, 1, 8, 8], seed=11))
    for row in rows:
        st = eng.run_frame()
        assert row == [st.frame, st.rays_traced, st.rays_reused, st.paths_replaced, st.paths_pruned,
                       st.paths_filled, st.visibility_rays]


REF_CALLS = os.path.join(ROOT, "tests", "cpp", "dropin_reference_calls.cpp")


def build_ref_calls(tmp_path):
    exe = os.path.join(str(tmp_path), "dropin_reference_calls")
    subprocess.check_call(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", REF_CALLS, f"-L{LIBDIR}", "-l:_prx.so",
                           f"-Wl,-rpath,{LIBDIR}", "-o", exe])
    return exe


def test_reference_call_patterns_compile(tmp_path):
    """gather_image(scene_state(), photon_map(), vertex_aux(), ...), segment_*, dm_layout,
    select_paths_to_prune: the reference's call sites compile against the drop-in header."""
    assert os.path.exists(build_ref_calls(tmp_path))


@pytest.mark.gpu
@pytest.mark.parametrize("scene,mode,frames", [("moving-cube", "error", 3), ("merry-go-round-analog", "naive", 3),
                                               ("villa-analog", "error", 2)])
def test_reference_call_patterns_match_reference(tmp_path, scene, mode, frames):
    import numpy as np

    from oracle import ref
    from paper_2111_06906_b200 import pathreuse as pr

    out = subprocess.run([build_ref_calls(tmp_path), scene, mode, str(frames)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    rows = {}
    for line in out.stdout.strip().splitlines():
        k, *v = line.split()
        rows.setdefault(k, []).append([int(x) for x in v])
    cfg = pr.make_config(mode=mode, paths=6000, bounces=5, dm=[1, 1, 8, 8], seed=7)
    rs = ref.RefScene.builtin(scene)
    eng = ref.RefEngine(rs, cfg)
    ref_rows = []
    for _ in range(frames):
        st = eng.run_frame()
        ref_rows.append([st.frame, st.rays_traced, st.rays_reused, st.paths_pruned, st.paths_filled,
                         st.visibility_rays])
    assert rows["group"] == ref_rows  # the 2-shard MultiGpuEngine: the reference's counters

    def fnv(b):
        h = 1469598103934665603
        for x in b:
            h = ((h ^ x) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
        return h

    img, _ = eng.gather(radius=0.25)
    assert rows["image"][0][0] == fnv(img.tobytes())          # byte-identical image
    assert rows["image_host"][0][0] == rows["image"][0][0]     # host-map path, same image
    meta = eng.download("meta")
    alive = meta[:, 2] == 1
    segs = int((meta[alive, 0].astype(np.int64) + meta[alive, 1].astype(np.int64)).sum())
    assert rows["segments"][0] == [segs, 0, 0]
    frame, n_dyn, n_tris, outside = rows["state"][0]
    desc = rs.describe()
    dyn = [desc.objects[i] for i in range(desc.n_objects)
           if any(desc.objects[i].keyframes[k].translation.x != desc.objects[i].keyframes[0].translation.x
                  or desc.objects[i].keyframes[k].translation.y != desc.objects[i].keyframes[0].translation.y
                  or desc.objects[i].keyframes[k].translation.z != desc.objects[i].keyframes[0].translation.z
                  or desc.objects[i].keyframes[k].rotation.w != desc.objects[i].keyframes[0].rotation.w
                  for k in range(desc.objects[i].n_keyframes))]
    assert frame == frames - 1 and n_dyn == len(dyn) and outside == 0
    assert n_tris == sum(o.n_triangles for o in dyn)
    for li, cells, size, t_total, c_total in rows["dm"]:
        assert size == cells == eng.download("dm_target", li).size
        assert t_total == int(eng.download("dm_target", li).sum())
        assert c_total == int(eng.download("dm_current", li).sum())
    want = ref.select_paths_to_prune(np.arange(100, 1100, dtype=np.uint32), 1000, 600, 5, 3)
    assert rows["prune"][0] == [len(want)] + [int(x) for x in want]
    assert rows["prune_exact"][0] == [0]
