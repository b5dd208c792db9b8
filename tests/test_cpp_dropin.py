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
