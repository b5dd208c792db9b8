"""The fast traversal's SAH trees stay within the device traversal stack (64 entries) on
adversarial inputs: fast_bvh.cpp caps the build depth at 48 and falls back to
centroid-median splits below it.  CPU only: the builder is host code, compiled here directly
(the GPU side of the same scene is tests/test_gpu_deep_bvh.py)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2111_06906_b200", "csrc")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("bvh") / "bvh_depth")
    subprocess.check_call(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", f"-I{CSRC}", "-I/usr/local/cuda/include",
                           os.path.join(ROOT, "tests", "cpp", "bvh_depth.cpp"), os.path.join(CSRC, "fast_bvh.cpp"),
                           os.path.join(CSRC, "host_scene.cpp"), "-o", out])
    return out


def depths(exe, args, env=None):
    return list(map(int, subprocess.check_output([exe] + args, env=dict(os.environ, **(env or {}))).split()))


@pytest.mark.parametrize("args", [["200", "1.5", "1e-3"], ["100", "2", "1e-3"], ["60", "16", "1e-3"], ["1", "2", "1"]])
def test_sah_depth_capped(exe, args):
    static_depth, dyn_depth, _ = depths(exe, args)
    assert 1 <= static_depth <= 48
    assert 0 <= dyn_depth and dyn_depth + 1 <= 63  # joint walk: parked static root + dynamic path


def test_chains_are_adversarial(exe):
    # without the cap the binned SAH peels the chains level by level past the 64-entry stack
    static_depth, dyn_depth, n = depths(exe, ["200", "1.5", "1e-3"], {"PRX_SAH_MAXDEPTH": "100000"})
    assert n == 600 and static_depth > 64
    assert dyn_depth == -1  # build_dyn_sah refuses a tree the traversal stack cannot hold
