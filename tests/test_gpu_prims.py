"""The device primitives the engine's prune, fill, trace and splat stages are built on
(csrc/prims.cu: stable LSD radix sort, stable compaction, exclusive scan), checked directly
against host std::stable_sort / loops on random inputs whose live counts sit in device
memory below the buffer capacity (tests/cpp/prims_check.cu)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2111_06906_b200", "csrc")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("prims") / "prims_check")
    subprocess.check_call(["nvcc", "-std=c++17", "-O2", "-gencode", "arch=compute_100a,code=sm_100a",
                           f"-I{CSRC}", "-o", out, os.path.join(ROOT, "tests", "cpp", "prims_check.cu"),
                           os.path.join(CSRC, "prims.cu")])
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("radix10", ["1", "0"])
@pytest.mark.parametrize("seed", [1, 2])
def test_prims_random(exe, seed, radix10):
    """radix10: 8-bit digits throughout (default) or 10-bit digits where they save a pass"""
    env = dict(os.environ, PRX_RADIX10=radix10)
    r = subprocess.run([exe, str(seed)], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr
