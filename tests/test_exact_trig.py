"""csrc/exact_trig.h (host build) against the host libm -- glibc, the reference's libm for
light.cpp:40-175.  The double-double sin/cos/atan2 are correctly rounded (checked with
mpmath at 200 bits on every disagreement); glibc agrees with them except for its own
misrounded results (~0.1%, glibc's bound is < 1 ulp, not correct rounding).  The device uses
them only when the +-2^-50 window around CUDA's value narrows to two different floats."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2111_06906_b200", "csrc")
mpmath = pytest.importorskip("mpmath")


@pytest.fixture(scope="module")
def run(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("xt") / "exact_trig_check")
    subprocess.check_call(["g++", "-std=c++20", "-O2", f"-I{CSRC}", os.path.join(ROOT, "tests", "cpp",
                                                                                 "exact_trig_check.cpp"), "-o", exe])
    out = subprocess.check_output([exe, "200000", "7"], text=True)
    rows = {}
    ex = []
    for line in out.splitlines():
        k, *v = line.split()
        if k == "example":
            ex.append(v)
        else:
            rows[k] = [int(x) for x in v]
    return rows, ex


def test_disagreements_are_glibc_misroundings(run):
    rows, examples = run
    mpmath.mp.prec = 200
    assert examples, "expected a few glibc misroundings in 200K samples"
    for kind, a, b, glibc, ours in examples:
        a, b = float.fromhex(a), float.fromhex(b)
        g, o = float.fromhex(glibc), float.fromhex(ours)
        if kind == "sin":
            true = mpmath.sin(mpmath.mpf(a))
        elif kind == "cos":
            true = mpmath.cos(mpmath.mpf(a))
        else:
            true = mpmath.atan2(mpmath.mpf(a), mpmath.mpf(b))
        ulp = abs(mpmath.mpf(g) - mpmath.mpf(o))
        assert abs(true - mpmath.mpf(o)) <= ulp / 2, (kind, a, b)   # ours: correctly rounded
        assert abs(true - mpmath.mpf(g)) >= ulp / 2, (kind, a, b)   # glibc: the misrounded one


def test_disagreement_rates_small(run):
    rows, _ = run
    for key in ("sincos", "sincos_any"):
        n, ms, mc = rows[key]
        assert ms / n < 5e-3 and mc / n < 5e-3, rows[key]
    n, ma = rows["atan2"]
    assert ma / n < 5e-3
