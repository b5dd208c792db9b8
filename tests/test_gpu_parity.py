"""GPU engine vs the reference engine (oracle/_ref) on identical scenes and seeds.

Bit-exact contract (SURVEY.md s8c classes A/B with the exact-trig table): per-frame
counters, photon records, path info, DM_C/DM_T, epochs, cells and origins must be
identical after every frame.
"""
import pytest

from tests.helpers import compare_state, counts, pair

CASES = [
    ("static-box", "naive"), ("static-box", "error"), ("moving-cube", "naive"),
    ("moving-cube", "error"), ("moving-cube", "baseline"), ("parallel-spot", "naive"),
    ("parallel-spot", "error"), ("merry-go-round-analog", "naive"),
    ("merry-go-round-analog", "error"), ("armadillo-analog", "error"),
    ("villa-analog", "error"), ("villa-analog", "naive"),
]


@pytest.mark.gpu
@pytest.mark.parametrize("scene,mode", CASES)
def test_frames_bit_exact(scene, mode):
    gpu, cpu = pair(scene, mode=mode, paths=6000, bounces=7, dm=[2, 2, 8, 8], threshold=0.001, seed=11)
    n_lights = gpu.info().n_lights
    for f in range(6):
        sg, sc = gpu.run_frame(), cpu.run_frame()
        assert counts(sg) == counts(sc), f"frame {f}: gpu {counts(sg)} ref {counts(sc)}"
        bad = compare_state(gpu, cpu, n_lights)
        assert all(v == 0 for v in bad.values()), f"frame {f}: mismatches {bad}"
