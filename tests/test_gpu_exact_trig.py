"""The light parametrisation's transcendentals (light.cpp:40-175) through the exact path.

PRX_XT_FORCE=1 makes every double sin/cos/atan2 of warp_canonical / canonical_of /
dir_from_angles take the double-double, correctly rounded evaluation (exact_trig.h) instead of
CUDA's libm + the checked narrowing.  Frames stay bit-identical to the reference: the exact
path is what the engine falls back to whenever a narrowing is not decided by CUDA's value."""
import pytest

from tests.helpers import compare_state, counts, pair


@pytest.mark.gpu
@pytest.mark.parametrize("name,synthetic,cfg", [
    ("villa-analog", False, dict(mode="error", paths=30000, bounces=5, dm=[4, 4, 16, 16], threshold=0.01)),
    ("parallel-spot", False, dict(mode="naive", paths=30000, bounces=4, dm=[4, 4, 16, 16])),
    ("C2", True, dict(mode="naive", paths=60000, bounces=5, dm=[8, 8, 64, 64])),
    ("C4", True, dict(mode="error", paths=60000, bounces=7, dm=[8, 8, 64, 64], threshold=0.001)),
])
def test_forced_exact_trig_bit_exact(monkeypatch, name, synthetic, cfg):
    monkeypatch.setenv("PRX_XT_FORCE", "1")
    gpu, cpu = pair(name, synthetic=synthetic, seed=3, **cfg)
    n_lights = gpu.info().n_lights
    for f in range(3):
        assert counts(gpu.run_frame()) == counts(cpu.run_frame()), f
        bad = compare_state(gpu, cpu, n_lights)
        assert all(v == 0 for v in bad.values()), (f, bad)
