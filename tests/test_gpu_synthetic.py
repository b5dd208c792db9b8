"""GPU engine vs the reference on the BASELINE workloads' own scenes at
reduced path counts: C1 (point light, moving 992-tri sphere), C2 (moving rect area light,
DM remap), C3 (282K static + 4 x 20K dynamic tris, error mode), C4 (1M static + 8 x 20K
dynamic, two moving lights).  Bit-exact per-frame counters and full state."""
import pytest

from tests.helpers import compare_state, counts, pair

CASES = [
    ("C1", dict(mode="naive", paths=8192, bounces=3, dm=[8, 8, 64, 64], threshold=0.001), 4),
    ("C2", dict(mode="naive", paths=16384, bounces=5, dm=[8, 8, 64, 64], threshold=0.001), 4),
    ("C2", dict(mode="error", paths=8192, bounces=5, dm=[4, 4, 16, 16], threshold=0.01), 3),
    ("C3", dict(mode="error", paths=2048, bounces=7, dm=[8, 8, 64, 64], threshold=0.01), 3),
    ("C4", dict(mode="error", paths=2048, bounces=7, dm=[8, 8, 64, 64], threshold=0.001), 3),
    ("C4", dict(mode="baseline", paths=1024, bounces=7, dm=[8, 8, 64, 64], threshold=0.001), 2),
]


@pytest.mark.gpu
@pytest.mark.parametrize("name,cfg,frames", CASES, ids=[f"{c[0]}-{c[1]['mode']}" for c in CASES])
def test_synthetic_bit_exact(name, cfg, frames):
    gpu, cpu = pair(name, synthetic=True, seed=1, **cfg)
    n_lights = gpu.info().n_lights
    for f in range(frames):
        sg, sc = gpu.run_frame(), cpu.run_frame()
        assert counts(sg) == counts(sc), f"frame {f}: gpu {counts(sg)} ref {counts(sc)}"
        bad = compare_state(gpu, cpu, n_lights)
        assert all(v == 0 for v in bad.values()), f"frame {f}: {bad}"


@pytest.mark.gpu
@pytest.mark.parametrize("dfs", [False, True])
def test_traversal_modes_agree(dfs):
    # the fast certified traversal and the reference-order DFS give identical frames
    gpu, cpu = pair("C3", synthetic=True, seed=2, mode="error", paths=3000, bounces=7,
                    dm=[8, 8, 64, 64], threshold=0.01, dfs_traversal=dfs)
    for f in range(3):
        assert counts(gpu.run_frame()) == counts(cpu.run_frame())
    assert gpu.download("photons").tobytes() == cpu.download("photons").tobytes()
