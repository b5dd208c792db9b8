"""Parity at the bench configuration (C4: 1.02M static + 8 x 20K dynamic tris, two moving
lights, error mode T=0.001, DM 8x8x64x64, 7 bounces) at bench-scale path counts, against the
compiled reference engine (oracle/_ref, `Engine::run_frame` engine.cpp:201-242 and
`gather_image` gather.cpp:35-75).

* `test_c4_1m_from_scratch`: 1,048,576 paths (the bench's CPU sample), frames 0-5 run on
  both engines from the same seed; every state field, the DMs, live aux and the image are
  compared every frame.
* `test_c4_5m_bench_frames`: the bench's own workload, 5,000,000 paths.  The GPU runs
  frames 0..k-1 alone; its full state is then injected into the reference (`copy_state`) and
  frame k runs on both -- so the bench's steady-state frames (k = 5 and 20: warm-up and timed
  region) are compared at full density (~19 paths per DM cell) without paying for k
  reference frames.

Per-frame mismatch counts are printed in the session's terminal summary
("scale parity" section, tests/conftest.py); the bar is zero everywhere.
"""
import time

import numpy as np
import pytest

from oracle import ref
from tests.conftest import report_parity
from tests.helpers import compare_state, counts, pair

C4 = dict(mode="error", bounces=7, dm=[8, 8, 64, 64], threshold=0.001, seed=1)


def _image_mismatch(gpu, cpu):
    img_g = gpu.splat(radius=0.25, mode=1)
    img_c, secs = cpu.gather(radius=0.25)
    return int(np.any(img_g != img_c, axis=-1).sum()), secs


@pytest.mark.gpu
def test_c4_1m_from_scratch():
    gpu, cpu = pair("C4", synthetic=True, paths=1 << 20, **C4)
    n_lights = gpu.info().n_lights
    failures = []
    for f in range(6):
        t0 = time.perf_counter()
        sc = cpu.run_frame()
        t_ref = time.perf_counter() - t0
        sg = gpu.run_frame()
        bad = compare_state(gpu, cpu, n_lights)
        bad["image_px"], _ = _image_mismatch(gpu, cpu)
        bad["counters"] = int(counts(sg) != counts(sc))
        report_parity(f"C4 1M frame {f}", dict(bad, ref_s=round(t_ref, 1),
                                               rays_traced=sg.rays_traced, vis_rays=sg.visibility_rays))
        if any(v for k, v in bad.items()):
            failures.append((f, bad))
    assert not failures, failures


@pytest.mark.gpu
@pytest.mark.parametrize("k", [5, 20])
def test_c4_5m_bench_frames(k):
    gpu, cpu = pair("C4", synthetic=True, paths=5_000_000, **C4)
    n_lights = gpu.info().n_lights
    for _ in range(k):
        gpu.run_frame()
    ref.copy_state(gpu, cpu, n_lights)
    cpu.set_frame_counter(k)
    t0 = time.perf_counter()
    sc = cpu.run_frame()
    t_ref = time.perf_counter() - t0
    sg = gpu.run_frame()
    bad = compare_state(gpu, cpu, n_lights)
    bad["image_px"], _ = _image_mismatch(gpu, cpu)
    bad["counters"] = int(counts(sg) != counts(sc))
    report_parity(f"C4 5M frame {k} (injected)", dict(bad, ref_s=round(t_ref, 1), rays_traced=sg.rays_traced,
                                                      vis_rays=sg.visibility_rays,
                                                      retraced=sg.paths_retraced))
    assert not any(bad.values()), bad


@pytest.mark.gpu
@pytest.mark.parametrize("name,cfg,k", [
    ("C2", dict(mode="naive", paths=1_048_576, bounces=5, dm=[8, 8, 64, 64], threshold=0.001, seed=1), 4),
    ("C3", dict(mode="error", paths=2_097_152, bounces=7, dm=[8, 8, 64, 64], threshold=0.01, seed=1), 4),
])
def test_full_size_injected_frame(name, cfg, k):
    """C2 and C3 at their BASELINE path counts: GPU frames 0..k-1, state injected into the
    reference, frame k on both -- every field, the DMs and the image bit-exact."""
    gpu, cpu = pair(name, synthetic=True, **cfg)
    n_lights = gpu.info().n_lights
    for _ in range(k):
        gpu.run_frame()
    ref.copy_state(gpu, cpu, n_lights)
    cpu.set_frame_counter(k)
    t0 = time.perf_counter()
    sc = cpu.run_frame()
    t_ref = time.perf_counter() - t0
    sg = gpu.run_frame()
    bad = compare_state(gpu, cpu, n_lights)
    bad["image_px"], _ = _image_mismatch(gpu, cpu)
    bad["counters"] = int(counts(sg) != counts(sc))
    report_parity(f"{name} {cfg['paths']} frame {k} (injected)",
                  dict(bad, ref_s=round(t_ref, 1), rays_traced=sg.rays_traced, retraced=sg.paths_retraced))
    assert not any(bad.values()), bad
