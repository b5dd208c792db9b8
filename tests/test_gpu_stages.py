"""Stage-level parity with state injection: the reference's full state
after frame f-1 is uploaded into the GPU engine, then each stage of frame f runs on both
sides from identical inputs and the outputs are compared bit for bit -- so a mismatch is
pinned to one stage (update_origins, occlusions, compute_dm, prune, fill, trace)."""
import pytest

from oracle import ref
from tests.helpers import compare_state, pair

STAGES = ["update_origins", "occlusions", "compute_dm", "prune", "fill", "trace"]
KEY = {"update_origins": "visibility_rays", "occlusions": "visibility_rays", "compute_dm": "paths_replaced",
       "prune": "paths_pruned", "fill": "paths_filled", "trace": "rays_traced"}


@pytest.mark.gpu
@pytest.mark.parametrize("scene,mode,synthetic", [("moving-cube", "error", False), ("parallel-spot", "naive", False),
                                                  ("villa-analog", "error", False), ("C2", "naive", True),
                                                  ("C1", "naive", True)])
def test_stagewise_injection(scene, mode, synthetic):
    cfg = dict(mode=mode, paths=6000, bounces=6, dm=[4, 4, 16, 16], seed=5, record_flags=True)
    gpu, cpu = pair(scene, synthetic=synthetic, **cfg)
    n_lights = gpu.info().n_lights
    for _ in range(3):  # advance the reference only
        cpu.run_frame()
    ref.copy_state(cpu, gpu, n_lights)
    gpu.set_frame_counter(3)
    cpu.set_frame_counter(3)
    gpu.frame_update()
    sc = cpu.frame_update()  # the reference accumulates stage counters into one FrameStats
    for stage in STAGES:
        sg = gpu.run_stage(stage)
        sc = cpu.run_stage(stage, sc)
        assert getattr(sg, KEY[stage]) == getattr(sc, KEY[stage]), stage
        fields = ("photons", "path_info", "meta", "cell", "epoch", "origin", "emission_dir", "canonical",
                  "retrace_start", "segment_flags")
        bad = compare_state(gpu, cpu, n_lights, fields=fields)
        assert all(v == 0 for v in bad.values()), f"after {stage}: {bad}"
