"""run_frame replays a frame whose host decisions repeat the previous frame's as one CUDA
graph (engine.cpp: run_frame / capture_graph). The graph path must give the same state,
counters and stage timings as plain stream launches, frame after frame, including frames
whose shape changes (first frame, static frames, moving lights or not)."""
import numpy as np
import pytest

from paper_2111_06906_b200 import pathreuse as pr
from tests.helpers import counts


def engine(monkeypatch, graphs, scene, synthetic, **cfg):
    monkeypatch.setenv("PRX_GRAPHS", "1" if graphs else "0")
    sc = pr.Scene.synthetic(scene) if synthetic else pr.Scene.builtin(scene)
    return pr.Engine(sc, pr.make_config(**cfg))


@pytest.mark.gpu
@pytest.mark.parametrize("scene,synthetic,mode", [("moving-cube", False, "error"), ("parallel-spot", False, "naive"),
                                                   ("static-box", False, "error"), ("C3", True, "error"),
                                                   ("merry-go-round-analog", False, "baseline")])
def test_graph_replay_matches_plain_launches(monkeypatch, scene, synthetic, mode):
    cfg = dict(mode=mode, paths=20_000, bounces=6, dm=[4, 4, 16, 16], threshold=0.001, seed=5)
    plain = engine(monkeypatch, False, scene, synthetic, **cfg)
    graph = engine(monkeypatch, True, scene, synthetic, **cfg)
    for f in range(6):
        sp, sg = plain.run_frame(), graph.run_frame()
        assert counts(sp) == counts(sg), f
        assert plain.photon_map().tobytes() == graph.photon_map().tobytes(), f
        for field in ("meta", "path_info", "cell", "epoch", "retrace_start"):
            assert np.array_equal(plain.download(field), graph.download(field)), (f, field)
        if f >= 1:  # stage timings come from event nodes inside the replayed graph
            assert sg.ms_retrace > 0.0 and sg.t_trace > 0.0, f
    assert plain.splat(radius=0.25).tobytes() == graph.splat(radius=0.25).tobytes()
