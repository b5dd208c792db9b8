"""The product's sharded prune/fill kernels on the GPU: 2 and 3 path shards of one
problem, driven in-process through the exchange protocol (distributed.run_frame_loopback),
must reproduce the single-engine frame bit for bit (counters and every state field)."""
import numpy as np
import pytest

from paper_2111_06906_b200 import pathreuse as pr
from paper_2111_06906_b200.distributed import GpuExecutor, run_frame_loopback, shard_range

FIELDS = ("photons", "path_info", "meta", "cell", "epoch", "origin", "emission_dir", "canonical")


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("scene,mode", [("moving-cube", "error"), ("parallel-spot", "naive"),
                                        ("villa-analog", "naive"), ("moving-cube", "baseline")])
def test_shards_match_single_engine(world, scene, mode):
    cfg = dict(mode=mode, paths=6001, bounces=6, dm=[2, 2, 8, 8], seed=7)
    sc = pr.Scene.builtin(scene)
    single = pr.Engine(sc, pr.make_config(**cfg))
    exs = [GpuExecutor(sc, pr.make_config(shard=shard_range(cfg["paths"], r, world), **cfg)) for r in range(world)]
    B, N = cfg["bounces"], cfg["paths"]
    for f in range(5):
        st = single.run_frame()
        got = run_frame_loopback(exs, f)
        for k in ("rays_traced", "rays_reused", "paths_replaced", "paths_pruned", "paths_filled", "visibility_rays"):
            assert got[k] == getattr(st, k), (f, k)
        for fld in FIELDS:
            ref = single.download(fld)
            parts = [ex.engine.download(fld) for ex in exs]
            if fld == "photons":
                cat = np.concatenate([p.reshape(B, -1) for p in parts], axis=1)
                ref = ref.reshape(B, N)
            else:
                cat = np.concatenate(parts, axis=0)
            assert cat.tobytes() == ref.tobytes(), (f, fld)
        for li in range(exs[0].n_lights):
            for ex in exs:
                assert np.array_equal(ex.engine.download("dm_current", li), single.download("dm_current", li))
