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


@pytest.mark.gpu
def test_multi_gpu_engine_matches_single_engine():
    """MultiGpuEngine over all visible devices (shards share the device when there is one)."""
    import torch

    from paper_2111_06906_b200.distributed import MultiGpuEngine

    devices = list(range(torch.cuda.device_count()))
    if len(devices) < 2:
        devices = [0, 0]
    cfg = dict(mode="error", paths=5003, bounces=5, dm=[2, 2, 8, 8], seed=9)
    sc = pr.Scene.builtin("moving-cube")
    single = pr.Engine(sc, pr.make_config(**cfg))
    multi = MultiGpuEngine(sc, devices=devices, **cfg)
    for f in range(4):
        st = single.run_frame()
        got = multi.run_frame()
        for k in ("rays_traced", "rays_reused", "paths_replaced", "paths_pruned", "paths_filled", "visibility_rays"):
            assert got[k] == getattr(st, k), (f, k)
    img_single = single.splat(radius=0.25)
    img_multi = multi.splat(radius=0.25)
    assert np.allclose(img_multi, img_single, rtol=1e-4, atol=0)  # shard sums reorder the fp32 adds
    assert np.array_equal(img_multi == 0, img_single == 0)


# ---- in-engine sharded frames (collectives enqueued by the engine itself, comm.cpp)
GROUP_CASES = [(w, sc) for w in (2, 3) for sc in (("moving-cube", "error", False), ("parallel-spot", "naive", False),
                                                  ("villa-analog", "naive", False), ("moving-cube", "baseline", False),
                                                  ("C4", "error", True))]
# Class A/B outputs bitwise identical for G in {1, 2, 4, 8}
GROUP_CASES += [(w, sc) for w in (4, 8) for sc in (("villa-analog", "error", False), ("C4", "error", True))]


@pytest.mark.gpu
@pytest.mark.parametrize("world,case", GROUP_CASES, ids=[f"{w}-{c[0]}-{c[1]}" for w, c in GROUP_CASES])
def test_engine_group_matches_single_engine(world, case):
    scene, mode, synthetic = case
    from paper_2111_06906_b200.distributed import EngineGroup

    cfg = dict(mode=mode, paths=6001, bounces=6, dm=[2, 2, 8, 8], seed=7)
    sc = pr.Scene.synthetic(scene) if synthetic else pr.Scene.builtin(scene)
    single = pr.Engine(sc, pr.make_config(**cfg))
    group = EngineGroup(sc, [0] * world, **cfg)
    B, N = cfg["bounces"], cfg["paths"]
    for f in range(4):
        st = single.run_frame()
        got = group.run_frame()
        for k in ("rays_traced", "rays_reused", "paths_replaced", "paths_pruned", "paths_filled", "visibility_rays",
                  "live_segments_before", "paths_retraced"):
            assert getattr(got, k) == getattr(st, k), (f, k)
        for fld in FIELDS:
            ref = single.download(fld)
            parts = [e.download(fld) for e in group.engines]
            if fld == "photons":
                cat = np.concatenate([p.reshape(B, -1) for p in parts], axis=1)
                ref = ref.reshape(B, N)
            else:
                cat = np.concatenate(parts, axis=0)
            assert cat.tobytes() == ref.tobytes(), (f, fld)
        for li in range(single.info().n_lights):
            for e in group.engines:
                assert np.array_equal(e.download("dm_current", li), single.download("dm_current", li))
    img_g, img_s = group.splat(radius=0.25), single.splat(radius=0.25)
    assert np.array_equal(img_g == 0, img_s == 0)
    assert np.allclose(img_g, img_s, rtol=1e-5, atol=0)  # per-shard sums, then the rank sum
    for _ in range(2):  # frames whose side streams precompute the splat prefix on every rank
        single.run_frame()
        group.run_frame()
    img_g, img_s = group.splat(radius=0.25), single.splat(radius=0.25)
    assert np.array_equal(img_g == 0, img_s == 0)
    assert np.allclose(img_g, img_s, rtol=1e-5, atol=0)
    group.close()


@pytest.mark.gpu
@pytest.mark.parametrize("backend", ["nccl", "local"])
def test_world1_collectives_bit_exact(backend):
    """One rank with a collectives table runs every exchange (identity sums): through NCCL
    (libnccl loaded at run time) and the local backend the frames and the image are the
    unsharded engine's, bit for bit."""
    from paper_2111_06906_b200.distributed import Communicator, attach

    cfg = dict(mode="error", paths=8000, bounces=5, dm=[2, 2, 8, 8], seed=5)
    sc = pr.Scene.builtin("villa-analog")
    single = pr.Engine(sc, pr.make_config(**cfg))
    eng = pr.Engine(sc, pr.make_config(**cfg))
    comm = (Communicator.nccl(Communicator.nccl_unique_id(), 0, 1, 0) if backend == "nccl"
            else Communicator.local_group(1)[0])
    attach(eng, comm)
    for f in range(4):
        a, b = eng.run_frame(), single.run_frame()
        for k in ("rays_traced", "rays_reused", "paths_pruned", "paths_filled", "visibility_rays"):
            assert getattr(a, k) == getattr(b, k), (f, k)
    assert eng.download("photons").tobytes() == single.download("photons").tobytes()
    assert eng.splat(radius=0.25).tobytes() == single.splat(radius=0.25).tobytes()
