"""World-size-2 gloo test of the multi-GPU exchange protocol on CPU.

Each rank drives one path shard of the C oracle through the product's protocol code
(paper_2111_06906_b200/distributed.py: DM_C all-reduce, prune-count all-gather with
prefix/total, dead-slot all-gather, counter all-reduce).  The concatenated shard states and
the reduced counters must equal a single-engine run bit for bit."""
import os
import pickle
import socket
import tempfile

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port
from paper_2111_06906_b200 import pathreuse as pr
from paper_2111_06906_b200.distributed import TorchCollectives, run_frame_distributed, shard_range

FIELDS = ("photons", "path_info", "meta", "cell", "epoch", "origin", "emission_dir", "canonical")
SLICED = {"photons": True}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port_no, case, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    scene_name, cfg, frames = case
    sc = pr.Scene.builtin(scene_name)
    sb, se = shard_range(cfg["paths"], rank, world)
    ex = port.PortShardExecutor(port.PortScene(sc.describe()), pr.make_config(shard=(sb, se), **cfg))
    coll = TorchCollectives()
    stats = [run_frame_distributed(ex, coll, f) for f in range(frames)]
    state = {}
    B = cfg["bounces"]
    N = cfg["paths"]
    for f in FIELDS:
        a = ex.engine.download(f)
        if f == "photons":
            a = a.reshape(B, N)[:, sb:se]
        else:
            a = a[sb:se]
        state[f] = a
    dms = [ex.engine.download("dm_current", li) for li in range(ex.n_lights)]
    with open(os.path.join(out_dir, f"rank{rank}.pkl"), "wb") as fh:
        pickle.dump({"stats": stats, "state": state, "dm": dms}, fh)
    dist.destroy_process_group()


CASES = [
    ("moving-cube", dict(mode="error", paths=3001, bounces=6, dm=[2, 2, 8, 8], seed=3), 5),
    ("parallel-spot", dict(mode="naive", paths=4000, bounces=5, dm=[1, 1, 8, 8], seed=11), 6),
    ("villa-analog", dict(mode="naive", paths=3000, bounces=6, dm=[4, 4, 8, 8], seed=1), 4),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] + "-" + c[1]["mode"] for c in CASES])
def test_two_rank_gloo_matches_single_engine(case):
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), case, d), nprocs=world, join=True)
        parts = [pickle.load(open(os.path.join(d, f"rank{r}.pkl"), "rb")) for r in range(world)]
    scene_name, cfg, frames = case
    sc = pr.Scene.builtin(scene_name)
    single = port.PortEngine(port.PortScene(sc.describe()), pr.make_config(**cfg))
    B, N = cfg["bounces"], cfg["paths"]
    for f in range(frames):
        st = single.run_frame()
        got = parts[0]["stats"][f]
        assert parts[1]["stats"][f] == got  # every rank sees the reduced counters
        for k in ("rays_traced", "rays_reused", "paths_replaced", "paths_pruned", "paths_filled",
                  "visibility_rays"):
            assert got[k] == getattr(st, k), (f, k, got[k], getattr(st, k))
    for fld in FIELDS:
        a = single.download(fld)
        cat = np.concatenate([p["state"][fld] for p in parts], axis=1 if fld == "photons" else 0)
        ref = a.reshape(B, N) if fld == "photons" else a
        assert cat.tobytes() == ref.tobytes(), fld
    for li, dm in enumerate(parts[0]["dm"]):
        assert np.array_equal(dm, single.download("dm_current", li))
        assert np.array_equal(parts[1]["dm"][li], dm)
