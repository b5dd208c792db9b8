"""Shared helpers for the parity tests (tests only)."""
import numpy as np

from paper_2111_06906_b200 import pathreuse as pr


def pair(scene_name, synthetic=False, **cfg):
    """A GPU engine and a reference engine on the identical scene and config."""
    from oracle import ref

    scene = pr.Scene.synthetic(scene_name) if synthetic else pr.Scene.builtin(scene_name)
    config = pr.make_config(**cfg)
    gpu = pr.Engine(scene, config)
    rscene = ref.RefScene.from_desc(scene.describe()) if synthetic else ref.RefScene.builtin(scene_name)
    cpu = ref.RefEngine(rscene, pr.make_config(**cfg))
    cpu.set_workers(0)
    return gpu, cpu


def counts(st):
    return tuple(getattr(st, k) for k in ("rays_traced", "rays_reused", "paths_replaced",
                                          "paths_pruned", "paths_filled", "visibility_rays"))


def compare_state(gpu, cpu, n_lights, fields=("photons", "path_info", "meta", "cell", "epoch",
                                              "origin", "emission_dir", "canonical", "retrace_start")):
    """Return {field: number of mismatching entries} (0 everywhere = bit-exact)."""
    bad = {}
    for f in fields:
        a, b = gpu.download(f), cpu.download(f)
        if a.dtype.names:
            a = a.view(np.uint8).reshape(a.shape[0], -1)
            b = b.view(np.uint8).reshape(b.shape[0], -1)
        else:
            a = a.view(np.uint8).reshape(a.shape[0], -1) if a.ndim > 1 else a.view(np.uint8).reshape(a.shape[0], -1)
            b = b.view(np.uint8).reshape(b.shape[0], -1) if b.ndim > 1 else b.view(np.uint8).reshape(b.shape[0], -1)
        bad[f] = int(np.any(a != b, axis=1).sum())
    for li in range(n_lights):
        bad[f"dm_current{li}"] = int((gpu.download("dm_current", li) != cpu.download("dm_current", li)).sum())
        bad[f"dm_target{li}"] = int((gpu.download("dm_target", li) != cpu.download("dm_target", li)).sum())
    # live aux positions / outgoing (stale aux of empty records is not part of the contract)
    pa, pb = gpu.download("photons"), cpu.download("photons")
    live = pb["object_id"] != 0xFFFFFFFF
    xa, xb = gpu.download("aux"), cpu.download("aux")
    bad["aux_live"] = int(np.any(xa[live].view(np.uint8).reshape(-1, 24) != xb[live].view(np.uint8).reshape(-1, 24), axis=1).sum())
    return bad
