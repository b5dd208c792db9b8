"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference engine (oracle/_ref/libpathreuse_ref.so, compiled from
/root/reference/proj by oracle/Makefile) on small builtin configurations and records the
per-frame FrameStats counters and SHA-256 digests of the full engine state, plus the
reference's own known-answer vectors.  Re-run after changing the case list:
    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2111_06906_b200 import pathreuse as pr  # noqa: E402

CASES = [
    ("static-box", "naive", 2000, 7, [1, 1, 8, 8], 11, 4),
    ("moving-cube", "naive", 3000, 7, [2, 2, 8, 8], 1, 5),
    ("moving-cube", "error", 3000, 7, [2, 2, 8, 8], 1, 5),
    ("moving-cube", "baseline", 2000, 5, [2, 2, 8, 8], 3, 3),
    ("parallel-spot", "naive", 3000, 6, [1, 1, 8, 8], 11, 5),
    ("merry-go-round-analog", "error", 3000, 7, [4, 4, 8, 8], 2, 4),
    ("armadillo-analog", "naive", 3000, 7, [4, 4, 8, 8], 1, 4),
    ("villa-analog", "error", 3000, 7, [4, 4, 8, 8], 1, 4),
]
STATE = ("photons", "path_info", "meta", "cell", "epoch", "origin", "emission_dir", "canonical",
         "retrace_start")
COUNTS = ("rays_traced", "rays_reused", "paths_replaced", "paths_pruned", "paths_filled",
          "visibility_rays")


def digest(eng, n_lights):
    h = hashlib.sha256()
    for f in STATE:
        h.update(eng.download(f).tobytes())
    for li in range(n_lights):
        h.update(eng.download("dm_current", li).tobytes())
        h.update(eng.download("dm_target", li).tobytes())
    return h.hexdigest()


def main():
    out = {"generator": "oracle/_ref (reference engine compiled from /root/reference/proj)",
           "state_fields": list(STATE), "cases": []}
    for scene, mode, paths, bounces, dm, seed, frames in CASES:
        cfg = pr.make_config(mode=mode, paths=paths, bounces=bounces, dm=dm, seed=seed, workers=1)
        eng = ref.RefEngine(ref.RefScene.builtin(scene), cfg)
        n_lights = eng.info().n_lights
        rows = []
        for _ in range(frames):
            st = eng.run_frame()
            rows.append({"counts": [getattr(st, k) for k in COUNTS], "state_sha256": digest(eng, n_lights)})
        img, _ = eng.gather(radius=0.25, workers=1)
        out["cases"].append({"scene": scene, "mode": mode, "paths": paths, "bounces": bounces, "dm": dm,
                             "seed": seed, "frames": rows,
                             "gather_sha256": hashlib.sha256(img.tobytes()).hexdigest()})
    # known-answer vectors of the reference's own tests
    out["kat"] = {
        "path_info_0x81800005": [5, 7, 0, False, True],           # test_photon_store.cpp:10-19
        "prune_probability": [[4, 2, 0.5], [7, 7, 0.0], [10, 0, 1.0], [0, 5, 0.0], [3, 9, 0.0]],
        "energies_close": [[[3, 4, 5], [3, 4, 5], 0.0, True],     # acceptance.cpp:74-76
                           [[100, 100, 100], [100.05, 100, 100], 0.001, True],
                           [[100, 100, 100], [101, 100, 100], 0.001, False]],
        "table1_mib": {"photon_map": 1068.0, "path_info": 19.07, "origin_positions": 57.22,
                       "distribution_maps": 8.00, "pruned_array": 19.07, "subtotal_reuse": 103.36},
        "select_paths_to_prune": [],
    }
    paths = list(range(1000))
    for seed, frame in [(5, 3), (1, 0), (7, 11)]:
        got = ref.select_paths_to_prune(paths, 1000, 600, seed, frame).tolist()
        out["kat"]["select_paths_to_prune"].append({"n": 1000, "dm_c": 1000, "dm_t": 600, "seed": seed,
                                                    "frame": frame, "pruned": got})
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_runs.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", len(out["cases"]), "cases")


if __name__ == "__main__":
    main()
