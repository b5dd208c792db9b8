"""Splat-stage timings per workload, mode (0 atomic, 1 ordered) and pixel-grouping policy.

usage: python profiles/splat_modes.py [C1 C2 C3 C4 ...]
For each workload: 6 frames, then the splat at the scene camera (120x90) and at 1920x1080,
PRX_GATHER_GROUPS=0/1/auto, median device ms of 5 (the engine's own CUDA events).
"""
import os
import statistics
import sys

sys.path.insert(0, __file__.rsplit("/profiles/", 1)[0])
import bench  # noqa: E402
from paper_2111_06906_b200 import _lib as L  # noqa: E402
from paper_2111_06906_b200 import pathreuse as pr  # noqa: E402


def main(names):
    for name in names:
        w = bench.WORKLOADS[name]
        scene = pr.Scene.synthetic(name)
        eng = pr.Engine(scene, pr.make_config(mode=w["mode"], paths=w["paths"], bounces=w["bounces"],
                                              dm=[8, 8, 64, 64], threshold=w["threshold"], seed=1))
        for _ in range(6):
            eng.run_frame()
        cam = scene.describe().camera
        for wpx, hpx in ((cam.width, cam.height), (1920, 1080)):
            c = L.Camera(cam.position, cam.look_at, cam.fov_deg, wpx, hpx)
            row = []
            for groups in ("0", "1", None):
                if groups is None:
                    os.environ.pop("PRX_GATHER_GROUPS", None)
                else:
                    os.environ["PRX_GATHER_GROUPS"] = groups
                for mode in (1, 0):
                    ts = []
                    for _ in range(6):
                        st = L.FrameStats()
                        eng.splat(camera=c, radius=0.25, mode=mode, st=st)
                        ts.append(st.ms_splat)
                    row.append(f"groups={groups or 'auto'} mode={mode}: {statistics.median(ts[1:]):.3f}")
            print(f"{name} {wpx}x{hpx} | " + " | ".join(row), flush=True)
        eng.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3", "C4"])
