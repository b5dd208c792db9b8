"""Secondary measurements of SURVEY.md s8d on one B200 (not bench lines; run on the GPU box):

  * C5 stress sweep: paths x dynamic objects, worst case EngineMode::Baseline (release all
    + full retrace, engine.cpp:228-232) and best case (a static frame: error mode with
    nothing moving, so occlusions early-exit);
  * frame 0 (cold fill) reported separately from steady-state frames;
  * the splat at 120x90 and at 1920x1080 (paper resolution), ordered gather.

Times are device times from the engine's CUDA events (FrameStats.ms_*), median over frames.
usage: python profiles/sweeps.py [--quick] > profiles/rNN_sweeps.md
"""
import argparse
import statistics
import sys
import time

sys.path.insert(0, __file__.rsplit("/profiles/", 1)[0])

from paper_2111_06906_b200 import _lib as L  # noqa: E402
from paper_2111_06906_b200 import pathreuse as pr  # noqa: E402


def frame_ms(st):
    return st.ms_frame_update + st.ms_verify + st.ms_retrace


def run(scene, mode, paths, frames=4, bounces=7):
    t0 = time.perf_counter()
    eng = pr.Engine(scene, pr.make_config(mode=mode, paths=paths, bounces=bounces, dm=[8, 8, 64, 64],
                                          threshold=0.001, seed=1))
    setup = time.perf_counter() - t0
    f0 = eng.run_frame()
    rest = [eng.run_frame() for _ in range(frames)]
    med = statistics.median(frame_ms(s) for s in rest)
    rays = statistics.median(s.rays_traced for s in rest)
    eng.close()
    return setup, frame_ms(f0), f0.rays_traced, med, rays


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    path_list = [1, 4, 16] if a.quick else [1, 2, 4, 8, 16, 32]
    dyn_list = [1, 16] if a.quick else [1, 4, 16, 64]
    print("# C5 sweep and splat resolutions (1 B200, device time)\n")
    print("Command: `python profiles/sweeps.py` on the GPU box. C5 = C4-like hall (~1.02M static tris) with "
          "n dynamic 20K-tri movers; 7 bounces; DM 8x8x64x64. Worst case = `baseline` mode (release all + "
          "full retrace every frame); best case = `error` mode on a frame where nothing moves is not available "
          "in a moving scene, so the best case is reported as the steady `error` frame.\n")
    print("| paths | movers | mode | engine setup s | frame 0 ms | frame 0 rays | steady frame ms | steady rays/frame |")
    print("|---:|---:|---|---:|---:|---:|---:|---:|")
    for nd in dyn_list:
        scene = pr.Scene.synthetic("C5", n_dynamic=nd)
        for p in path_list:
            for mode in ("baseline", "error"):
                try:
                    setup, f0, r0, med, rays = run(scene, mode, p * 1_000_000)
                    print(f"| {p}M | {nd} | {mode} | {setup:.2f} | {f0:.1f} | {r0} | {med:.2f} | {rays:.0f} |", flush=True)
                except Exception as exc:  # report, keep sweeping
                    print(f"| {p}M | {nd} | {mode} | failed: {type(exc).__name__}: {exc} | | | | |", flush=True)
    print("\n## Splat (ordered gather, bit-exact) at 120x90 and 1920x1080, C4 after 3 frames\n")
    print("| resolution | splat ms (median of 3) |")
    print("|---|---:|")
    scene = pr.Scene.synthetic("C4")
    eng = pr.Engine(scene, pr.make_config(mode="error", paths=5_000_000, bounces=7, dm=[8, 8, 64, 64], seed=1))
    for _ in range(3):
        eng.run_frame()
    cam = scene.describe().camera
    for w, h in ((120, 90), (1920, 1080)):
        c = L.Camera(cam.position, cam.look_at, cam.fov_deg, w, h)
        ts = []
        for _ in range(3):
            st = L.FrameStats()
            eng.splat(camera=c, radius=0.25, mode=1, st=st)
            ts.append(st.ms_splat)
        print(f"| {w}x{h} | {statistics.median(ts):.2f} |", flush=True)


if __name__ == "__main__":
    main()
