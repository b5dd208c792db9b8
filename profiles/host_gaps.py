"""Host-side overhead per frame: wall time of run_frame / splat vs their device-timed stages.
usage: python profiles/host_gaps.py [C4]"""
import sys
import time

sys.path.insert(0, __file__.rsplit("/profiles/", 1)[0])
from paper_2111_06906_b200 import _lib as L  # noqa: E402
from paper_2111_06906_b200 import pathreuse as pr  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
scene = pr.Scene.synthetic(name)
eng = pr.Engine(scene, pr.make_config(mode="error", paths=5_000_000, bounces=7, dm=[8, 8, 64, 64], seed=1))
for _ in range(3):
    eng.run_frame()
    eng.splat(radius=0.25)
for _ in range(5):
    t0 = time.perf_counter()
    st = eng.run_frame()
    t1 = time.perf_counter()
    sst = L.FrameStats()
    eng.splat(radius=0.25, st=sst)
    t2 = time.perf_counter()
    dev = st.ms_frame_update + st.ms_verify + st.ms_retrace
    print(f"run_frame wall {1e3 * (t1 - t0):.2f} ms (device stages {dev:.2f}: update {st.ms_frame_update:.2f} "
          f"verify {st.ms_verify:.2f} retrace {st.ms_retrace:.2f}) | splat wall {1e3 * (t2 - t1):.2f} ms "
          f"(device {sst.ms_splat:.2f})")
