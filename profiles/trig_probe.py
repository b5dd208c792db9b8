"""Cost of the exact-trig table lookup in the bounce sampler: C4 frames with the host-libm
table (bit-exact) vs device cosf/sinf (not bit-exact; timing only).
usage: python profiles/trig_probe.py"""
import statistics
import sys

sys.path.insert(0, __file__.rsplit("/profiles/", 1)[0])
from paper_2111_06906_b200 import pathreuse as pr  # noqa: E402

scene = pr.Scene.synthetic("C4")
for exact in (True, False, True, False):
    eng = pr.Engine(scene, pr.make_config(mode="error", paths=5_000_000, bounces=7, dm=[8, 8, 64, 64],
                                          threshold=0.001, seed=1, exact_trig=exact))
    for _ in range(3):
        eng.run_frame()
    st = [eng.run_frame() for _ in range(8)]
    print("table" if exact else "device sincos",
          "trace %.3f ms" % statistics.median(s.t_trace * 1e3 for s in st),
          "verify %.3f ms" % statistics.median(s.ms_verify for s in st), flush=True)
    eng.close()
