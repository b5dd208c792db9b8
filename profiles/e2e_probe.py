"""Host-API step time (run_frame + splat to a host image): the bench's e2e loop, split into
its calls, on torch's stream (as bench.py) and on the engine's own stream.
usage: python profiles/e2e_probe.py"""
import statistics
import sys
import time

sys.path.insert(0, __file__.rsplit("/profiles/", 1)[0])
import torch  # noqa: E402

from paper_2111_06906_b200 import pathreuse as pr  # noqa: E402

sc = pr.Scene.synthetic("C4")
for use_torch in (True, False, True):
    eng = pr.Engine(sc, pr.make_config(mode="error", paths=5_000_000, bounces=7, dm=[8, 8, 64, 64],
                                       threshold=0.001, seed=1))
    if use_torch:
        eng.set_stream(torch.cuda.current_stream().cuda_stream)
    for _ in range(4):
        eng.run_frame()
        eng.splat(radius=0.25)
    torch.cuda.synchronize()
    rf, sp = [], []
    t0 = time.perf_counter()
    for _ in range(10):
        a = time.perf_counter()
        st = eng.run_frame()
        b = time.perf_counter()
        eng.splat(radius=0.25)
        c = time.perf_counter()
        rf.append((b - a) * 1e3 - (st.ms_frame_update + st.ms_verify + st.ms_retrace))
        sp.append((c - b) * 1e3)
    t1 = time.perf_counter()
    print("torch stream" if use_torch else "own stream", f"{(t1 - t0) * 100:.2f} ms/step;",
          f"run_frame host-minus-device {statistics.median(rf):.3f} ms, splat wall {statistics.median(sp):.3f} ms",
          flush=True)
    eng.close()
