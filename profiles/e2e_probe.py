"""Host-API step time (run_frame + splat to a host image) on the engine stream vs torch's stream.
usage: python profiles/e2e_probe.py"""
import sys, time
sys.path.insert(0, '/root/repo')
import torch
from paper_2111_06906_b200 import pathreuse as pr
sc = pr.Scene.synthetic("C4")
for use_torch in (False, True, False, True):
    eng = pr.Engine(sc, pr.make_config(mode="error", paths=5_000_000, bounces=7, dm=[8, 8, 64, 64], threshold=0.001, seed=1))
    if use_torch:
        eng.set_stream(torch.cuda.current_stream().cuda_stream)
    for _ in range(4):
        eng.run_frame(); eng.splat(radius=0.25)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        eng.run_frame(); eng.splat(radius=0.25)
    t1 = time.perf_counter()
    print("torch stream" if use_torch else "own stream", f"{(t1 - t0) * 100:.2f} ms/step")
    eng.close()
