# Small C4 error-mode run for compute-sanitizer (memcheck / racecheck): python profiles/sanitize_run.py
import numpy as np
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.helpers import pair
gpu, cpu = pair("C4", synthetic=True, mode="error", paths=20000, bounces=5, dm=[2, 2, 8, 8], seed=3)
for f in range(4):
    gpu.run_frame(); cpu.run_frame()
    assert gpu.download("photons").tobytes() == cpu.download("photons").tobytes(), f
assert np.array_equal(gpu.splat(radius=0.25), cpu.gather(radius=0.25)[0])
print("sanitized run ok")
