"""One C4 frame, then splats at 1920x1080 (for a launch-list profile of the splat kernels)."""
import sys

sys.path.insert(0, __file__.rsplit("/profiles/", 1)[0])
from paper_2111_06906_b200 import _lib as L  # noqa: E402
from paper_2111_06906_b200 import pathreuse as pr  # noqa: E402

scene = pr.Scene.synthetic("C4")
eng = pr.Engine(scene, pr.make_config(mode="error", paths=5_000_000, bounces=7, dm=[8, 8, 64, 64], seed=1))
for _ in range(2):
    eng.run_frame()
cam = scene.describe().camera
c = L.Camera(cam.position, cam.look_at, cam.fov_deg, 1920, 1080)
for _ in range(2):
    st = L.FrameStats()
    eng.splat(camera=c, radius=0.25, mode=1, st=st)
    print("splat 1920x1080 ms", st.ms_splat)
