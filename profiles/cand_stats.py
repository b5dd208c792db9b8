import sys, numpy as np
sys.path.insert(0, '.')
from paper_2111_06906_b200 import pathreuse as pr
from paper_2111_06906_b200 import _lib as L
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
import bench
w = bench.WORKLOADS[name]
sc = pr.Scene.synthetic(name)
eng = pr.Engine(sc, pr.make_config(mode=w["mode"], paths=w["paths"], bounces=w["bounces"], dm=[8,8,64,64], threshold=w["threshold"], seed=1))
for _ in range(6): eng.run_frame()
cam = sc.describe().camera
W, H = cam.width, cam.height
def v(a): return np.array([a.x, a.y, a.z], dtype=np.float32)
pos, at = v(cam.position), v(cam.look_at)
fwd = at - pos; fwd = fwd / np.linalg.norm(fwd)
up = np.array([0,1,0], np.float32)
if abs(fwd @ up) > 0.999: up = np.array([1,0,0], np.float32)
right = np.cross(fwd, up); right /= np.linalg.norm(right); upv = np.cross(right, fwd)
th = np.tan(cam.fov_deg * np.pi / 360); asp = W / H
px, py = np.meshgrid(np.arange(W), np.arange(H))
sx = (2 * (px + 0.5) / W - 1) * th * asp; sy = (1 - 2 * (py + 0.5) / H) * th
d = fwd[None, None] + right[None, None] * sx[..., None] + upv[None, None] * sy[..., None]
d = (d / np.linalg.norm(d, axis=-1, keepdims=True)).reshape(-1, 3).astype(np.float32)
rays = np.zeros((len(d), 8), np.float32); rays[:, :3] = pos; rays[:, 3:6] = d; rays[:, 7] = 3.4e38
hits = eng.intersect(rays)
obj = hits[:, 1].view(np.uint32); ok = obj != 0xFFFFFFFF
hp = hits[ok, 3:6]; ho = obj[ok]
r = 0.25
cells = np.floor(hp / r).astype(np.int64)
# registered cells with object sets and AABBs
from collections import defaultdict
reg = defaultdict(lambda: [set(), np.full(3, np.inf), np.full(3, -np.inf)])
for c, o, p in zip(cells, ho, hp):
    for dz in (-1,0,1):
        for dy in (-1,0,1):
            for dx in (-1,0,1):
                e = reg[(c[0]+dx, c[1]+dy, c[2]+dz)]
                e[0].add(int(o)); e[1] = np.minimum(e[1], p); e[2] = np.maximum(e[2], p)
ph = eng.download("pos_obj").reshape(-1, 4)
pobj = ph[:, 3].view(np.uint32); live = pobj != 0xFFFFFFFF
pp = ph[live, :3]; po = pobj[live]
pc = np.floor(pp / r).astype(np.int64)
keys = list(reg.keys())
idx = {k: i for i, k in enumerate(keys)}
objsets = [reg[k][0] for k in keys]
lo = np.array([reg[k][1] for k in keys]) - r; hi = np.array([reg[k][2] for k in keys]) + r
ci = np.array([idx.get((a, b, c), -1) for a, b, c in map(tuple, pc)])
cand = ci >= 0
objok = np.array([cand_i >= 0 and int(o) in objsets[cand_i] for cand_i, o in zip(ci, po)])
boxok = cand.copy()
boxok[cand] = np.all((pp[cand] >= lo[ci[cand]]) & (pp[cand] <= hi[ci[cand]]), axis=1)
print(name, "pixels hit", ok.sum(), "registered cells", len(keys), "live photons", live.sum())
print("candidates", cand.sum(), "obj-filtered", objok.sum(), "box-filtered", boxok.sum(), "both", (objok & boxok).sum())
