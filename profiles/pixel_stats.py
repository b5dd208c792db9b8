"""Per-pixel work of the ordered gather on a BASELINE workload (after 6 frames): candidate
photons tested (live photons in the reachable neighbour cells of the pixel's hit point) and
contributors (same object, |x_ph - x|^2 <= r^2), as k_gather_staged sees them.
usage: python profiles/pixel_stats.py [C4|C2|C3]"""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2111_06906_b200 import pathreuse as pr  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
w = bench.WORKLOADS[name]
sc = pr.Scene.synthetic(name)
eng = pr.Engine(sc, pr.make_config(mode=w["mode"], paths=w["paths"], bounces=w["bounces"], dm=[8, 8, 64, 64],
                                   threshold=w["threshold"], seed=1))
for _ in range(6):
    eng.run_frame()
cam = sc.describe().camera
W, H = cam.width, cam.height


def v(a):
    return np.array([a.x, a.y, a.z], dtype=np.float32)


pos, at = v(cam.position), v(cam.look_at)
fwd = at - pos
fwd /= np.linalg.norm(fwd)
up = np.array([0, 1, 0], np.float32)
if abs(fwd @ up) > 0.999:
    up = np.array([1, 0, 0], np.float32)
right = np.cross(fwd, up)
right /= np.linalg.norm(right)
upv = np.cross(right, fwd)
th = np.tan(cam.fov_deg * np.pi / 360)
asp = W / H
px, py = np.meshgrid(np.arange(W), np.arange(H))
sx = (2 * (px + 0.5) / W - 1) * th * asp
sy = (1 - 2 * (py + 0.5) / H) * th
d = fwd[None, None] + right[None, None] * sx[..., None] + upv[None, None] * sy[..., None]
d = (d / np.linalg.norm(d, axis=-1, keepdims=True)).reshape(-1, 3).astype(np.float32)
rays = np.zeros((len(d), 8), np.float32)
rays[:, :3] = pos
rays[:, 3:6] = d
rays[:, 7] = 3.4e38
hits = eng.intersect(rays)
obj = hits[:, 1].view(np.uint32)
ok = obj != 0xFFFFFFFF
hp, ho = hits[ok, 3:6], obj[ok]
r = 0.25
ph = eng.download("pos_obj").reshape(-1, 4)
pobj = ph[:, 3].view(np.uint32)
live = pobj != 0xFFFFFFFF
pp, po = ph[live, :3], pobj[live]
pc = np.floor(pp / r).astype(np.int64)
key = (pc[:, 0] + (1 << 20)) * (1 << 42) + (pc[:, 1] + (1 << 20)) * (1 << 21) + (pc[:, 2] + (1 << 20))
order = np.argsort(key, kind="stable")
ks = key[order]
uk, start, cnt = np.unique(ks, return_index=True, return_counts=True)
cand, contrib = np.zeros(len(hp), np.int64), np.zeros(len(hp), np.int64)
for q, (x, o) in enumerate(zip(hp, ho)):
    c = np.floor(x / r).astype(np.int64)
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                cc = c + np.array([dx, dy, dz])
                lo, hi = cc * r, (cc + 1) * r
                gap = np.maximum(0, np.maximum(lo - x, x - hi))
                if gap @ gap > r * r * (1 + 1e-4):
                    continue
                k = (cc[0] + (1 << 20)) * (1 << 42) + (cc[1] + (1 << 20)) * (1 << 21) + (cc[2] + (1 << 20))
                j = np.searchsorted(uk, k)
                if j >= len(uk) or uk[j] != k:
                    continue
                idx = order[start[j]:start[j] + cnt[j]]
                cand[q] += cnt[j]
                dd = pp[idx] - x
                contrib[q] += int(np.count_nonzero(((dd * dd).sum(1) <= r * r) & (po[idx] == o)))


def dist(a):
    return (f"sum {a.sum():.3e} mean {a.mean():.0f} p50 {np.percentile(a, 50):.0f} p90 {np.percentile(a, 90):.0f} "
            f"p99 {np.percentile(a, 99):.0f} max {a.max()}")


print(name, "hit pixels", len(hp), "of", W * H, "live photons", int(live.sum()))
print("candidates/pixel  ", dist(cand))
print("contributors/pixel", dist(contrib))
