"""GPU analogues of the reference's acceptance gate and engine invariants (SURVEY.md s8c:
criteria 4, 5, 6, 7, 8, 9, 11 of `tests/acceptance/acceptance.cpp` and the invariants of
`tests/test_engine.cpp`), checked on the GPU engine alone -- plus the size-independent ones
again at BASELINE.json's full C3/C4 sizes, where the CPU reference is too slow to compare
against frame by frame.
"""
import numpy as np
import pytest

from paper_2111_06906_b200 import pathreuse as pr

LIVE = 1  # path status kLive (engine.cpp:17-19)


def make(scene, synthetic=False, **cfg):
    sc = pr.Scene.synthetic(scene) if synthetic else pr.Scene.builtin(scene)
    return pr.Engine(sc, pr.make_config(**cfg))


def path_state(eng):
    info = eng.info()
    meta = eng.download("meta")
    return info, meta[:, 0].astype(np.int64), meta[:, 1].astype(np.int64), meta[:, 2] == LIVE


def light_of(info, n):
    li = np.zeros(n, dtype=np.int64)
    for k in range(info.n_lights):
        li[info.light_path_begin[k]:info.light_path_end[k]] = k
    return li


def stats_row(st):
    return tuple(getattr(st, k) for k in ("rays_traced", "rays_reused", "paths_replaced", "paths_pruned",
                                          "paths_filled", "visibility_rays"))


# ------------------------------------------------------------------ criterion 4
@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["naive", "error"])
@pytest.mark.parametrize("paths", [100_000, 2_000_000])
def test_static_full_reuse(mode, paths):
    """acceptance.cpp:110-127 + test_engine.cpp:83-99: a static scene traces nothing after
    frame 0, keeps its photon map byte-identical and renders the same image."""
    eng = make("static-box", mode=mode, paths=paths, bounces=7, dm=[8, 8, 64, 64])
    eng.run_frame()
    photons0 = eng.photon_map().tobytes()
    image0 = eng.splat(radius=0.25).tobytes()
    for f in range(1, 6):
        st = eng.run_frame()
        assert (st.rays_traced, st.paths_pruned, st.paths_filled, st.visibility_rays) == (0, 0, 0, 0), f
        assert eng.photon_map().tobytes() == photons0, f
        assert eng.splat(radius=0.25).tobytes() == image0, f


# ------------------------------------------------------------------ criterion 5
@pytest.mark.gpu
@pytest.mark.parametrize("scene,synthetic,paths", [("moving-cube", False, 10_000), ("C3", True, 2_000_000)])
def test_naive_prefix_preservation(scene, synthetic, paths):
    """acceptance.cpp:129-154: a naive retrace never changes the photons before its start."""
    eng = make(scene, synthetic, mode="naive", paths=paths, bounces=7, dm=[8, 8, 64, 64])
    eng.run_frame()
    n = eng.info().n_paths
    for f in range(1, 4):
        before = eng.photon_map().view(np.uint8).reshape(-1, 32)
        epoch = eng.download("epoch")
        eng.run_frame()
        _, count, _, alive = path_state(eng)
        start = eng.download("retrace_start").astype(np.int64)
        keep = np.where(start == 0xFF, count, start)
        now = eng.photon_map().view(np.uint8).reshape(-1, 32)
        same_epoch = alive & (eng.download("epoch") == epoch)
        checked = 0
        for b in range(eng.info().max_bounces):
            rows = np.nonzero(same_epoch & (b < keep))[0]
            idx = b * n + rows
            assert np.array_equal(now[idx], before[idx]), f"frame {f} bounce {b}"
            checked += rows.size
        assert checked > 0


# ------------------------------------------------------------------ criterion 6
def _segments(eng, two_diag):
    info, count, esc, alive = path_state(eng)
    n = info.n_paths
    aux = eng.vertex_aux()
    pos = aux["position"].reshape(info.max_bounces, n, 3)
    out = aux["outgoing"].reshape(info.max_bounces, n, 3)
    origin = eng.download("origin")[:, :3]
    emis = eng.download("emission_dir")[:, :3]
    A, Bv, P, S = [], [], [], []
    for i in range(info.max_bounces + 1):
        rows = np.nonzero(alive & (i < count + esc))[0]
        if rows.size == 0:
            continue
        a = origin[rows] if i == 0 else pos[i - 1, rows]
        d = emis[rows] if i == 0 else out[i - 1, rows]
        inner = i < count[rows]
        b = np.where(inner[:, None], pos[min(i, info.max_bounces - 1), rows],
                     (a + d * np.float32(two_diag)).astype(np.float32))
        A.append(a), Bv.append(b), P.append(rows), S.append(np.full(rows.size, i))
    return (np.concatenate(A).astype(np.float32), np.concatenate(Bv).astype(np.float32), np.concatenate(P),
            np.concatenate(S))


def _first_interior_hit(probe, a, b, eps):
    """conservativeness::first_interior_hit (acceptance.cpp:168-177): closest hit of the scene
    at the probe's current frame inside (eps, len - eps) along a -> b, or -1."""
    d = (b - a).astype(np.float32)
    ln = np.sqrt((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]).astype(np.float32)
    dirs = (d / ln[:, None]).astype(np.float32)
    rays = np.zeros((len(a), 8), dtype=np.float32)
    rays[:, :3], rays[:, 3:6], rays[:, 6], rays[:, 7] = a, dirs, eps, ln - np.float32(eps)
    hits = probe.intersect(rays)
    miss = hits[:, 1].view(np.uint32) == 0xFFFFFFFF
    return np.where(miss, np.float32(-1), hits[:, 0])


@pytest.mark.gpu
def test_conservativeness_oracle():
    """acceptance.cpp:156-237: every segment whose first interior hit changed between two
    frames is flagged (the scene is queried through a second engine one frame behind)."""
    eng = make("moving-cube", mode="naive", paths=10_000, bounces=7, dm=[8, 8, 64, 64], record_flags=True)
    probe = make("moving-cube", mode="naive", paths=100, bounces=1, dm=[2, 2, 4, 4])
    eng.run_frame()
    probe.run_frame()
    info = eng.info()
    eps = np.float32(info.eps_world)
    changed_total = 0
    for f in range(1, 5):
        a, b, p, i = _segments(eng, 2.0 * info.diagonal)
        t_prev = _first_interior_hit(probe, a, b, eps)
        eng.run_frame()
        probe.run_frame()
        t_cur = _first_interior_hit(probe, a, b, eps)
        flags = eng.download("segment_flags")
        changed = ((t_prev < 0) != (t_cur < 0)) | ((t_prev >= 0) & (np.abs(t_prev - t_cur) > eps))
        flagged = (flags[p] >> i.astype(np.uint32)) & 1
        missed = np.nonzero(changed & (flagged == 0))[0]
        assert missed.size == 0, f"frame {f}: {missed.size} changed segments not flagged, e.g. {p[missed[:3]]}"
        changed_total += int(changed.sum())
    assert changed_total > 0, "the oracle exercised changed segments"


# ------------------------------------------------------------------ criterion 7
@pytest.mark.gpu
@pytest.mark.parametrize("scene", ["armadillo-analog", "merry-go-round-analog", "villa-analog"])
def test_never_worse_ray_ordering(scene):
    """acceptance.cpp:239-272: error <= naive <= baseline rays every frame for 100 frames;
    armadillo naive <= 0.6 x baseline over frames 10-99."""
    cfg = dict(paths=20_000, bounces=7, dm=[4, 4, 8, 8])
    base, naive, err = (make(scene, mode=m, **cfg) for m in ("baseline", "naive", "error"))
    base_tail = naive_tail = 0
    for f in range(100):
        sb, sn, se = base.run_frame(), naive.run_frame(), err.run_frame()
        assert se.rays_traced <= sn.rays_traced <= sb.rays_traced, (f, se.rays_traced, sn.rays_traced,
                                                                    sb.rays_traced)
        assert sb.rays_reused == 0
        if f >= 10:
            base_tail += sb.rays_traced
            naive_tail += sn.rays_traced
    if scene == "armadillo-analog":
        assert naive_tail / base_tail <= 0.6


# ------------------------------------------------------------------ criterion 8
def _max_energy_deviation(eng, albedo):
    """max_energy_deviation (acceptance.cpp:274-295), vectorised in double."""
    info, count, _, alive = path_state(eng)
    n = info.n_paths
    ph = eng.photon_map()
    flux = np.array([list(info.flux_per_path[k]) for k in range(info.n_lights)], dtype=np.float64)
    e = flux[light_of(info, n)].copy()
    worst = 0.0
    for b in range(info.max_bounces):
        rows = np.nonzero(alive & (b < count))[0]
        if rows.size == 0:
            break
        rec = ph[b * n + rows]
        e[rows] *= albedo[rec["object_id"]]
        ref = e[rows]
        ok = ref > 1e-12
        dev = np.abs(rec["energy"].astype(np.float64) - ref)[ok] / ref[ok]
        if dev.size:
            worst = max(worst, float(dev.max()))
    return worst


@pytest.mark.gpu
def test_error_bound_drift():
    """acceptance.cpp:297-324: T=0 keeps every stored energy within 1e-5 of the path product
    for 20 frames; T=0.001 stays within (1.001)^7 - 1 over 100 frames."""
    scene = pr.Scene.builtin("moving-cube")
    desc = scene.describe()
    albedo = np.array([[desc.objects[k].material.albedo.x, desc.objects[k].material.albedo.y,
                        desc.objects[k].material.albedo.z] for k in range(desc.n_objects)],
                      dtype=np.float32).astype(np.float64)
    eng = pr.Engine(scene, pr.make_config(mode="error", paths=10_000, bounces=7, dm=[8, 8, 64, 64], threshold=0.0))
    for f in range(20):
        eng.run_frame()
        assert _max_energy_deviation(eng, albedo) <= 1e-5, f
    eng = pr.Engine(scene, pr.make_config(mode="error", paths=10_000, bounces=7, dm=[8, 8, 64, 64],
                                          threshold=0.001))
    worst = 0.0
    for _ in range(100):
        eng.run_frame()
        worst = max(worst, _max_energy_deviation(eng, albedo))
    assert worst <= 1.001 ** 7 - 1.0


# ------------------------------------------------------------------ criterion 9
@pytest.mark.gpu
def test_dm_convergence():
    """acceptance.cpp:326-379 + test_engine.cpp:191-207: DM_C equals DM_T after every fill,
    every live path's cell agrees with DM_C, and the live emission cells pass the chi-square
    test against DM_T at alpha = 0.01."""
    eng = make("parallel-spot", mode="naive", paths=100_000, bounces=7, dm=[8, 8, 64, 64])
    for f in range(23):
        eng.run_frame()
        dm_c, dm_t = eng.download("dm_current", 0), eng.download("dm_target", 0)
        assert np.array_equal(dm_c, dm_t), f
        _, _, _, alive = path_state(eng)
        observed = np.bincount(eng.download("cell")[alive], minlength=dm_t.size)
        assert np.array_equal(observed, dm_c), f
    assert int(alive.sum()) == int(dm_t.sum())
    nz = dm_t > 0
    assert not observed[~nz].any()
    chi2 = float((((observed[nz] - dm_t[nz]).astype(np.float64)) ** 2 / dm_t[nz]).sum())
    df = float(nz.sum() - 1)
    z = 2.3263478740
    crit = df * (1.0 - 2.0 / (9.0 * df) + z * np.sqrt(2.0 / (9.0 * df))) ** 3
    assert chi2 <= crit


# ------------------------------------------------------------------ criterion 11 + invariants
@pytest.mark.gpu
@pytest.mark.parametrize("scene,synthetic,paths,mode", [("moving-cube", False, 20_000, "error"),
                                                        ("parallel-spot", False, 20_000, "naive"),
                                                        ("C3", True, 2_000_000, "error")])
def test_run_to_run_determinism(scene, synthetic, paths, mode):
    """acceptance.cpp:403-433 reinterpreted for the GPU: two engines on the same
    inputs produce byte-identical stats, photon maps and images frame after frame, however
    the device scheduled their atomics."""
    cfg = dict(mode=mode, paths=paths, bounces=7, dm=[8, 8, 64, 64])
    e1, e2 = make(scene, synthetic, **cfg), make(scene, synthetic, **cfg)
    for f in range(4):
        assert stats_row(e1.run_frame()) == stats_row(e2.run_frame()), f
        assert e1.photon_map().tobytes() == e2.photon_map().tobytes(), f
        assert e1.splat(radius=0.25).tobytes() == e2.splat(radius=0.25).tobytes(), f


@pytest.mark.gpu
def test_frame_zero_identical_across_modes():
    """test_engine.cpp:70-81: frame 0 is the same full trace in every mode."""
    engines = [make("moving-cube", mode=m, paths=20_000, bounces=7, dm=[8, 8, 64, 64])
               for m in ("baseline", "naive", "error")]
    rows = [stats_row(e.run_frame()) for e in engines]
    assert rows[0] == rows[1] == rows[2]
    maps = [e.photon_map().tobytes() for e in engines]
    assert maps[0] == maps[1] == maps[2]


@pytest.mark.gpu
@pytest.mark.parametrize("scene,synthetic,paths", [("moving-cube", False, 20_000), ("C4", True, 5_000_000)])
def test_ray_accounting_and_dm_at_scale(scene, synthetic, paths):
    """test_engine.cpp:143-153 and :191-207 as size-independent properties, up to C4's full
    5M paths x 7 bounces: traced + reused rays equal the stored segments of live paths, and
    DM_C equals DM_T per light after every frame."""
    eng = make(scene, synthetic, mode="error", paths=paths, bounces=7, dm=[8, 8, 64, 64])
    for f in range(4):
        st = eng.run_frame()
        info, count, esc, alive = path_state(eng)
        assert st.rays_traced + st.rays_reused == int((count + esc)[alive].sum()), f
        for li in range(info.n_lights):
            assert np.array_equal(eng.download("dm_current", li), eng.download("dm_target", li)), (f, li)
