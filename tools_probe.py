import sys, time, json
sys.path.insert(0, '.')
from paper_2111_06906_b200 import pathreuse as pr
cfgs = {
 "C1": dict(mode="naive", paths=65536, bounces=3, dm=[8,8,64,64]),
 "C2": dict(mode="naive", paths=1048576, bounces=5, dm=[8,8,64,64]),
 "C3": dict(mode="error", paths=2097152, bounces=7, dm=[8,8,64,64], threshold=0.01),
 "C4": dict(mode="error", paths=5000000, bounces=7, dm=[8,8,64,64], threshold=0.001),
}
for name in sys.argv[1:]:
    t=time.time(); sc = pr.Scene.synthetic(name); tb=time.time()-t
    eng = pr.Engine(sc, pr.make_config(**cfgs[name])); ti=time.time()-t-tb
    print(name, sc.counts(), f"scene {tb:.2f}s engine {ti:.2f}s", flush=True)
    for f in range(6):
        t=time.time(); st = eng.run_frame(); st2 = pr.L.FrameStats() if False else None
        import ctypes
        img_st = pr.L.FrameStats()
        img = eng.splat(st=img_st)
        wall=time.time()-t
        d = st.as_dict()
        print(f" f{f} wall {wall*1e3:8.1f}ms upd {d['ms_frame_update']:.2f} ver {d['ms_verify']:.2f} (orig {d['t_update']*1e3:.2f} occl {d['t_occlusion']*1e3:.2f} dm {d['t_dm']*1e3:.2f}) ret {d['ms_retrace']:.2f} (prune {d['t_prune']*1e3:.2f} fill {d['t_fill']*1e3:.2f} trace {d['t_trace']*1e3:.2f}) splat {img_st.ms_splat:.2f} | traced {d['rays_traced']} reused {d['rays_reused']} vis {d['visibility_rays']} pruned {d['paths_pruned']} filled {d['paths_filled']} repl {d['paths_replaced']} retr {d['paths_retraced']}", flush=True)
