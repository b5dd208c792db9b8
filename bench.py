#!/usr/bin/env python
"""Benchmark of the per-frame photon-path verification + reuse pipeline (BASELINE.json).

One step = one animated frame of the north_star hot path on the configured workload:
frame_update -> verify_paths -> retrace_invalid -> splat (120x90), i.e. Engine::run_frame
(engine.cpp:201-242) + gather_image (gather.cpp:35-75) of the reference.

  value   whole-job paths/s = n_paths * steps / device time of the timed steps (CUDA events
          on the engine's stream, max over ranks); every live path is verified each frame
          and the invalid ones are retraced.
  e2e     the same metric through the public Python API (Engine.run_frame + Engine.splat
          returning the host image), wall clock, host<->device copies included.
  --impl reference: the reference CPU engine (oracle/_ref, built from /root/reference) on a
          bounded path-prefix sample of the same workload, all host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "C1": dict(desc="Cornell box (~1K static tris), point light, translating 992-tri sphere",
               mode="naive", paths=65536, bounces=3, threshold=0.001),
    "C2": dict(desc="Cornell box, rect area light translating in its plane (DM remap)",
               mode="naive", paths=1048576, bounces=5, threshold=0.001),
    "C3": dict(desc="Sponza-scale synthetic (282K static tris + 4 x 20K dynamic), disc light",
               mode="error", paths=2097152, bounces=7, threshold=0.01),
    "C4": dict(desc="Villa-scale synthetic (1.02M static tris + 8 x 20K dynamic + 2 moving lights)",
               mode="error", paths=5000000, bounces=7, threshold=0.001),
}
# reference CPU sample sizes (~10 s of CPU work for the bench line, per-path cost scales linearly)
CPU_SAMPLE_PATHS = {"C1": 65536, "C2": 1048576, "C3": 524288, "C4": 1048576}
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C4", choices=sorted(WORKLOADS))
    ap.add_argument("--paths", type=int, default=0, help="override n_paths")
    ap.add_argument("--splat-mode", type=int, default=1, help="0 atomic splat, 1 ordered bit-exact gather")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the e2e replay (profiling passes)")
    ap.add_argument("--cpu-sample", type=int, default=0)
    ap.add_argument("--no-splat-sweep", action="store_true", help="skip the per-mode splat timings")
    ap.add_argument("--splat-overlap", type=int, default=1,
                    help="1: the device-timed loop runs each frame's splat on the engine's side stream, "
                         "overlapping the next frame's scene update and occlusion flags "
                         "(prx_engine_set_splat_overlap); 0: splat, then the next frame")
    ap.add_argument("--extra", default="C1,C2,C3,C5w,C5b",
                    help="secondary workloads measured after the headline (N=1 only; 'none' skips): "
                         "C1-C3, C5w = C5 worst case (32M paths, 64 movers, baseline: full retrace), "
                         "C5b = C5 best case (32M paths, 1 mover, error mode)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: N x the workload's paths over N GPUs; strong: the workload's paths split over N")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        loaded = [s for s in sm if smax and s > 0.3 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(kernel):
    """DRAM bytes (read + write) of one steady-state launch of `kernel` from the newest
    committed ncu --set full summary (profiles/rNN_traffic.json, C4 workload), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r*_traffic.json")))
    for f in reversed(files):
        try:
            with open(f) as fh:
                k = json.load(fh)["kernels"].get(kernel)
            if k:
                return float(k["dram_bytes"]), os.path.relpath(f, os.path.dirname(os.path.abspath(__file__)))
        except (OSError, ValueError, KeyError):
            continue
    return None, None


def peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def scene_for(pr, name):
    return pr.Scene.synthetic(name)


def run_reference(args, name, n_paths, steps, warmup):
    """The reference CPU engine on a path-prefix sample; returns (paths/s, detail).

    Only oracle/_ref is loaded: the scene comes from the generators compiled into the oracle
    library (oracle/scene_gen.cpp), the config from pure-Python make_config (no _prx.so)."""
    from oracle import ref
    from paper_2111_06906_b200.pathreuse import make_config

    w = WORKLOADS[name]
    rscene = ref.RefScene.synthetic(name)
    cfg = make_config(mode=w["mode"], paths=n_paths, bounces=w["bounces"],
                      dm=[8, 8, 64, 64], threshold=w["threshold"], seed=1, workers=0)
    eng = ref.RefEngine(rscene, cfg)
    eng.set_workers(0)
    for _ in range(warmup):
        eng.run_frame()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        eng.run_frame()
        eng.gather(radius=0.25, workers=0)
        times.append(time.perf_counter() - t0)
    mean = sum(times) / len(times)
    return n_paths / mean, {"frame_s_mean": mean, "frames": steps, "warmup": warmup}


EXTRA = {  # the other BASELINE.json configurations, one B200
    "C1": dict(scene=("C1", 0), **{k: WORKLOADS["C1"][k] for k in ("mode", "paths", "bounces", "threshold")}),
    "C2": dict(scene=("C2", 0), **{k: WORKLOADS["C2"][k] for k in ("mode", "paths", "bounces", "threshold")}),
    "C3": dict(scene=("C3", 0), **{k: WORKLOADS["C3"][k] for k in ("mode", "paths", "bounces", "threshold")}),
    "C5w": dict(scene=("C5", 64), mode="baseline", paths=32 << 20, bounces=7, threshold=0.001),
    "C5b": dict(scene=("C5", 1), mode="error", paths=32 << 20, bounces=7, threshold=0.001),
}


def measure_extra(pr, L, torch, stream, key, steps=5, warmup=3, overlap=True):
    """Device ms/frame (frame + 120x90 ordered splat) of one secondary workload (with the
    overlapped splat like the headline loop, unless overlap=False)."""
    import ctypes as C

    w = EXTRA[key]
    scene = pr.Scene.synthetic(*w["scene"])
    eng = pr.Engine(scene, pr.make_config(mode=w["mode"], paths=w["paths"], bounces=w["bounces"],
                                          dm=[8, 8, 64, 64], threshold=w["threshold"], seed=1))
    eng.set_stream(stream.cuda_stream)
    cam = scene.describe().camera
    img = torch.zeros(cam.height * cam.width * 3, dtype=torch.float32, device="cuda")
    sts = []
    eng.set_splat_overlap(overlap)

    def one(collect, timed_splat=False):
        st, sst = L.FrameStats(), L.FrameStats()
        L.check(L.lib().prx_run_frame(eng.handle, C.byref(st)))
        L.check(L.lib().prx_splat(eng.handle, C.byref(cam), 0.25, 1, None, C.c_void_p(img.data_ptr()),
                                  C.byref(sst) if timed_splat or not overlap else None))
        if collect:
            sts.append((st, sst))

    for _ in range(warmup):
        one(False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        one(True)
    if overlap:
        L.check(L.lib().prx_engine_synchronize(eng.handle))  # (joins the last splat before e1)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    splat_alone = []
    if overlap:  # the splat stage alone (serial splats with their own events) on the last frames
        for _ in range(3):
            sst = L.FrameStats()
            L.check(L.lib().prx_splat(eng.handle, C.byref(cam), 0.25, 1, None, C.c_void_p(img.data_ptr()),
                                      C.byref(sst)))
            splat_alone.append(sst.ms_splat)
    counts = scene.counts()
    out = {"scene": f"{w['scene'][0]} ({counts['static_triangles']} static + {counts['dynamic_triangles']} dynamic tris)",
           "mode": w["mode"], "paths": w["paths"], "bounces": w["bounces"], "ms_per_step": ms,
           "paths_per_s": w["paths"] / (ms * 1e-3),
           "stages_ms": {k: statistics.median(getattr(a, f) for a, _ in sts)
                         for k, f in (("verify", "ms_verify"), ("retrace", "ms_retrace"))},
           "rays_traced_per_frame": statistics.median(a.rays_traced for a, _ in sts)}
    out["stages_ms"]["splat"] = statistics.median(splat_alone) if overlap else statistics.median(b.ms_splat for _, b in sts)
    out["splat_overlap"] = overlap
    eng.close()
    return out


def main():
    args = parse_args()
    rank, world, local = dist_env()
    name = args.workload
    w = WORKLOADS[name]
    # weak scaling (default): every GPU holds the workload's full path count (a contiguous shard
    # of the N-times-larger problem), so per-GPU work is fixed as N grows; strong scaling: the
    # workload's path count is split over the N GPUs (north_star: a 5M-path frame on 8 B200)
    per_job = args.paths or w["paths"]
    strong = args.scaling == "strong" and args.impl == "ours"
    n_paths = per_job if strong else per_job * (world if args.impl == "ours" else 1)
    paths_per_gpu = n_paths // world if strong else per_job
    unit = "paths/s"
    metric = "verified+retraced photon paths/s (frame = verify+retrace+splat)"
    config = {"workload": f"{name}: {w['desc']}", "n_paths": n_paths, "paths_per_gpu": paths_per_gpu,
              "parallelism": f"contiguous path shards x{world} (in-engine NCCL DM/prune/fill/counter/image exchanges)",
              "max_bounces": w["bounces"],
              "mode": w["mode"], "threshold": w["threshold"], "dm_dims": [8, 8, 64, 64],
              "image": "120x90", "gather_radius": 0.25,
              "l2": "inputs larger than L2 (path store >= 1 GB for C2-C4)"}

    if args.impl == "reference":
        if rank != 0:
            return
        sample = args.cpu_sample or CPU_SAMPLE_PATHS[name]
        value, det = run_reference(args, name, sample, args.steps, args.warmup)
        cores = os.cpu_count()
        line = {"impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": 0,
                "steps": args.steps, "warmup": args.warmup,
                # measured: one step = one frame (+ gather_image) of the `sample`-path prefix
                "ms_per_step": det["frame_s_mean"] * 1e3, "sample_paths": sample,
                # linear extrapolation to the full path count (per-path work is independent)
                "ms_per_full_frame_extrapolated": det["frame_s_mean"] * 1e3 * (n_paths / sample),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (procedural scene, seed 1)", "config": config,
                "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "reference",
                                 "sample": f"the {name} scene and configuration with {sample} of its "
                                           f"{n_paths} paths (per-path cost is independent of the path "
                                           f"count), {args.warmup} warm-up + {args.steps} timed frames "
                                           f"incl. gather_image"},
                "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch

    # one process per GPU; PRX_DIST_BACKEND=gloo with fewer GPUs than ranks is a functional
    # check of the sharded path only (ranks share a device), never a measurement
    backend = os.environ.get("PRX_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2111_06906_b200 import pathreuse as pr
    from paper_2111_06906_b200 import _lib as L

    scene = scene_for(pr, name)
    scene_counts = scene.counts()
    shard = (0, 0)
    if world > 1:
        shard = (n_paths * rank // world, n_paths * (rank + 1) // world)
    cfg = pr.make_config(mode=w["mode"], paths=n_paths, bounces=w["bounces"], dm=[8, 8, 64, 64],
                         threshold=w["threshold"], seed=1, device=local, shard=shard)
    import ctypes as C

    # one non-default stream shared by torch and the engine, so the CUDA events below time the
    # engine's device work (torch's default stream handle is 0, which the engine would replace
    # by a private stream)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    legacy = world > 1 and backend != "nccl"
    if legacy:
        config["parallelism"] = f"contiguous path shards x{world} (host-phased {backend} exchanges: functional check)"
    comm = None
    if legacy:  # functional multi-rank check on one device (gloo): the host-phased protocol
        from paper_2111_06906_b200.distributed import GpuExecutor, TorchCollectives, run_frame_distributed

        ex = GpuExecutor(scene, cfg, stream)
        eng = ex.engine
        coll = TorchCollectives()
    else:
        eng = pr.Engine(scene, cfg)
        eng.set_stream(stream.cuda_stream)
    if world > 1 and not legacy:
        # path-sharded frames: the exchanges run inside the engine over NCCL (comm.cpp); the
        # unique id travels once through torch.distributed
        from paper_2111_06906_b200.distributed import Communicator, attach

        obj = [Communicator.nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        comm = Communicator.nccl(obj[0], rank, world, local)
        attach(eng, comm)
    cam = scene.describe().camera
    img_dev = torch.zeros(cam.height * cam.width * 3, dtype=torch.float32, device="cuda")
    frame_no = [0]

    overlap = bool(args.splat_overlap) and not legacy
    L.check(L.lib().prx_engine_set_splat_overlap(eng.handle, 1 if overlap else 0))
    config["splat_overlap"] = ("on: each frame's splat runs on the engine's side stream during the next frame's "
                               "scene update and occlusion flags (the frame's verify stage time includes its wait; "
                               "the last splat completes inside the timed region)") if overlap else "off"

    def step(collect=None, sync_splat=False):
        if legacy:
            d = run_frame_distributed(ex, coll, frame_no[0])
            st = L.FrameStats()
            for k in L.FrameStats.COUNTS + ("live_segments_before", "paths_retraced"):
                setattr(st, k, int(d[k]))
        else:  # one prx_run_frame (+ its exchanges when sharded), one read-back
            st = L.FrameStats()
            L.check(L.lib().prx_run_frame(eng.handle, C.byref(st)))
        frame_no[0] += 1
        sst = L.FrameStats()
        # (stats request a host wait for the splat's timing: the overlapped loop passes none)
        L.check(L.lib().prx_splat(eng.handle, C.byref(cam), 0.25, args.splat_mode, None,
                                  C.c_void_p(img_dev.data_ptr()),
                                  None if overlap and not sync_splat else C.byref(sst)))
        if legacy:
            torch.distributed.all_reduce(img_dev)
        if collect is not None:
            collect.append((st, sst))

    first = []
    step(first, sync_splat=True)  # frame 0: the cold fill (reported separately)
    for _ in range(max(3, args.warmup) - 1):
        step()
    stats = []
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = eng.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step(stats)
    if overlap:  # the engine stream waits for the last step's splat (side stream) before ev1
        L.check(L.lib().prx_engine_synchronize(eng.handle))
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clk = clocks.stop()
    launches = eng.launch_count() - launches0
    elapsed_ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([elapsed_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    value = n_paths * args.steps / (elapsed_ms * 1e-3)

    # stage breakdown (device events inside the engine)
    def med(f):
        return statistics.median(f(a, b) for a, b in stats)

    verify_ms = med(lambda a, b: a.ms_verify)
    retrace_ms = med(lambda a, b: a.ms_retrace)
    splat_ms = med(lambda a, b: b.ms_splat)
    update_ms = med(lambda a, b: a.ms_frame_update)
    trace_ms = med(lambda a, b: a.t_trace * 1e3)
    occl_ms = med(lambda a, b: a.t_occlusion * 1e3)
    seg_before = med(lambda a, b: a.live_segments_before)
    retraced = med(lambda a, b: a.paths_retraced)
    traced = med(lambda a, b: a.rays_traced)
    vis = med(lambda a, b: a.visibility_rays)

    # splat stage alone, both modes, at the scene camera and at the paper's 1920x1080, on the
    # final photon map (device time from the engine's own events, median of 5)
    def time_splat(mode, w_px, h_px, reps=5):
        c = L.Camera(cam.position, cam.look_at, cam.fov_deg, w_px, h_px)
        buf = img_dev if w_px * h_px == cam.width * cam.height else \
            torch.zeros(w_px * h_px * 3, dtype=torch.float32, device="cuda")
        ts = []
        for _ in range(reps + 1):
            sst = L.FrameStats()
            L.check(L.lib().prx_splat(eng.handle, C.byref(c), 0.25, mode, None, C.c_void_p(buf.data_ptr()),
                                      C.byref(sst)))
            ts.append(sst.ms_splat)
        return statistics.median(ts[1:])

    splat_modes = {}
    if not args.no_splat_sweep:
        for mode, tag in ((1, "ordered"), (0, "atomic")):
            for w_px, h_px in ((cam.width, cam.height), (1920, 1080)):
                splat_modes[f"{tag}_{w_px}x{h_px}"] = time_splat(mode, w_px, h_px)
    if overlap:  # the overlapped splats carry no timing: the splat stage alone on the final map
        splat_ms = splat_modes.get(f"{'ordered' if args.splat_mode == 1 else 'atomic'}_{cam.width}x{cam.height}") \
            or time_splat(args.splat_mode, cam.width, cam.height)

    # e2e through the public API with host buffers (stats + image read back every step), on a
    # fresh engine replaying the same frames as the timed loop (the workload drifts with the
    # animation, so later frames would not be comparable)
    if args.no_e2e:
        eng2 = eng
    elif legacy:
        ex2 = GpuExecutor(scene, cfg, stream)
        eng2 = ex2.engine
    else:
        eng2 = pr.Engine(scene, cfg)
        eng2.set_stream(stream.cuda_stream)
        if comm is not None:  # the same communicator: its collectives are stream-ordered
            attach(eng2, comm)
    frame2 = [0]
    e2e_dev = []  # device stage times of the e2e frames (diagnostic: host overhead = wall - this)
    e2e_img = []
    host_img = np.zeros((cam.height, cam.width, 3), dtype=np.float32)
    if overlap and not args.no_e2e:
        eng2.set_splat_overlap(True)

    def step_e2e(collect):
        if legacy:  # sharded frame + reduced image read back to the host
            run_frame_distributed(ex2, coll, frame2[0])
            L.check(L.lib().prx_splat(eng2.handle, C.byref(cam), 0.25, args.splat_mode, None,
                                      C.c_void_p(img_dev.data_ptr()), None))
            torch.distributed.all_reduce(img_dev)
            img_dev.cpu()
        elif overlap:  # the public Python API, pipelined: run_frame returns with the previous
            # step's host image in place; this step's splat fills it by the next call
            st = eng2.run_frame()
            e2e_img.append(float(host_img[0, 0, 0]))  # (the host reads the previous step's image)
            eng2.splat_into(host_img, radius=0.25, mode=args.splat_mode)
            if collect:
                e2e_dev.append(st.ms_frame_update + st.ms_verify + st.ms_retrace)
        else:  # the public Python API: counters and the host image every step
            st = eng2.run_frame()
            sst = L.FrameStats()
            eng2.splat(radius=0.25, mode=args.splat_mode, st=sst)
            if collect:
                e2e_dev.append(st.ms_frame_update + st.ms_verify + st.ms_retrace + sst.ms_splat)
        frame2[0] += 1

    e2e_steps = 0 if args.no_e2e else args.steps
    for _ in range(max(3, args.warmup) if e2e_steps else 0):
        step_e2e(False)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    xfer0 = eng2.transfer_bytes()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        step_e2e(True)
    if overlap and e2e_steps:  # the last step's host image lands inside the timed region
        eng2.synchronize()
        e2e_img.append(float(host_img[0, 0, 0]))
    e2e_s = max(time.perf_counter() - t0, 1e-9)
    xfer1 = eng2.transfer_bytes()
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = n_paths * e2e_steps / e2e_s if e2e_steps else None
    # bytes the engine itself copied per step (counted inside the library), plus the reduced
    # image read back by torch on the sharded path
    h2d = (xfer1[0] - xfer0[0]) // max(e2e_steps, 1)
    d2h = (xfer1[1] - xfer0[1]) // max(e2e_steps, 1) + (12 * cam.width * cam.height if legacy else 0)

    # roofline of the dominant kernel stage (trace): algorithmic bytes per traced segment =
    # 64 B written (4 x float4 vertex streams) + 64 B per retraced path start (meta, rstart,
    # epoch, origin/emission or previous vertex, truncation of the tail records).
    hbm, peak_src = peaks()
    trace_bytes = traced * 64 + retraced * 64
    achieved = trace_bytes / (trace_ms * 1e-3) / 1e9 if trace_ms > 0 else 0.0
    traffic, traffic_src = ncu_traffic("k_trace") if name == "C4" else (None, None)
    roofline = {"bound": "hbm", "kernel": "k_trace (stage_trace: compaction + trace + finalize)",
                "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": trace_bytes, "peak_source": peak_src,
                "note": "traversal is latency/issue-bound: BVH reads are implementation-defined "
                        "and not in the algorithmic bytes"}

    line = {"metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (procedural scene, seed 1)", "config": config,
            "stages_ms": {"frame_update": update_ms, "verify": verify_ms, "occlusions": occl_ms,
                          "retrace": retrace_ms, "trace": trace_ms, "splat": splat_ms},
            "splat_ms": splat_modes,
            "verified_segments_per_s": seg_before / (verify_ms * 1e-3) if verify_ms else None,
            "retraced_paths_per_s": retraced / (retrace_ms * 1e-3) if retrace_ms else None,
            "rays_traced_per_s": traced / (trace_ms * 1e-3) if trace_ms else None,
            "frame0_ms": {"frame_update": first[0][0].ms_frame_update, "verify": first[0][0].ms_verify,
                          "retrace": first[0][0].ms_retrace, "splat": first[0][1].ms_splat,
                          "rays_traced": first[0][0].rays_traced},
            "retraced_paths_per_frame": retraced, "rays_traced_per_frame": traced,
            "visibility_rays_per_frame": vis,
            "e2e": {"value": e2e_value, "unit": unit, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3 / e2e_steps if e2e_steps else None,
                    "device_ms_per_step": (statistics.mean(e2e_dev) if e2e_dev else None),
                    "api": ("Engine.run_frame() + Engine.splat_into(host image), pipelined: each run_frame "
                            "returns with the previous step's image filled" if overlap and not legacy
                            else "Engine.run_frame() + Engine.splat() (host image)")},
            "gpu_launches": launches, "clocks": clk, "roofline": roofline,
            "scene_counts": {"static_tris": scene_counts["static_triangles"],
                             "dynamic_tris": scene_counts["dynamic_triangles"]}}

    if world == 1 and args.extra != "none":  # the other BASELINE configurations, device time
        if not args.no_e2e:
            eng2.close()
        eng.close()
        torch.cuda.synchronize()
        line["workloads"] = {}
        for key in [k for k in args.extra.split(",") if k]:
            line["workloads"][key] = measure_extra(pr, L, torch, stream, key, overlap=bool(args.splat_overlap))

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = args.cpu_sample or CPU_SAMPLE_PATHS[name]
        try:
            cpu_value, det = run_reference(args, name, sample, 2, 1)
            line["cpu_baseline"] = {"value": cpu_value, "unit": unit, "cores": os.cpu_count(),
                                    "kind": "reference",
                                    "sample": f"the {name} scene and configuration with {sample} of its "
                                              f"{n_paths} paths (per-path cost is independent of the path "
                                              f"count), 1 warm-up + 2 timed frames incl. gather_image"}
        except Exception as exc:  # oracle not built on this box
            line["cpu_baseline"] = {"value": None, "unit": unit, "cores": os.cpu_count(),
                                    "kind": "reference", "sample": f"unavailable: {exc}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
