"""Path-sharded frames across GPUs.

Paths are split into contiguous id ranges, one per rank.  Scene, BVHs and DM_T are
replicated; the only cross-rank data of a frame are
  * DM_C per light                     -> all-reduce(sum)       (stage_compute_dm)
  * per-cell unmarked prune counts     -> all-gather -> exclusive prefix over lower
                                          ranks + total (stage_prune's "trim from the
                                          highest path id down", engine.cpp:459-466)
  * per-light dead-slot counts         -> all-gather -> prefix + total (stage_fill's
                                          "deficit cells ascending <-> free slots
                                          ascending", engine.cpp:503-519)
  * 8 frame counters                   -> all-reduce(sum)
and, for the image, the per-rank splat buffers (reduce).  With these exchanges every rank
computes exactly what the single-engine reference computes for its slice.

Two drivers of the same protocol:
  * in-engine (the product path): an engine with a collectives table (Communicator: NCCL,
    or the in-process local backend of EngineGroup) enqueues every exchange on its own
    stream inside prx_run_frame / prx_splat -- one host read-back per frame;
  * host-phased (run_frame_distributed / run_frame_loopback): the frame written as phases
    over an *executor* (one shard, the C engine's prx_prune_count/apply, prx_fill_count/apply
    entry points, or the C oracle port in the gloo CPU tests) with torch.distributed
    collectives between the phases -- the protocol's CPU test harness.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence

import numpy as np

from . import _lib as L
from .pathreuse import Engine, Scene, make_config

COUNTER_KEYS = ("rays_traced", "paths_replaced", "paths_pruned", "paths_filled", "visibility_rays",
                "live_segments_before", "paths_retraced", "segments")


def shard_range(n_paths: int, rank: int, world: int) -> tuple:
    return n_paths * rank // world, n_paths * (rank + 1) // world


class _CudaArray:
    """Zero-copy torch view of a device buffer owned by the engine."""

    def __init__(self, ptr: int, n: int, typestr: str = "<u4"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


class GpuExecutor:
    """One path shard on one CUDA device, driven through the C ABI."""

    def __init__(self, scene: Scene, config: L.Config, torch_stream=None):
        import torch

        self.torch = torch
        self.engine = Engine(scene, config)
        self.stream = torch_stream
        if torch_stream is not None:
            self.engine.set_stream(torch_stream.cuda_stream)
        self._ev = {}
        info = self.engine.info()
        self.n_lights = info.n_lights
        self.cells = [info.dm_cells[i] for i in range(self.n_lights)]
        self.mode = config.mode
        self.device = torch.device("cuda", config.device)
        self._unm = [torch.zeros(c, dtype=torch.int32, device=self.device) for c in self.cells]
        self.st = L.FrameStats()

    def _mark(self, name: str, end: bool):
        """CUDA event on the engine's stream (stage times of this shard, for reporting)."""
        if self.stream is None:
            return
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record(self.stream)
        self._ev.setdefault(name, [None, None])[1 if end else 0] = ev

    def frame_update(self):
        self.st = L.FrameStats()
        self._ev = {}
        self._mark("frame_update", False)
        self.engine.frame_update(self.st)
        self._mark("frame_update", True)

    def verify(self):
        self._mark("verify", False)
        self.engine.verify_paths(self.st)
        self._mark("verify", True)

    def dm_buffers(self) -> list:
        self.engine.synchronize()
        out = []
        for li in range(self.n_lights):
            ptr, cells = C.c_void_p(), C.c_uint32()
            L.check(L.lib().prx_engine_dm_current(self.engine.handle, li, C.byref(ptr), C.byref(cells)))
            t = self.torch.as_tensor(_CudaArray(ptr.value, cells.value, "<i4"), device=self.device)
            out.append(t)
        return out

    def dm_commit(self, bufs):  # buffers alias the engine's DM_C
        # the all-reduce ran on torch's stream, which need not be the engine's (a 0 handle
        # gives the engine a private stream): a device-wide sync orders it before the next
        # engine kernel in every mode (baseline frames have no prune sync)
        self.torch.cuda.synchronize(self.device)

    def prune_count(self) -> list:
        self.torch.cuda.synchronize(self.device)
        arr = (C.c_void_p * self.n_lights)(*[t.data_ptr() for t in self._unm])
        L.check(L.lib().prx_prune_count(self.engine.handle, C.cast(arr, C.POINTER(C.POINTER(C.c_uint32)))))
        self.engine.synchronize()
        return self._unm

    def prune_apply(self, prefix: list, total: list):
        self._keep = (prefix, total)
        pa = (C.c_void_p * self.n_lights)(*[t.data_ptr() for t in prefix])
        ta = (C.c_void_p * self.n_lights)(*[t.data_ptr() for t in total])
        self.torch.cuda.synchronize(self.device)
        L.check(L.lib().prx_prune_apply(self.engine.handle, C.cast(pa, C.POINTER(C.POINTER(C.c_uint32))),
                                        C.cast(ta, C.POINTER(C.POINTER(C.c_uint32))), C.byref(self.st)))

    def fill_count(self) -> list:
        out = (C.c_uint32 * self.n_lights)()
        L.check(L.lib().prx_fill_count(self.engine.handle, out))
        return list(out)

    def fill_apply(self, prefix: Sequence[int], total: Sequence[int]):
        pa = (C.c_uint64 * self.n_lights)(*prefix)
        ta = (C.c_uint64 * self.n_lights)(*total)
        L.check(L.lib().prx_fill_apply(self.engine.handle, pa, ta, C.byref(self.st)))

    def trace(self) -> dict:
        self._mark("trace", False)
        st = self.engine.run_stage("trace")
        self._mark("trace", True)
        d = {k: getattr(st, k) for k in COUNTER_KEYS if k != "segments"}
        d["segments"] = st.rays_traced + st.rays_reused
        # this shard's device stage times (CUDA events on its stream), for reporting
        self.local_ms = {}
        if self.stream is not None:
            self.stream.synchronize()
            self.local_ms = {k: a.elapsed_time(b) for k, (a, b) in self._ev.items() if a is not None and b is not None}
        return d

    def new_tensor(self, values, dtype="int64"):
        return self.torch.tensor(values, dtype=getattr(self.torch, dtype), device=self.device)


# ------------------------------------------------------------------------------ phases
def _prefix_total(torch, gathered: List, rank: int):
    stacked = torch.stack(gathered)
    total = stacked.sum(0).to(gathered[0].dtype)
    prefix = stacked[:rank].sum(0).to(gathered[0].dtype) if rank > 0 else torch.zeros_like(gathered[0])
    return prefix.contiguous(), total.contiguous()


def _frame_counts(local: dict) -> list:
    return [int(local[k]) for k in COUNTER_KEYS]


def _stats_from(total: Sequence[int], frame: int, mode: int) -> dict:
    d = dict(zip(COUNTER_KEYS, [int(x) for x in total]))
    d["rays_reused"] = d["segments"] - d["rays_traced"]
    d["frame"] = frame
    d["mode"] = L.MODE_NAMES[mode]
    return d


class TorchCollectives:
    """torch.distributed process group (NCCL for CUDA tensors, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allreduce_sum_(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def allgather(self, t) -> list:
        out = [t.new_empty(t.shape) for _ in range(self.world)]
        self.dist.all_gather(out, t.contiguous(), group=self.group)
        return out


def run_frame_distributed(ex, coll, frame: int) -> dict:
    """One sharded frame on this rank (all ranks call it collectively)."""
    import torch

    ex.frame_update()
    ex.verify()
    bufs = ex.dm_buffers()
    for t in bufs:
        coll.allreduce_sum_(t)
    ex.dm_commit(bufs)
    if ex.mode != L.MODES["baseline"]:
        unm = ex.prune_count()
        prefix, total = [], []
        for t in unm:
            p, s = _prefix_total(torch, coll.allgather(t), coll.rank)
            prefix.append(p)
            total.append(s)
        ex.prune_apply(prefix, total)
    dead = ex.fill_count()
    parts = coll.allgather(ex.new_tensor(dead))
    stacked = torch.stack(parts).cpu().numpy()
    prefix = [int(x) for x in stacked[: coll.rank].sum(0)] if coll.rank else [0] * len(dead)
    total = [int(x) for x in stacked.sum(0)]
    ex.fill_apply(prefix, total)
    local = ex.trace()
    cnt = ex.new_tensor(_frame_counts(local))
    coll.allreduce_sum_(cnt)
    out = _stats_from(cnt.cpu().tolist(), frame, ex.mode)
    out["local_ms"] = dict(getattr(ex, "local_ms", {}))
    return out


def run_frame_loopback(exs: List, frame: int) -> dict:
    """The same protocol over several executors in one process (shards on one device)."""
    import torch

    world = len(exs)
    for ex in exs:
        ex.frame_update()
        ex.verify()
    bufs = [ex.dm_buffers() for ex in exs]
    dev0 = bufs[0][0].device if bufs[0] else None
    for li in range(len(bufs[0])):
        s = sum(b[li].to(dev0) for b in bufs)  # shards may live on different devices
        for b in bufs:
            b[li].copy_(s)
    for ex, b in zip(exs, bufs):
        ex.dm_commit(b)
    if exs[0].mode != L.MODES["baseline"]:
        unms = [[t.clone() for t in ex.prune_count()] for ex in exs]
        for r, ex in enumerate(exs):
            prefix, total = [], []
            for li in range(len(unms[0])):
                p, s = _prefix_total(torch, [unms[q][li].to(ex.device) for q in range(world)], r)
                prefix.append(p)
                total.append(s)
            ex.prune_apply(prefix, total)
    deads = np.array([ex.fill_count() for ex in exs], dtype=np.int64)
    for r, ex in enumerate(exs):
        ex.fill_apply([int(x) for x in deads[:r].sum(0)] if r else [0] * deads.shape[1],
                      [int(x) for x in deads.sum(0)])
    total = np.zeros(len(COUNTER_KEYS), dtype=np.int64)
    for ex in exs:
        total += np.array(_frame_counts(ex.trace()), dtype=np.int64)
    return _stats_from(total.tolist(), frame, exs[0].mode)


# ------------------------------------------------------------------ in-engine collectives
class Communicator:
    """prx_comm (include/prx.h): a collectives table for in-engine sharded frames.

    nccl():        one rank of an NCCL communicator (libnccl loaded by _prx.so at run time);
    local_group(): `world` in-process communicators, one per host thread / shard.
    """

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self):
        self.close()

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            L.lib().prx_comm_destroy(self._h)
            self._h = None

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        L.check(L.lib().prx_comm_nccl_unique_id(buf))
        return bytes(buf)

    @classmethod
    def nccl(cls, unique_id: bytes, rank: int, world: int, device: int) -> "Communicator":
        buf = (C.c_uint8 * 128)(*unique_id)
        h = C.c_void_p()
        L.check(L.lib().prx_comm_nccl_create(buf, int(rank), int(world), int(device), C.byref(h)))
        return cls(h.value)

    @classmethod
    def local_group(cls, world: int) -> list:
        arr = (C.c_void_p * world)()
        L.check(L.lib().prx_comm_local_create(int(world), arr))
        return [cls(arr[r]) for r in range(world)]

    def collectives(self) -> L.Collectives:
        out = L.Collectives()
        L.check(L.lib().prx_comm_collectives(self._h, C.byref(out)))
        return out


def attach(engine: Engine, comm: Communicator) -> None:
    """Make `engine` (one rank's path shard) run sharded frames over `comm` in-engine."""
    L.check(L.lib().prx_engine_set_collectives(engine.handle, C.byref(comm.collectives())))
    engine._comm = comm  # keep the communicator alive as long as the engine uses it


class EngineGroup:
    """One process, `world` path shards (on `devices`; several may share one device), driven by
    the C++ group (prx_group_*, csrc/group.cpp): one persistent host thread per shard, the
    exchanges inside the engines over the local collectives backend (comm.cpp), so a sharded
    frame is each engine's own prx_run_frame with one host read-back.  Frames are
    bit-identical to one engine; the image is the sum of the per-shard splats (fp32 order
    differs across shards)."""

    def __init__(self, scene: Scene, devices: Sequence[int], **cfg):
        self.world = len(devices)
        self.scene = scene
        self.config = make_config(**cfg)
        devs = (C.c_int32 * self.world)(*devices)
        h = C.c_void_p()
        L.check(L.lib().prx_group_create(scene.handle, C.byref(self.config), devs, self.world, C.byref(h)))
        self._h = h
        self.engines = []
        for r in range(self.world):
            c = make_config(shard=shard_range(self.config.n_paths, r, self.world), device=devices[r], **cfg)
            self.engines.append(Engine._borrowed(L.lib().prx_group_engine(h, r), scene, c, self))

    def run_frame(self) -> L.FrameStats:
        st = L.FrameStats()
        L.check(L.lib().prx_group_run_frame(self._h, C.byref(st)))  # all-shard counters
        return st

    def splat(self, camera=None, radius: float = 0.25, mode: int = 1) -> np.ndarray:
        cam = camera if camera is not None else self.scene.describe().camera
        out = np.zeros((int(cam.height), int(cam.width), 3), dtype=np.float32)
        L.check(L.lib().prx_group_splat(self._h, C.byref(cam), float(radius), int(mode),
                                        out.ctypes.data_as(C.c_void_p)))
        return out

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            L.lib().prx_group_destroy(self._h)
        self._h = None
        self.engines = []

    def __del__(self):
        self.close()


class ShardedEngine:
    """User-facing sharded engine: this rank's slice of a multi-GPU path store, one process per
    GPU (torch.distributed initialised).  The exchanges run inside the engine over NCCL; the
    NCCL unique id travels through torch.distributed once."""

    def __init__(self, scene: Scene, rank: int, world: int, device: int = 0, group=None, **cfg):
        import torch.distributed as dist

        n = cfg.get("paths", 10000)
        self.config = make_config(shard=shard_range(n, rank, world), device=device, **cfg)
        self.engine = Engine(scene, self.config)
        self.comm = None
        if world > 1:
            obj = [Communicator.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            self.comm = Communicator.nccl(obj[0], rank, world, device)
            attach(self.engine, self.comm)

    def run_frame(self) -> dict:
        st = self.engine.run_frame()
        d = {k: getattr(st, k) for k in L.FrameStats.COUNTS}
        d.update(frame=st.frame, mode=L.MODE_NAMES[st.mode])
        return d

    def splat(self, camera=None, radius: float = 0.25, mode: int = 1) -> np.ndarray:
        return self.engine.splat(camera=camera, radius=radius, mode=mode)


class MultiGpuEngine(EngineGroup):
    """One process driving path shards on several GPUs (default: every visible device; shards
    share the device when there is one) -- the reference's single Engine object over N GPUs."""

    def __init__(self, scene: Scene, devices: Sequence[int] | None = None, **cfg):
        import torch

        devs = list(devices) if devices is not None else list(range(torch.cuda.device_count()))
        super().__init__(scene, devs, **cfg)

    def run_frame(self) -> dict:
        st = super().run_frame()
        d = {k: getattr(st, k) for k in L.FrameStats.COUNTS}
        d.update(frame=st.frame, mode=L.MODE_NAMES[st.mode])
        return d
