"""Sharded run_pipeline_on_scene: one process per GPU.

The reference parallelises propagate over initial hits (proj/src/tracer.cpp:476-533,
`parallel_for` + a merge in task order + a global κ) and refines candidates
independently (proj/src/pipeline.cpp:148-187). Here each rank is one shard:

1. ``pcr_shard_trace``: validate, build_grid and transmission_phase on every rank
   (all O(N) or O(n_IE), < 1 ms for C2), propagate over the initial hits
   ``t ≡ rank (mod world)`` of every TX with the rank's own first-κ;
2. the candidate rows (DFS key, group hash, candidate; ``csrc/shard_rows.cuh``) are
   all-gathered — the only data-path exchange of the trace stage;
3. ``pcr_shard_refine``: the global κ over all rows gives the reference's candidate
   list on every rank; the rank refines candidates ``i ≡ rank (mod world)``;
4. outcome rows and the summed work counters go to rank 0, whose
   ``pcr_shard_finish`` runs dedup + final order and returns the unsharded RunSummary.

The byte exchange is plain ``torch.distributed`` (NCCL on GPUs, gloo on CPU) over
uint8 tensors; the library never sees the transport.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import abi, pcray


def shard_of(index: int, world: int) -> int:
    """Owner of initial hit / candidate `index` under the cyclic split."""
    return index % world


def shard_indices(n: int, shard: int, world: int) -> range:
    """Indices a shard owns among n (tasks or candidates): shard, shard + world, ..."""
    return range(shard, n, world)


def all_gather_bytes(buf: torch.Tensor, group=None) -> torch.Tensor:
    """Concatenation, in rank order, of every rank's 1-D uint8 tensor (sizes may differ).
    NCCL moves device tensors directly; under gloo a device tensor is staged through
    host memory (gloo's all-gather is host-side)."""
    if buf.is_cuda and dist.get_backend(group) == "gloo":
        return all_gather_bytes(buf.cpu(), group).to(buf.device)
    world = dist.get_world_size(group)
    dev = buf.device
    size = torch.tensor([buf.numel()], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(size) for _ in range(world)]
    dist.all_gather(sizes, size, group=group)
    sizes = [int(s.item()) for s in sizes]
    cap = max(sizes) if sizes else 0
    if cap == 0:
        return torch.empty(0, dtype=torch.uint8, device=dev)
    padded = torch.zeros(cap, dtype=torch.uint8, device=dev)
    padded[: buf.numel()] = buf
    out = torch.empty(world * cap, dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(out, padded, group=group)
    return torch.cat([out[r * cap: r * cap + sizes[r]] for r in range(world)])


def gather_bytes(buf: torch.Tensor, dst: int = 0, group=None):
    """Concatenation in rank order of every rank's 1-D uint8 tensor on rank `dst` (None
    elsewhere): only the destination receives the bytes (the outcome rows go to the
    one rank that finishes)."""
    if buf.is_cuda and dist.get_backend(group) == "gloo":
        out = gather_bytes(buf.cpu(), dst, group)
        return None if out is None else out.to(buf.device)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    dev = buf.device
    size = torch.tensor([buf.numel()], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(size) for _ in range(world)]
    dist.all_gather(sizes, size, group=group)
    sizes = [int(x.item()) for x in sizes]
    cap = max(sizes) if sizes else 0
    if cap == 0:
        return torch.empty(0, dtype=torch.uint8, device=dev) if rank == dst else None
    padded = torch.zeros(cap, dtype=torch.uint8, device=dev)
    padded[: buf.numel()] = buf
    parts = [torch.empty(cap, dtype=torch.uint8, device=dev) for _ in range(world)] if rank == dst else None
    dist.gather(padded, parts, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([parts[r][: sizes[r]] for r in range(world)])


def sum_stats(stats: np.ndarray, group=None, device=None) -> np.ndarray:
    """Element-wise sum of every rank's pcr_shard_stats counters."""
    if dist.get_backend(group) == "gloo":
        device = None
    t = torch.tensor(stats.astype(np.int64), dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy().astype(np.uint64)


def _rows_tensor(n: int, row_bytes: int, device) -> torch.Tensor:
    return torch.empty(n * row_bytes, dtype=torch.uint8, device=device)


def run_pipeline_sharded(scene: pcray.DeviceScene, config: abi.RunConfig | None = None, group=None):
    """run_pipeline_on_scene across the ranks of `group` (one GPU each, scene resident on
    every rank). Returns the RunSummary dict on rank 0 and None elsewhere."""
    config = config or pcray.default_run_config()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    ctx = scene.ctx
    n, rb = pcray.shard_trace(scene, config, rank, world)
    rows = _rows_tensor(n, rb, dev)
    if n:
        pcray.shard_rows(ctx, rows.data_ptr())
    all_rows = all_gather_bytes(rows, group)
    torch.cuda.current_stream().synchronize()  # the library reads it on its own stream
    n_out, ob = pcray.shard_refine(scene, all_rows.data_ptr() if all_rows.numel() else 0, all_rows.numel() // rb)
    outs = _rows_tensor(n_out, ob, dev)
    if n_out:
        pcray.shard_outcomes(ctx, outs.data_ptr())
    totals = sum_stats(pcray.shard_stats(ctx), group, dev)
    all_outs = gather_bytes(outs, 0, group)
    torch.cuda.current_stream().synchronize()
    if rank != 0:
        return None
    return pcray.shard_finish(ctx, all_outs.data_ptr() if all_outs.numel() else 0, all_outs.numel() // ob, totals)


def build_grid_sharded(scene: pcray.DeviceScene, params=None, group=None) -> pcray.DeviceGrid:
    """build_grid across the ranks of `group`: every rank holds the scene,
    builds the part of its voxel range (about N / world points), the parts are
    all-gathered (NCCL: device to device over NVLink) and every rank assembles the
    whole grid — the unsharded grid bit for bit."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    nb = pcray.grid_part_build(scene, rank, world, params)
    part = torch.empty(nb, dtype=torch.uint8, device=dev)
    pcray.grid_part_copy(scene.ctx, part.data_ptr())
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev if dist.get_backend(group) != "gloo" else "cpu")
             for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([nb], dtype=torch.int64, device=sizes[0].device), group=group)
    sizes = [int(x.item()) for x in sizes]
    allp = all_gather_bytes(part, group)
    torch.cuda.current_stream().synchronize()
    offsets = np.concatenate([[0], np.cumsum(sizes)[:-1]]).tolist()
    return pcray.grid_assemble(scene.ctx, allp.data_ptr(), offsets, sizes)


def build_grid_sharded_local(scene, params=None, n_shards: int = 2, device: int = 0) -> pcray.DeviceGrid:
    """All shards of build_grid_sharded in one process on one GPU, one after another,
    the parts concatenated on the device (proves the split exact without more GPUs)."""
    dev = torch.device("cuda", device)
    ds = scene if isinstance(scene, pcray.DeviceScene) else pcray.DeviceScene(scene, pcray.Context(device))
    parts, sizes = [], []
    for r in range(n_shards):
        nb = pcray.grid_part_build(ds, r, n_shards, params)
        t = torch.empty(nb, dtype=torch.uint8, device=dev)
        pcray.grid_part_copy(ds.ctx, t.data_ptr())
        parts.append(t)
        sizes.append(nb)
    allp = torch.cat(parts)
    torch.cuda.synchronize(dev)
    offsets = np.concatenate([[0], np.cumsum(sizes)[:-1]]).tolist()
    return pcray.grid_assemble(ds.ctx, allp.data_ptr(), offsets, sizes)


def run_pipeline_sharded_local(scene, config: abi.RunConfig | None = None, n_shards: int = 2,
                               order=None, device: int = 0, times: dict | None = None):
    """All shards of run_pipeline_sharded in one process on one GPU, one context each,
    run one after another (no shard waits on another): the exchange is a device-side
    concatenation in `order` (default rank order). Used to prove the split exact
    without more GPUs."""
    config = config or pcray.default_run_config()
    order = list(order) if order is not None else list(range(n_shards))
    dev = torch.device("cuda", device)
    ctxs = [pcray.Context(device) for _ in range(n_shards)]
    scenes = [pcray.DeviceScene(scene, c) for c in ctxs]
    rows, rb = [], 0
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t_trace, t_refine = [], []
    for r in range(n_shards):
        stream = torch.cuda.ExternalStream(pcray.stream_ptr(ctxs[r]))
        a, b = ev(), ev()
        a.record(stream)
        n, rb = pcray.shard_trace(scenes[r], config, r, n_shards)
        b.record(stream)
        b.synchronize()
        t_trace.append(a.elapsed_time(b) / 1e3)
        t = _rows_tensor(n, rb, dev)
        if n:
            pcray.shard_rows(ctxs[r], t.data_ptr())
        rows.append(t)
    all_rows = torch.cat([rows[r] for r in order])
    torch.cuda.synchronize(dev)  # the library reads it on its own streams
    outs, ob, totals = [], 0, np.zeros(len(abi.SHARD_STATS_FIELDS), dtype=np.uint64)
    for r in range(n_shards):
        stream = torch.cuda.ExternalStream(pcray.stream_ptr(ctxs[r]))
        a, b = ev(), ev()
        a.record(stream)
        n_out, ob = pcray.shard_refine(scenes[r], all_rows.data_ptr() if all_rows.numel() else 0,
                                       all_rows.numel() // rb)
        b.record(stream)
        b.synchronize()
        t_refine.append(a.elapsed_time(b) / 1e3)
        t = _rows_tensor(n_out, ob, dev)
        if n_out:
            pcray.shard_outcomes(ctxs[r], t.data_ptr())
        outs.append(t)
        totals = totals + pcray.shard_stats(ctxs[r])
    all_outs = torch.cat([outs[r] for r in order])
    torch.cuda.synchronize(dev)
    if times is not None:  # per-shard device seconds of the trace and refine calls (load balance)
        times["trace"] = t_trace
        times["refine"] = t_refine
    return pcray.shard_finish(ctxs[0], all_outs.data_ptr() if all_outs.numel() else 0, all_outs.numel() // ob,
                              totals)
