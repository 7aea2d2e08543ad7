"""CPU arm of bench.py — BENCH/TEST INFRASTRUCTURE ONLY.

Times the unmodified reference (oracle/_ref) on the host cores through its own
public API on a deterministic task subset of the bench workload:
build_grid, transmission_phase on every IE of every TX, propagate on every
`stride`-th initial hit, refine_path on the resulting candidates (LOS rows pass
through as in run_pipeline_on_scene). Launched rays are counted with the
instrumented build (oracle/ref_count.cpp) in a separate, untimed run of the same
sample, on the same definition as the GPU arm: sum over TX of n_IE transmission
rays + voxel_cone_trace invocations.
"""
from __future__ import annotations

import math
import os
import time

import numpy as np

from paper_2402_13747_b200 import abi

from . import ref


INTERACTION_KEYS = {"kind", "position", "label", "normal", "ie_index", "edge_index"}


def concat_paths(parts):
    parts = [p for p in parts if p["n"] > 0]
    if not parts:
        return {"n": 0, "stride": 1}
    s = max(p["stride"] for p in parts)
    out = {"n": sum(p["n"] for p in parts), "stride": s}
    for k, v in parts[0].items():
        if not isinstance(v, np.ndarray):
            continue
        arrs = []
        for p in parts:
            a = p[k]
            if k in INTERACTION_KEYS and a.shape[1] != s:
                pad = np.zeros((a.shape[0], s) + a.shape[2:], a.dtype)
                pad[:, : a.shape[1]] = a
                a = pad
            arrs.append(a)
        out[k] = np.concatenate(arrs)
    return out


def subset_hits(h, stride):
    if stride <= 1:
        return h
    out = {"n": len(range(0, h["n"], stride))}
    for k, v in h.items():
        if isinstance(v, np.ndarray):
            out[k] = np.ascontiguousarray(v[::stride])
    return out


def run_sample(scene, run: dict, stride: int = 1, threads: int = 0):
    """One timed pass of the reference over the sample; returns counts and seconds."""
    cfg = ref.default_run_config(**run)
    vp = abi.voxel_params(cfg.voxel_size_m, cfg.division_factor)
    tp = abi.trace_params(cfg.max_interactions, cfg.kappa, cfg.cone_apex_angle_deg * math.pi / 180.0,
                          cfg.diffraction_ray_count, cfg.max_diffractions)
    rp = abi.refine_params(cfg.delta, cfg.rho, cfg.step_size, bool(cfg.fresnel_enabled))
    rs = ref.RefScene(scene)
    n_tx = len(rs.scene.tx_id)
    t0 = time.perf_counter()
    grid = ref.build_grid(rs, vp)
    parts = []
    n_hits = 0
    for t in range(n_tx):
        los, hits = ref.transmission_phase(grid, rs, t, tp)
        sub = subset_hits(hits, stride)
        n_hits += sub["n"]
        parts += [los, ref.propagate(grid, rs, t, sub, tp, thread_count=threads)]
    cands = concat_paths(parts)
    # refine_path + the pipeline's dedup: "exact" counts what RunSummary::exact_paths counts
    # (pipeline.cpp:181-208), the same definition as the GPU arm's exact_paths
    exact = ref.refine_dedup_count(grid, rs, cands, rp, thread_count=threads,
                                   carrier_frequency_hz=cfg.carrier_frequency_hz) if cands["n"] else 0
    seconds = time.perf_counter() - t0
    n_ies = len(grid.to_dict()["ie_kind"])
    return {"seconds": seconds, "candidates": int(cands["n"]), "exact": int(exact),
            "transmission_rays": n_ies * n_tx, "initial_hits_traced": n_hits, "stride": stride}


def count_rays(scene, run: dict, stride: int = 1, threads: int = 0):
    with ref.counting() as c:
        c.read(reset=True)
        r = run_sample(scene, run, stride, threads)
        cone, vis = c.read(reset=True)
    r["cone_traces"] = cone
    r["visibility_tests"] = vis
    return r


def choose_stride(scene, run: dict, budget_s: float, probe_stride: int = 64, threads: int = 0) -> int:
    """Smallest task stride whose sample should take about budget_s seconds."""
    probe = run_sample(scene, run, probe_stride, threads)
    est_full = probe["seconds"] * probe_stride
    return max(1, int(math.ceil(est_full / max(budget_s, 1e-3))))


def measure(scene, run: dict, budget_s: float = 20.0, threads: int = 0, stride: int | None = None):
    """Bounded CPU baseline: Mrays/s, exact paths/s and candidates refined/s of the reference."""
    threads = threads or (os.cpu_count() or 1)
    if stride is None:
        stride = choose_stride(scene, run, budget_s, threads=threads)
    counted = count_rays(scene, run, stride, threads)
    timed = run_sample(scene, run, stride, threads)
    rays = counted["transmission_rays"] + counted["cone_traces"]
    return {
        "seconds": timed["seconds"], "stride": stride, "threads": threads, "rays": rays,
        "mrays_per_s": rays / timed["seconds"] / 1e6,
        "exact_paths_per_s": timed["exact"] / timed["seconds"],
        "candidates_per_s": timed["candidates"] / timed["seconds"],
        "counts": {k: counted[k] for k in ["transmission_rays", "cone_traces", "visibility_tests", "candidates",
                                           "exact", "initial_hits_traced"]},
    }
