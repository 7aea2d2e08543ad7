"""Every BASELINE.json config on one B200, beside the reference on
the host cores. Writes one JSON document (default profiles/configs_r02.json).

  C1-C4  full pipeline (run_pipeline_device, scene resident): step seconds, launched
         Mrays/s, exact paths/s, candidates refined/s, stage and kernel split. The CPU
         arm runs the reference (oracle/_ref) on a bounded task-stride sample of the
         same scene (oracle/bench_ref.py) and reports rates.
  C5     voxelization sweep on the C3 geometry: 1M-100M points x (voxel, D_v);
         build_grid + compute_march_distances device time, algorithmic bytes
         56 N + 96 n_IE + 16 cells, GB/s against MEASURED_PEAKS.json hbm_gbs; the
         reference's build_grid timed at the sizes it finishes in seconds.

Development/measurement tool: bench.py stays the driver's single-config contract.
  python tools/bench_configs.py [--configs C1,C2,C3,C4] [--c5] [--cpu-budget 15]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2402_13747_b200 import abi, pcray, scenes  # noqa: E402


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    return 6650.0, "fallback"


def gpu_pipeline(name, reps, mi=None):
    import torch

    scene, cfg = scenes.build_scene(name)
    run = dict(cfg.run)
    if mi is not None:
        run["max_interactions"] = mi
    ctx = pcray.Context.default()
    ds = pcray.DeviceScene(scene, ctx)
    conf = abi.default_run_config(**run)
    stream = torch.cuda.ExternalStream(pcray.stream_ptr(ctx))
    big = name in ("C2", "C3", "C4", "C2np")
    if not big:
        pcray.run_pipeline_device(ds, conf)  # warm-up (first-call allocations; noise next to C3/C4 steps)
    ms, s = [], None
    pcray.kernel_times(reset=True, ctx=ctx)
    pcray.set_profiling(True, ctx)
    for _ in range(1 if big else reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        s = pcray.run_pipeline_device(ds, conf)
        b.record(stream)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    kt = pcray.kernel_times(reset=True, ctx=ctx)
    pcray.set_profiling(False, ctx)
    step = sum(ms) / len(ms) / 1e3
    rays = s["transmission_rays"] + s["cone_traces"]
    tot = sum(v[0] for v in kt.values()) or 1.0
    return scene, run, {
        "config": name, "note": cfg.note, "points": scene.n_points, "tx": int(len(scene.tx)),
        "rx": int(len(scene.rx)), "edges": int(len(scene.edges)), "run": run, "step_s": step,
        "mrays_per_s": rays / step / 1e6, "exact_paths_per_s": s["exact_paths"] / step,
        "candidates_per_s": s["coarse_paths"] / step, "rays": rays,
        "counts": {k: s[k] for k in ["ie_count", "coarse_paths", "refined_paths", "exact_paths", "cone_traces",
                                     "visibility_tests", "refine_iterations"]},
        "rejected": list(s["rejected"]), "stage_s": dict(s["timings"]),
        "kernel_share": {k: round(v[0] / tot, 4) for k, v in sorted(kt.items(), key=lambda kv: -kv[1][0])},
    }


def cpu_pipeline(scene, run, budget, probe):
    from oracle import bench_ref

    t = time.time()
    stride = bench_ref.choose_stride(scene, run, budget, probe_stride=probe)
    m = bench_ref.measure(scene, run, budget_s=budget, stride=stride)
    return {"kind": "reference", "cores": m["threads"], "task_stride": m["stride"],
            "mrays_per_s": m["mrays_per_s"], "exact_paths_per_s": m["exact_paths_per_s"],
            "candidates_per_s": m["candidates_per_s"], "sample_rays": m["rays"], "sample_s": m["seconds"],
            "tool_s": time.time() - t}


def c5_sweep(cpu_max_points):
    import torch

    peak, src = hbm_peak()
    base = scenes.config("C3")
    out = []
    ctx = pcray.Context.default()
    stream = torch.cuda.ExternalStream(pcray.stream_ptr(ctx))
    for target in [1_000_000, 3_000_000, 10_000_000, 30_000_000, 100_000_000]:
        scene = scenes.scene_from_planar(base.planar, scenes.scaled_density(base, target), base.seed)
        ds = pcray.DeviceScene(scene, ctx)
        for vs, dv in [(1.0, 2), (0.5, 1), (0.5, 2), (0.5, 4), (0.5, 8), (0.25, 2)]:
            vp = abi.voxel_params(vs, dv)
            try:
                g = pcray.build_grid(ds, vp)  # warm-up
                pcray.compute_march_distances(g)
                del g
            except pcray.PcrError as e:
                out.append({"points": scene.n_points, "voxel": vs, "dv": dv, "error": str(e)})
                continue
            ms = []
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                g = pcray.build_grid(ds, vp)
                pcray.compute_march_distances(g)
                b.record(stream)
                b.synchronize()
                ms.append(a.elapsed_time(b))
            gd = g.to_dict()
            n_ie, n_cells = len(gd["ie_kind"]), len(gd["cell_march"])
            del g
            nbytes = 56 * scene.n_points + 96 * n_ie + 16 * n_cells
            t = min(ms) / 1e3
            row = {"points": scene.n_points, "voxel": vs, "dv": dv, "ies": n_ie, "cells": n_cells, "gpu_s": t,
                   "gb_per_s": nbytes / t / 1e9, "hbm_frac": nbytes / t / 1e9 / peak, "algorithmic_bytes": nbytes,
                   "mpoints_per_s": scene.n_points / t / 1e6}
            if scene.n_points <= cpu_max_points and (vs, dv) == (0.5, 2):
                try:
                    from oracle import ref

                    rs = ref.RefScene(scene)
                    t0 = time.perf_counter()
                    rg = ref.build_grid(rs, vp)  # includes compute_march_distances
                    row["cpu_reference_s"] = time.perf_counter() - t0
                    del rg
                except Exception as e:  # oracle is test infrastructure; say why it is missing
                    row["cpu_reference_s"] = f"unavailable: {e}"
            out.append(row)
            print(json.dumps(row), flush=True)
        del ds
    return {"peak_gbs": peak, "peak_source": src, "rows": out}


def ply_ingest(points, cpu):
    """Binary PLY -> device scene (pcr_scene_load_ply): file bytes / wall seconds (file in
    the page cache after a first read), beside the reference's load_point_cloud."""
    import tempfile

    import numpy as np

    rng = np.random.default_rng(1)
    rows = np.zeros(points, dtype=[("x", "<f4"), ("y", "<f4"), ("z", "<f4"), ("nx", "<f4"), ("ny", "<f4"),
                                   ("nz", "<f4"), ("label", "<u4")])
    for k in ["x", "y", "z"]:
        rows[k] = rng.uniform(0, 100, points)
    rows["nz"] = 1.0
    rows["label"] = rng.integers(0, 1000, points)
    path = os.path.join(tempfile.gettempdir(), f"pcr_ingest_{points}.ply")
    with open(path, "wb") as f:
        f.write(b"ply\nformat binary_little_endian 1.0\nelement vertex %d\n" % points)
        for k in ["x", "y", "z", "nx", "ny", "nz"]:
            f.write(b"property float %s\n" % k.encode())
        f.write(b"property uint label\nend_header\n")
        rows.tofile(f)
    size = os.path.getsize(path)
    ctx = pcray.Context.default()
    pcray.DeviceScene.from_ply(path, ctx=ctx, host_mirror=False)  # warm: page cache, allocator
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        ds = pcray.DeviceScene.from_ply(path, ctx=ctx, host_mirror=False)
        ts.append(time.perf_counter() - t)
        del ds
    row = {"points": points, "file_bytes": size, "gpu_s": min(ts), "gb_per_s": size / min(ts) / 1e9,
           "note": "wall time of pcr_scene_load_ply (file in the page cache)"}
    if cpu:
        try:
            from oracle import ref

            t = time.perf_counter()
            ref.load_point_cloud(path)
            row["cpu_reference_s"] = time.perf_counter() - t
        except Exception as e:
            row["cpu_reference_s"] = f"unavailable: {e}"
    os.unlink(path)
    print(json.dumps(row), flush=True)
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2d3,C2,C3")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--c5", action="store_true")
    ap.add_argument("--ply", type=int, default=0, help="PLY ingest benchmark with this many points")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--cpu-c5-max", type=int, default=10_000_000)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "configs_r02.json"))
    args = ap.parse_args()
    doc = {"device": None, "pipelines": [], "c5": None}
    try:
        import torch

        doc["device"] = torch.cuda.get_device_name(0)
    except Exception:
        pass
    for name in [c for c in args.configs.split(",") if c]:
        scene, run, row = gpu_pipeline(name, args.reps)
        print(json.dumps(row), flush=True)
        if not args.no_cpu:
            try:
                row["cpu"] = cpu_pipeline(scene, run, args.cpu_budget, probe=64 if name in ("C1", "C2", "C2d3") else 4096)
            except Exception as e:
                row["cpu"] = {"kind": "reference", "error": str(e)}
            print(json.dumps(row["cpu"]), flush=True)
        doc["pipelines"].append(row)
        with open(args.out, "w") as f:
            json.dump(doc, f, indent=1)
    if args.ply:
        doc["ply_ingest"] = ply_ingest(args.ply, not args.no_cpu)
        with open(args.out, "w") as f:
            json.dump(doc, f, indent=1)
    if args.c5:
        doc["c5"] = c5_sweep(0 if args.no_cpu else args.cpu_c5_max)
        with open(args.out, "w") as f:
            json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
