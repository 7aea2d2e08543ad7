"""Golden digests of the full contract runs (SURVEY.md §8.0 C2 at 4 / 1 and C2 at
depth 3), generated from the ORACLE (oracle/_ref: the unmodified reference compiled
here) — TEST INFRASTRUCTURE ONLY.

For each config the reference runs through its own API on the whole scene:
  * build_grid, then per TX transmission_phase + propagate on every initial hit
    (tracer.cpp:207-255, 476-533): the coarse candidate list (LOS rows first, as
    run_pipeline_on_scene orders them, pipeline.cpp:136-146);
  * refine_path on every candidate (refine.cpp:189-286): reasons + refined geometry;
  * run_pipeline_on_scene under the counting build (oracle/ref_count.cpp): RunSummary
    counts, the final (deduplicated, sorted) paths, and the number of
    voxel_cone_trace / segment_visible calls.
Digests (tests/digest.py) of the three tables and the counts go to
tests/golden/contract_<config>.json; tests/test_contract_gpu.py recomputes them from
the CUDA path. The full depth-4 run takes ~25 min on 8 host cores.

  python tests/golden/make_contract_golden.py [C2d3 C2 ...]
"""
from __future__ import annotations

import json
import math
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import digest  # noqa: E402
from oracle import bench_ref, ref  # noqa: E402
from paper_2402_13747_b200 import abi, scenes  # noqa: E402


def candidates_and_outcomes(scene, run, threads):
    cfg = ref.default_run_config(**run)
    tp = abi.trace_params(cfg.max_interactions, cfg.kappa, cfg.cone_apex_angle_deg * math.pi / 180.0,
                          cfg.diffraction_ray_count, cfg.max_diffractions)
    rp = abi.refine_params(cfg.delta, cfg.rho, cfg.step_size, bool(cfg.fresnel_enabled))
    rs = ref.RefScene(scene)
    grid = ref.build_grid(rs, abi.voxel_params(cfg.voxel_size_m, cfg.division_factor))
    los_parts, prop_parts, n_hits = [], [], 0
    for t in range(len(scene.tx)):
        los, hits = ref.transmission_phase(grid, rs, t, tp)
        n_hits += hits["n"]
        los_parts.append(los)
        prop_parts.append(ref.propagate(grid, rs, t, hits, tp, thread_count=threads))
    # run_pipeline_on_scene's candidate order: per TX, LOS then propagated (pipeline.cpp:136-146)
    parts = []
    for a, b in zip(los_parts, prop_parts):
        parts += [a, b]
    cands = bench_ref.concat_paths(parts)
    out = ref.refine_batch(grid, rs, cands, rp, thread_count=threads)
    return cands, out, n_hits


def main(names):
    threads = os.cpu_count() or 1
    for name in names:
        scene, cfg = scenes.build_scene(name)
        run = dict(cfg.run)
        slots = run["max_interactions"]
        t0 = time.time()
        cands, outs, n_hits = candidates_and_outcomes(scene, run, threads)
        t1 = time.time()
        with ref.counting() as c:
            c.read(reset=True)
            s = ref.run_pipeline_on_scene(ref.RefScene(scene), ref.default_run_config(**run))
            cone, vis = c.read(reset=True)
        t2 = time.time()
        doc = {
            "config": name, "run": run, "points": scene.n_points, "generated_by": "tests/golden/make_contract_golden.py",
            "oracle_threads": threads, "oracle_seconds": {"trace+refine": t1 - t0, "pipeline(counting)": t2 - t1},
            "initial_hits": n_hits,
            "summary": {k: s[k] for k in ["ie_count", "coarse_paths", "refined_paths", "rejected", "exact_paths", "hash"]},
            "cone_traces": cone, "visibility_tests": vis,
            "transmission_rays": s["ie_count"] * len(scene.tx),
            "candidates": digest.candidates_digest(cands, slots),
            "outcomes": digest.outcomes_digest(outs, slots),
            "paths": digest.paths_digest(s["paths"], slots),
        }
        assert doc["candidates"]["n"] == s["coarse_paths"]
        path = os.path.join(HERE, f"contract_{name}.json")
        with open(path, "w") as f:
            json.dump(doc, f, indent=1)
        print(f"{name}: {cands['n']} candidates, {s['exact_paths']} exact paths, {cone} cone traces, "
              f"{t2 - t0:.0f} s -> {path}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C2d3", "C2"])
