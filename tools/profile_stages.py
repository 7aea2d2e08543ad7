"""Run one config end to end on the GPU and print the summary, stage timings and
per-kernel CUDA-event totals (development aid; not part of the measured bench)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2402_13747_b200 import abi, pcray, scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--mi", type=int, default=None)
    ap.add_argument("--md", type=int, default=None)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--oracle", action="store_true", help="also run the CPU reference and compare counts")
    args = ap.parse_args()
    t = time.time()
    scene, cfg = scenes.build_scene(args.config)
    run = dict(cfg.run)
    if args.mi is not None:
        run["max_interactions"] = args.mi
    if args.md is not None:
        run["max_diffractions"] = args.md
    print(f"scene {args.config}: {scene.n_points} points, {len(scene.tx)} TX, {len(scene.rx)} RX, "
          f"{len(scene.edges)} edges, gen {time.time() - t:.2f}s, run {run}", flush=True)
    ds = pcray.DeviceScene(scene)
    conf = abi.default_run_config(**run)
    for rep in range(args.reps):
        pcray.set_profiling(rep == args.reps - 1)
        t = time.time()
        s = pcray.run_pipeline_device(ds, conf)
        wall = time.time() - t
        print(f"rep {rep}: wall {wall:.3f}s timings {[(a, round(b, 4)) for a, b in s['timings']]}", flush=True)
    kt = pcray.kernel_times()
    pcray.set_profiling(False)
    out = {k: s[k] for k in ["ie_count", "grid_dims", "coarse_paths", "refined_paths", "rejected", "exact_paths",
                             "transmission_rays", "cone_traces", "visibility_tests", "refine_iterations", "refine_trials", "refine_marches", "walk_cells", "walk_ies"]}
    print(json.dumps(out))
    tot = sum(v[0] for v in kt.values())
    for k, (ms, n) in sorted(kt.items(), key=lambda kv: -kv[1][0]):
        print(f"  {k:16s} {ms:10.3f} ms  {n:6d} launches  {100 * ms / max(tot, 1e-9):5.1f}%")
    if args.oracle:
        from oracle import ref

        t = time.time()
        r = ref.run_pipeline_on_scene(ref.RefScene(scene), ref.default_run_config(**run))
        print(f"oracle wall {time.time() - t:.2f}s timings {[(a, round(b, 3)) for a, b in r['timings']]}")
        for k in ["ie_count", "coarse_paths", "refined_paths", "rejected", "exact_paths"]:
            print(f"  {k}: gpu {s[k]} ref {r[k]} {'OK' if s[k] == r[k] else 'MISMATCH'}")


if __name__ == "__main__":
    main()
