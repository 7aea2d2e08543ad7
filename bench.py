#!/usr/bin/env python
"""bench.py — launched Mrays/s and exact paths/s of the B200 point-cloud ray launcher.

Workload (BASELINE.json configs[1]): synthetic indoor office,
1,000,902 labeled points sampled with the reference's rectangle sampler, 1 TX /
64 RX, 40 diffraction edges, max 4 interactions incl. <= 1 diffraction ("3 reflections +
1 diffraction"; SURVEY.md §8.0 fixes C2 at max_interactions 4 / max_diffractions 1), every other
RunConfig field at the paper's Table-1 defaults. A step is one full pass of the hot
path over the scene: validate -> voxelize -> transmission + propagation -> refinement
-> dedup (run_pipeline_on_scene semantics, outputs identical to the reference).

  value  = launched rays / step time (inputs resident in HBM: pcr_run_pipeline_device)
  e2e    = same metric through pcr_run_pipeline_on_scene with pinned host buffers,
           host<->device copies inside the timed region
  rays   = sum_TX n_IE transmission rays + voxel_cone_trace invocations

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

with open(os.path.join(ROOT, "BASELINE.json")) as _f:
    BASELINE = json.load(_f)
METRIC = BASELINE["metric"]
CONFIG = "C2"


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = tempfile.mktemp(prefix="pcr_clocks_", suffix=".csv")

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()
        return False

    def summary(self):
        if not self.proc or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax.append(float(parts[2]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------------------
# algorithmic work per kernel (SURVEY §8d units; FP64 op counts read off the kernels)
FLOP_TRIAL_PER_NODE = 26.0   # parameter update + node point + one chain segment
FLOP_TRIAL_BASE = 10.0       # closing segment to RX
FLOP_MARCH = 60.0            # planar march_segment (window, two SDF samples, snap)
FLOP_ITER_PER_NODE = 95.0    # gradient (40) + polish (20) + local_frame (20) + new point/segment (15)
BYTES_CELL = 16.0            # int4 VoxelCell record
BYTES_IE = 72.0              # IE label + sphere (32) + reception point (32) + meta


def measured_traffic(kernel):
    """DRAM bytes per launch of `kernel` from a committed ncu capture (profiles/ncu_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)[kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


def roofline(kernel, ms_total, launches, summary, peaks, peaks_kind, fp64_tflops):
    if kernel == "refine":
        # per-path node counts weight the per-node terms (counted by the kernel:
        # refine_trial_nodes = sum over trials of d, refine_iter_nodes = sum over iterations of d)
        flops = (summary["refine_trial_nodes"] * FLOP_TRIAL_PER_NODE + summary["refine_trials"] * FLOP_TRIAL_BASE
                 + summary["refine_marches"] * FLOP_MARCH
                 + summary["refine_iter_nodes"] * FLOP_ITER_PER_NODE)
        per_launch = flops / max(launches, 1)
        achieved = per_launch / (ms_total / max(launches, 1) * 1e-3) / 1e12
        return {"bound": "fp64", "kernel": kernel, "achieved": achieved, "peak": fp64_tflops, "unit": "TFLOP/s",
                "frac": achieved / fp64_tflops if fp64_tflops else None, "traffic": measured_traffic(kernel),
                "traffic_note": "DRAM bytes per launch (ncu, profiles/ncu_traffic.json): per-lane local memory (path state, call frames); "
                                "the kernel's algorithmic inputs are L2-resident",
                "algorithmic_per_launch": per_launch, "avg_launch_ms": ms_total / max(launches, 1),
                "peak_source": "in-run non-FMA FP64 probe (pcr_fp64_probe); MEASURED_PEAKS.json has no FP64 figure"}
    # traversal kernels: bytes of cell and IE records the walk reads
    nbytes = summary["walk_cells"] * BYTES_CELL + summary["walk_ies"] * BYTES_IE
    per_launch = nbytes / max(launches, 1)
    achieved = per_launch / (ms_total / max(launches, 1) * 1e-3) / 1e9
    peak = peaks["hbm_gbs"]
    return {"bound": "hbm", "kernel": kernel, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": None, "algorithmic_per_launch": per_launch,
            "avg_launch_ms": ms_total / max(launches, 1), "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peaks_kind})"}


# ---------------------------------------------------------------------------------------------
def reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU implementation (oracle/_ref) on this host."""
    if rank != 0:
        return 0
    from oracle import bench_ref
    from paper_2402_13747_b200 import scenes

    scene, cfg = scenes.build_scene(CONFIG)
    threads = os.cpu_count() or 1
    budget = max(5.0, 150.0 / max(1, args.steps + 1))
    stride = bench_ref.choose_stride(scene, cfg.run, budget, threads=threads)
    counted = bench_ref.count_rays(scene, cfg.run, stride, threads)
    rays = counted["transmission_rays"] + counted["cone_traces"]
    for _ in range(args.warmup):  # bounded warm-up samples (CPU needs none; contract keeps W)
        bench_ref.run_sample(scene, cfg.run, max(stride, 64), threads)
    secs, exact, cands = [], 0, 0
    for _ in range(args.steps):
        r = bench_ref.run_sample(scene, cfg.run, stride, threads)
        secs.append(r["seconds"])
        exact += r["exact"]
        cands += r["candidates"]
    total = sum(secs)
    value = rays * args.steps / total / 1e6
    sample = (f"{CONFIG}: build_grid + transmission_phase (all {counted['transmission_rays']} IE rays) + "
              f"propagate on every {stride}-th initial hit + refine_path on the resulting "
              f"{counted['candidates']} candidates; {rays} launched rays per step")
    line = {"metric": METRIC, "value": value, "unit": "Mrays/s", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C2 synthetic office, 3 reflections + 1 diffraction = max_interactions 4 / "
                                   "max_diffractions 1 (SURVEY.md §8.0)", "points": scene.n_points,
                       "tx": 1, "rx": 64, "max_interactions": cfg.run["max_interactions"],
                       "max_diffractions": cfg.run["max_diffractions"], "task_stride": stride},
            "exact_paths_per_s": exact / total, "candidates_refined_per_s": cands / total,
            "cpu_baseline": {"value": value, "unit": "Mrays/s", "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": "Mrays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def b200_arm(args, rank, world, local_rank):
    import numpy as np
    import torch

    from paper_2402_13747_b200 import abi, pcray, scenes, shard

    # one GPU per rank; --backend gloo on a box with fewer GPUs than ranks (a dry run of
    # the N > 1 code path) places ranks round-robin — gloo's host-side collectives never
    # make one rank's kernels wait on another's
    dev = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(args.backend)

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if args.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if args.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    scene, cfg = scenes.build_scene(CONFIG)
    ctx = pcray.Context(dev)
    pcray.Context._default = ctx
    conf = abi.default_run_config(**cfg.run)
    ds = pcray.DeviceScene(scene, ctx)
    stream = torch.cuda.ExternalStream(pcray.stream_ptr(ctx))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2

    def timed_steps(fn, k, profile=False):
        """k steps, L2 flushed before each (outside the events); device time via events."""
        ms, outs = [], []
        pcray.kernel_times(reset=True, ctx=ctx)
        pcray.set_profiling(profile, ctx)
        l0 = pcray.kernel_launches()
        t0 = pcray.transfer_bytes()
        for _ in range(k):
            flush.zero_()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            outs.append(fn())
            b.record(stream)
            b.synchronize()
            ms.append(a.elapsed_time(b))
        launches = pcray.kernel_launches() - l0
        t1 = pcray.transfer_bytes()
        kt = pcray.kernel_times(reset=True, ctx=ctx)
        pcray.set_profiling(False, ctx)
        return ms, outs, launches, (t1[0] - t0[0], t1[1] - t0[1]), kt

    # N = 1: the whole pipeline on one device. N > 1: one shard per rank (
    # shard.py): the same scene and total work, split by initial hit and by candidate,
    # rows exchanged over NCCL — strong scaling, rank 0 holds the RunSummary.
    if world > 1:
        def step():
            return shard.run_pipeline_sharded(ds, conf)
    else:
        def step():
            return pcray.run_pipeline_device(ds, conf)

    for _ in range(args.warmup):
        step()
    # kernel shares from one profiled step outside the timed region (events around every
    # launch would add host work to the timed steps)
    _, _, _, _, kshares = timed_steps(step, 1, profile=1)
    barrier()
    with ClockSampler(dev) as clocks:
        barrier()
        # timed steps: events only around the refine launch (the roofline's kernel, one
        # launch per step) — its average duration over the timed region
        ms, outs, launches, _, ktimes = timed_steps(step, args.steps, profile=2)
        barrier()
    step_ms = max_over_ranks(sum(ms)) / args.steps
    launches = int(sum_over_ranks(launches))
    s0 = outs[-1]
    if world > 1:
        own = dict(zip(abi.SHARD_STATS_FIELDS, (int(x) for x in pcray.shard_stats(ctx))))
    else:
        own = s0
    rays = s0["transmission_rays"] + s0["cone_traces"] if rank == 0 else 0
    value = rays / (step_ms * 1e-3) / 1e6
    exact_per_s = (s0["exact_paths"] if rank == 0 else 0) / (step_ms * 1e-3)
    cand_per_s = (s0["coarse_paths"] if rank == 0 else 0) / (step_ms * 1e-3)
    clk = clocks.summary()

    # e2e: host buffers (pinned), copies inside the timed region, through the public C-ABI call
    pin = {}
    for name in ["position", "normal", "label", "edges", "edge_label", "tx", "tx_id", "rx", "rx_id"]:
        a = np.ascontiguousarray(getattr(scene, name))
        t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
        t.numpy()[...] = a
        pin[name] = t.numpy()
    host_scene = abi.Scene(pin["position"], pin["normal"], pin["label"], pin["edges"], pin["edge_label"], pin["tx"],
                           pin["tx_id"], pin["rx"], pin["rx_id"], scene.carrier_frequency_hz)
    if world > 1:
        def e2e_step():  # scene upload from pinned host memory + sharded run + result on rank 0's host
            return shard.run_pipeline_sharded(pcray.DeviceScene(host_scene, ctx), conf)
    else:
        def e2e_step():
            return pcray.run_pipeline_on_scene(host_scene, conf, ctx)
    e2e_step()
    barrier()
    e_steps = min(args.steps, 5)  # a full C2 step is ~9 s; 5 host-buffer steps bound the run time
    e_ms, e_outs, _, (h2d, d2h), _ = timed_steps(e2e_step, e_steps)
    e_step = max_over_ranks(sum(e_ms)) / e_steps
    e_value = rays / (e_step * 1e-3) / 1e6

    # parity self-check of the timed runs: identical summaries step to step
    for s in outs + e_outs:
        if s is not None:
            assert s["exact_paths"] == s0["exact_paths"] and s["coarse_paths"] == s0["coarse_paths"]

    peaks, peaks_kind = measured_peaks()
    fp64 = pcray.fp64_probe(ctx)
    dom = max(ktimes.items(), key=lambda kv: kv[1][0]) if ktimes else ("none", (0.0, 1))
    rl = roofline(dom[0], dom[1][0] / args.steps, max(1, dom[1][1] // args.steps), own, peaks, peaks_kind, fp64)
    total_k = sum(v[0] for v in kshares.values())
    shares = {k: round(v[0] / total_k, 4) for k, v in sorted(kshares.items(), key=lambda kv: -kv[1][0])}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import bench_ref

            m = bench_ref.measure(scene, cfg.run, budget_s=args.cpu_budget)
            cpu = {"value": m["mrays_per_s"], "unit": "Mrays/s", "cores": m["threads"], "kind": "reference",
                   "sample": (f"{CONFIG} reference API (oracle/_ref): build_grid + transmission_phase on all "
                              f"{m['counts']['transmission_rays']} IEs + propagate on every {m['stride']}-th "
                              f"initial hit + refine_path on the {m['counts']['candidates']} candidates; "
                              f"{m['rays']} rays in {m['seconds']:.1f} s"),
                   "exact_paths_per_s": m["exact_paths_per_s"], "candidates_refined_per_s": m["candidates_per_s"]}
        except Exception as e:  # the oracle is test infrastructure; report why it is missing
            cpu = {"value": None, "unit": "Mrays/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Mrays/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C2 synthetic office, 3 reflections + 1 diffraction = max_interactions 4 / "
                                   "max_diffractions 1 (SURVEY.md §8.0; BASELINE configs[1])",
                       "points": scene.n_points, "tx": int(len(scene.tx)), "rx": int(len(scene.rx)),
                       "edges": int(len(scene.edges)), "max_interactions": cfg.run["max_interactions"],
                       "max_diffractions": cfg.run["max_diffractions"], "kappa": conf.kappa,
                       "parallelism": (f"{world} shards: initial hits and candidates split cyclically, "
                                       f"rows all-gathered over {args.backend.upper()}" if world > 1 else "single GPU"),
                       "l2": "flushed (256 MB write) before every timed step"},
            "rays_per_step": rays, "exact_paths_per_s": exact_per_s, "candidates_refined_per_s": cand_per_s,
            # Mrays/s over the trace stage alone (R / t_trace), beside `value` (R / step)
            "mrays_per_s_trace": rays / dict(s0["timings"]).get("trace", float("nan")) / 1e6,
            "exact_paths": s0["exact_paths"], "coarse_paths": s0["coarse_paths"],
            # knife-edge atan2/asin cone decisions not certified against glibc (trace.cuh libm_le): 0
            # means every cone decision of the step is the reference's
            "libm_unresolved": s0.get("libm_unresolved") if rank == 0 else None,
            "stage_seconds": dict(s0["timings"]), "kernel_share": shares,
            "roofline": rl,
            "cpu_baseline": cpu,
            "e2e": {"value": e_value, "unit": "Mrays/s", "h2d_bytes_per_step": h2d // e_steps,
                    "d2h_bytes_per_step": d2h // e_steps, "ms_per_step": e_step, "steps": e_steps},
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of CPU work for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"], help="N > 1 process group backend")
    args = ap.parse_args()
    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    return b200_arm(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
