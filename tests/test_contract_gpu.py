"""Per-path parity at the contract depths, on the whole scene.

Golden digests come from the oracle (tests/golden/make_contract_golden.py: the
unmodified reference compiled in oracle/_ref, run here on the full scene); the CUDA
path recomputes them on the same in-memory scene:

* coarse candidates — transmission_phase + propagate per TX, LOS rows first
  (pipeline.cpp:136-146): tx/rx ids and positions, coarse length, and per used slot
  kind, label, IE and edge index, position and normal, all bitwise;
* refine outcomes per candidate — RejectReason, has_path, and for every refined path
  the kinds, labels, positions and total length, bitwise;
* run_pipeline_on_scene — RunSummary counts and the final deduplicated, sorted paths
  (every JSONL field), bitwise;
* the launched-ray numerator: the GPU's cone-trace counter equals the counting
  oracle's number of voxel_cone_trace calls (oracle/ref_count.cpp).

C2 is the bench workload at SURVEY §8.0's 4 interactions / 1 diffraction (1.65 M
candidates); C2d3 the same scene at depth 3; C1 the acceptance box room.
"""
import json
import math
import os

import numpy as np
import pytest

import digest
from paper_2402_13747_b200 import abi, pcray, scenes

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _golden(name):
    with open(os.path.join(HERE, "golden", f"contract_{name}.json")) as f:
        return json.load(f)


def _concat(parts):
    parts = [p for p in parts if p["n"] > 0]
    s = max(p["stride"] for p in parts)
    out = {"n": sum(p["n"] for p in parts), "stride": s}
    for k, v in parts[0].items():
        if not isinstance(v, np.ndarray):
            continue
        arrs = []
        for p in parts:
            a = p[k]
            if a.ndim >= 2 and k not in ("tx_position", "rx_position") and a.shape[1] != s:
                pad = np.zeros((a.shape[0], s) + a.shape[2:], a.dtype)
                pad[:, : a.shape[1]] = a
                a = pad
            arrs.append(a)
        out[k] = np.concatenate(arrs)
    return out


CONFIGS = [c for c in ["C1", "C2d3", "C2"] if os.path.exists(os.path.join(HERE, "golden", f"contract_{c}.json"))]


@pytest.mark.parametrize("name", CONFIGS)
def test_contract_config_per_path(gpu, name):
    gold = _golden(name)
    scene, cfg = scenes.build_scene(name)
    run = dict(cfg.run)
    assert run == gold["run"], "golden digests were made for another config"
    assert scene.n_points == gold["points"]
    slots = run["max_interactions"]
    conf = abi.default_run_config(**run)
    tp = abi.trace_params(conf.max_interactions, conf.kappa, conf.cone_apex_angle_deg * math.pi / 180.0,
                          conf.diffraction_ray_count, conf.max_diffractions)
    rp = abi.refine_params(conf.delta, conf.rho, conf.step_size, bool(conf.fresnel_enabled))
    ds = pcray.DeviceScene(scene)
    dg = pcray.build_grid(ds, abi.voxel_params(conf.voxel_size_m, conf.division_factor))

    parts, cones, n_hits = [], 0, 0
    for t in range(len(scene.tx)):
        los, hits = pcray.transmission_phase(t, dg, ds, tp)
        n_hits += hits["n"]
        parts += [los, pcray.propagate(t, hits, dg, ds, tp)]
        st = pcray.last_trace_stats()
        cones += st["cone_traces"]
        assert st["libm_unresolved"] == 0  # every knife-edge cone decision certified against glibc
    assert n_hits == gold["initial_hits"]
    # the Mrays/s numerator: GPU cone traces = the reference's voxel_cone_trace calls
    assert cones == gold["cone_traces"], f"cone traces {cones} vs counting oracle {gold['cone_traces']}"
    cands = _concat(parts)
    digest.compare(digest.candidates_digest(cands, slots), gold["candidates"], f"{name} coarse candidates")

    outs = pcray.refine_paths(cands, dg, ds, rp)
    digest.compare(digest.outcomes_digest(outs, slots), gold["outcomes"], f"{name} refine outcomes")
    del cands, outs

    s = pcray.run_pipeline_device(ds, conf)
    for k, v in gold["summary"].items():
        assert s[k] == v, f"{name} summary {k}: {s[k]} vs {v}"
    assert s["cone_traces"] == gold["cone_traces"]
    assert s["libm_unresolved"] == 0
    assert s["transmission_rays"] == gold["transmission_rays"]
    digest.compare(digest.paths_digest(s["paths"], slots), gold["paths"], f"{name} final paths")
