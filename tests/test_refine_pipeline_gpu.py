"""Stage-3 and end-to-end parity: refine_path outcomes and run_pipeline_on_scene
summaries against the oracle. Reject reasons, counts, kinds and labels are exact;
refined points and lengths must agree within 1e-4 m / 1e-6 relative (north_star
tolerance) and are expected bit-identical (FP64, same operation order)."""
import numpy as np
import pytest

from conftest import assert_bitwise
from fixtures import add_wall, box_room, make_scene
from paper_2402_13747_b200 import abi, pcray, scenes

pytestmark = pytest.mark.gpu

TOL_ABS, TOL_REL = 1e-4, 1e-6


def acceptance_screen():
    """Screen with a diffracting top edge, TX/RX in mutual shadow
    (proj/tests/acceptance/acceptance_main.cpp:197-206, criterion 2)."""
    p = scenes.PlanarScene()
    p.add_rect((-2, 0, 0), (4, 0, 0), (0, 0, 1), 0)
    p.add_rect((-2, 0, 0), (0, 0, 1), (4, 0, 0), 1)
    p.edges.append(((-2, 0, 1), (2, 0, 1), (0, -1, 0), (0, 1, 0), 2))
    p.tx.append([0.3, -1.5, 0.4])
    p.rx.append([-0.2, 1.8, 0.55])
    return scenes.scene_from_planar(p, 5000.0, 11)


def assert_close(name, a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape
    ok = np.abs(a - b) <= np.maximum(TOL_ABS, TOL_REL * np.abs(b))
    assert ok.all(), f"{name}: max diff {np.max(np.abs(a - b))}"


def compare_outcomes(got, ref, exact_bits=True):
    assert_bitwise("reason", got["reason"], ref["reason"])
    assert_bitwise("has_path", got["has_path"], ref["has_path"])
    sel = np.nonzero(ref["has_path"])[0]
    bitwise_ok = True
    for i in sel:
        k = int(ref["n_inter"][i])
        assert_bitwise("label", got["label"][i, :k], ref["label"][i, :k])
        assert_bitwise("kind", got["kind"][i, :k], ref["kind"][i, :k])
        assert_close("position", got["position"][i, :k], ref["position"][i, :k])
        bitwise_ok &= np.array_equal(got["position"][i, :k].view(np.uint64), ref["position"][i, :k].view(np.uint64))
    assert_close("length", got["length"][sel], ref["length"][sel])
    bitwise_ok &= np.array_equal(got["length"][sel].view(np.uint64), ref["length"][sel].view(np.uint64))
    if exact_bits:
        assert bitwise_ok, "refined geometry within tolerance but not bit-identical"


def test_refine_reference_cases(oracle, gpu):
    """proj/tests/test_refine.cpp:200-317 candidates through the batch API."""
    pts = []
    add_wall(pts, (-0.2, -0.6, 0), (1.4, 0, 0), (0, 1.2, 0), (0, 0, 1), 0, 0.03)
    scene = make_scene(pts, tx=[(0, 0, 1)], rx=[(1, 0, 1)])

    def cand(tx, rx, inters):
        n = len(inters)
        s = max(1, n)
        d = {"n": 1, "stride": s, "tx_position": np.array([tx], float), "rx_position": np.array([rx], float),
             "n_inter": np.array([n], np.uint32), "kind": np.zeros((1, s), np.uint8),
             "position": np.zeros((1, s, 3)), "label": np.zeros((1, s), np.uint32), "normal": np.zeros((1, s, 3)),
             "ie_index": np.full((1, s), abi.NO_IE, np.uint32), "edge_index": np.zeros((1, s), np.uint32),
             "length": np.zeros(1)}
        for k, (kind, p, lab, nrm, e) in enumerate(inters):
            d["kind"][0, k] = kind
            d["position"][0, k] = p
            d["label"][0, k] = lab
            d["normal"][0, k] = nrm
            d["edge_index"][0, k] = e
        return d

    cases = [
        (scene, cand((0, 0, 1), (1, 0, 1), [(0, (0.4, 0, 0), 0, (0, 0, 1), 0)])),
        (scene, cand((0, 0, 1), (1, 0, 1), [(0, (0, 0, 1), 0, (0, 0, 1), 0)])),  # degenerate
    ]
    pts2 = []
    add_wall(pts2, (0, -0.6, 0), (1, 0, 0), (0, 1.2, 0), (0, 0, 1), 0, 0.03)
    miss = make_scene(pts2, tx=[(5, 0, 1)], rx=[(6, 0, 1)])
    cases.append((miss, cand((5, 0, 1), (6, 0, 1), [(0, (5.3, 0, 0), 0, (0, 0, 1), 0)])))
    pts3 = list(pts)
    add_wall(pts3, (0.1, -0.3, 0.5), (0.3, 0, 0), (0, 0.6, 0), (0, 0, 1), 9, 0.03)
    occl = make_scene(pts3, tx=[(0, 0, 1)], rx=[(1, 0, 1)])
    cases.append((occl, cand((0, 0, 1), (1, 0, 1), [(0, (0.4, 0, 0), 0, (0, 0, 1), 0)])))
    screen = make_scene([], tx=[(0, -1, 1)], rx=[(0, 1, 1)], edges=[((-1, 0, 0), (1, 0, 0), (0, 0, 1), (0, 0, -1), 5)])
    cases.append((screen, cand((0, -1, 1), (0, 1, 1), [(1, (0.3, 0, 0), 5, (0, 0, 1), 0)])))
    clamp = make_scene([], tx=[(3, -1, 1)], rx=[(3, 1, 1)], edges=[((-1, 0, 0), (1, 0, 0), (0, 0, 1), (0, 0, -1), 5)])
    cases.append((clamp, cand((3, -1, 1), (3, 1, 1), [(1, (0.5, 0, 0), 5, (0, 0, 1), 0)])))
    pts4 = []
    add_wall(pts4, (-0.5, -0.6, 0), (5, 0, 0), (0, 1.2, 0), (0, 0, 1), 0, 0.04)
    add_wall(pts4, (-0.5, -0.6, 3), (5, 0, 0), (0, 1.2, 0), (0, 0, -1), 1, 0.04)
    corridor = make_scene(pts4, tx=[(0, 0, 1)], rx=[(4, 0, 1)])
    cases.append((corridor, cand((0, 0, 1), (4, 0, 1), [(0, (0.8, 0.05, 0), 0, (0, 0, 1), 0),
                                                        (0, (2.4, -0.05, 3), 1, (0, 0, -1), 0)])))
    reasons = []
    for sc, c in cases:
        rs = oracle.RefScene(sc)
        rg = oracle.build_grid(rs)
        ds = pcray.DeviceScene(sc)
        dg = pcray.build_grid(ds)
        ref = oracle.refine_batch(rg, rs, c)
        got = pcray.refine_paths(c, dg, ds)
        compare_outcomes(got, ref)
        reasons.append(int(ref["reason"][0]) if not ref["has_path"][0] else -1)
    assert abi.DEGENERATE in reasons and abi.RAY_MISSED in reasons and abi.OCCLUDED in reasons


@pytest.mark.parametrize("name,mi,md", [("box", 2, 0), ("screen", 2, 1)])
def test_refine_propagated_candidates(oracle, gpu, name, mi, md):
    if name == "box":
        sc = make_scene(box_room((2, 2, 2), 0.05), tx=[(0.6, 0.7, 0.9)], rx=[(1.3, 1.2, 1.1)])
    else:
        sc = acceptance_screen()
    rs = oracle.RefScene(sc)
    rg = oracle.build_grid(rs)
    ds = pcray.DeviceScene(sc)
    dg = pcray.build_grid(ds)
    tp = abi.trace_params(max_interactions=mi, max_diffractions=md)
    _, hits = oracle.transmission_phase(rg, rs, 0, tp)
    cands = oracle.propagate(rg, rs, 0, hits, tp)
    assert cands["n"] > 0
    ref = oracle.refine_batch(rg, rs, cands)
    got = pcray.refine_paths(cands, dg, ds)
    compare_outcomes(got, ref)


def compare_summaries(got, ref):
    for k in ["point_count", "edge_count", "ie_count", "grid_dims", "coarse_paths", "refined_paths", "rejected",
              "exact_paths", "hash"]:
        assert got[k] == ref[k], f"{k}: {got[k]} vs {ref[k]}"
    assert [t for t, _ in got["timings"]] == [t for t, _ in ref["timings"]]
    gp, rp = got["paths"], ref["paths"]
    for f in ["tx_id", "rx_id", "n_inter", "converged"]:
        assert_bitwise(f, gp[f], rp[f])
    for i in range(rp["n"]):
        k = int(rp["n_inter"][i])
        assert_bitwise("kind", gp["kind"][i, :k], rp["kind"][i, :k])
        assert_bitwise("label", gp["label"][i, :k], rp["label"][i, :k])
        assert_close("position", gp["position"][i, :k], rp["position"][i, :k])
    assert_close("length", gp["length"], rp["length"])
    assert_close("delay", gp["delay"] * 1e9, rp["delay"] * 1e9)


@pytest.mark.parametrize("name", ["empty_los", "box1", "box2", "screen"])
def test_pipeline_small(oracle, gpu, name):
    if name == "empty_los":
        sc, cfg = make_scene([], tx=[(0, 0, 1)], rx=[(3, 2, 1)]), {}
    elif name.startswith("box"):
        sc = make_scene(box_room((2, 2, 2), 0.06), tx=[(0.6, 0.7, 0.9)], rx=[(1.3, 1.2, 1.1)])
        cfg = {"max_interactions": int(name[-1])}
    else:
        sc = acceptance_screen()
        cfg = {"max_interactions": 2}
    ref = oracle.run_pipeline_on_scene(oracle.RefScene(sc), oracle.default_run_config(**cfg))
    got = pcray.run_pipeline_on_scene(sc, abi.default_run_config(**cfg))
    compare_summaries(got, ref)


def test_pipeline_c1(oracle, gpu):
    scene, cfg = scenes.build_scene("C1")
    ref = oracle.run_pipeline_on_scene(oracle.RefScene(scene), oracle.default_run_config(**cfg.run))
    got = pcray.run_pipeline_on_scene(scene, abi.default_run_config(**cfg.run))
    compare_summaries(got, ref)


@pytest.mark.parametrize("mi,md", [(1, 1), (2, 1)])
def test_pipeline_office_c2_reduced_depth(oracle, gpu, mi, md):
    """C2 geometry (1M points, 64 RX, 40 diffraction edges) at reduced depth so the CPU
    oracle finishes in seconds; the full depth runs in bench.py."""
    scene, cfg = scenes.build_scene("C2")
    kw = dict(max_interactions=mi, max_diffractions=md)
    ref = oracle.run_pipeline_on_scene(oracle.RefScene(scene), oracle.default_run_config(**kw))
    got = pcray.run_pipeline_on_scene(scene, abi.default_run_config(**kw))
    compare_summaries(got, ref)


def test_pipeline_stage_errors(gpu):
    bad = make_scene([((0, 0, 0), (0, 0, 2), 0)], tx=[(0, 0, 1)], rx=[(1, 0, 1)])
    with pytest.raises(pcray.PcrError, match="validate: point_normal_unit"):
        pcray.run_pipeline_on_scene(bad)
    huge = make_scene([((0, 0, 0), (0, 0, 1), 0), ((2000, 2000, 2000), (0, 0, 1), 0)], tx=[(0, 0, 1)], rx=[(1, 0, 1)])
    with pytest.raises(pcray.PcrError, match="voxelize: grid too large"):
        pcray.run_pipeline_on_scene(huge, abi.default_run_config(voxel_size_m=0.01))


def test_config_hash_matches(oracle, gpu):
    for kw in [{}, {"kappa": 99}, {"fresnel_enabled": False}, {"voxel_size_m": 0.25}, {"thread_count": 8}]:
        c = abi.default_run_config(**kw)
        assert pcray.config_hash(c) == oracle.config_hash(c)


@pytest.mark.parametrize("vs,dv", [(0.5, 1), (0.5, 4), (0.25, 2), (0.3, 3)])
def test_refine_voxel_params(oracle, gpu, vs, dv):
    """The warp kernel's cooperative same-label scan applies when the reprojection box is
    a cell's 3x3x3 neighbourhood (division_factor 2); other grids take the serial cell
    walk per lane. Both against the reference on the same candidates."""
    sc = make_scene(box_room((2, 2, 2), 0.05), tx=[(0.6, 0.7, 0.9)], rx=[(1.3, 1.2, 1.1)])
    vp = abi.voxel_params(vs, dv)
    rs = oracle.RefScene(sc)
    rg = oracle.build_grid(rs, vp)
    ds = pcray.DeviceScene(sc)
    dg = pcray.build_grid(ds, vp)
    tp = abi.trace_params(max_interactions=3, max_diffractions=0)
    _, hits = oracle.transmission_phase(rg, rs, 0, tp)
    cands = oracle.propagate(rg, rs, 0, hits, tp)
    assert cands["n"] > 0
    compare_outcomes(pcray.refine_paths(cands, dg, ds), oracle.refine_batch(rg, rs, cands))


def test_refine_kernels_agree():
    """The warp-cooperative kernel (default) and the thread-per-path kernel
    (PCR_REFINE_MODE=1) give the same RunSummary, counters included (C2 at depth 2)."""
    import json
    import os
    import subprocess
    import sys

    code = ("import json,sys; sys.path.insert(0, %r); from paper_2402_13747_b200 import abi, pcray, scenes; "
            "s, _ = scenes.build_scene('C2'); r = pcray.run_pipeline_on_scene(s, abi.default_run_config("
            "max_interactions=2, max_diffractions=1)); p = r['paths']; "
            "print(json.dumps([r['coarse_paths'], r['refined_paths'], list(r['rejected']), r['exact_paths'], "
            "r['refine_iterations'], r['refine_trials'], r['refine_marches'], p['length'].tolist()]))"
            % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    out = []
    for mode in ["0", "1"]:
        env = dict(os.environ, PCR_REFINE_MODE=mode)
        res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-2000:]
        out.append(json.loads(res.stdout.strip().splitlines()[-1]))
    assert out[0] == out[1]
