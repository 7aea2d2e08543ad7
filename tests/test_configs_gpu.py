"""Parity on the large BASELINE configs at sizes the CPU
oracle finishes in seconds, plus size-independent properties at full size:

* C3 (street canyon, 10M points, 4 TX / 256 RX) and C4 (dense floor, 10M points,
  16 TX / 1024 RX, diffraction edges): the full grid bitwise, transmission_phase of
  two TXs bitwise, propagate on a deterministic sample of initial hits (the
  reference API takes the hit list, tracer.hpp:122) bitwise, and refine_path on the
  resulting candidates (reasons exact, geometry bitwise / within 1e-4 m).
* C2-np (the office with tilted normals, every IE non-planar) the same way at its
  contract depth 4 / 1: every march, projection and polish through the Gaussian SDF.
* C5 (voxelization sweep): the grid bitwise at 1M and 3M points for several
  (voxel, D_v), and at 30M points the properties the reference's own tests state:
  point_indices is a permutation, IE ranges tile it, every point sits in its IE's
  voxel, cells cover the IEs in order, march is 0 exactly at occupied cells.
"""
import numpy as np
import pytest

from conftest import assert_bitwise, assert_grid_equal
from test_refine_pipeline_gpu import compare_outcomes
from test_trace_gpu import assert_paths_equal
from paper_2402_13747_b200 import abi, pcray, scenes

pytestmark = pytest.mark.gpu


def _subset(hits, idx):
    out = {"n": len(idx)}
    for k in ["ie_index", "kind", "position", "normal", "incoming"]:
        out[k] = np.ascontiguousarray(hits[k][idx])
    return out


@pytest.fixture(scope="module")
def big(oracle, gpu):
    cache = {}

    def get(name):
        if name not in cache:
            scene, cfg = scenes.build_scene(name)
            rs = oracle.RefScene(scene)
            rg = oracle.build_grid(rs)  # build_grid ends with compute_march_distances
            ds = pcray.DeviceScene(scene)
            dg = pcray.build_grid(ds)
            cache[name] = (scene, cfg, rs, rg, ds, dg)
        return cache[name]

    return get


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_config_grid(big, name):
    scene, cfg, rs, rg, ds, dg = big(name)
    assert_grid_equal(dg.to_dict(), rg.to_dict())


# initial-hit samples per TX at the contract depth (C3 3 / 0, C4 5 / 1, C2-np 4 / 1):
# sized so the oracle finishes in seconds; C4's and C2-np's samples include edge hits
# (Keller fans, ~270 rays each). C2-np's candidates refine through the Gaussian SDF on
# both sides (the oracle's refine is the slow part: ~100 candidates in ~10 s).
SAMPLES = {"C3": (6, 0), "C4": (8, 2), "C2np": (4, 1)}


@pytest.mark.parametrize("name", ["C3", "C4", "C2np"])
def test_config_trace_and_refine_sample(oracle, big, name):
    """transmission_phase bitwise for the first and last TX; propagate at the contract
    depth (no depth cap) on a deterministic initial-hit sample, per path bitwise, with
    the GPU's cone-trace count equal to the counting oracle's voxel_cone_trace calls;
    refine_path on every resulting candidate (reasons exact, geometry bitwise)."""
    scene, cfg, rs, rg, ds, dg = big(name)
    run = cfg.run
    n_tasks, n_edge = SAMPLES[name]
    tp = abi.trace_params(max_interactions=run["max_interactions"], max_diffractions=run["max_diffractions"])
    for tx in sorted({0, len(scene.tx) - 1}):
        ref_los, ref_hits = oracle.transmission_phase(rg, rs, tx, tp)
        los, hits = pcray.transmission_phase(tx, dg, ds, tp)
        assert_paths_equal(los, ref_los, ["tx_id", "rx_id", "tx_position", "rx_position", "length", "n_inter"])
        assert hits["n"] == ref_hits["n"]
        for f in ["ie_index", "kind", "position", "normal", "incoming"]:
            assert_bitwise(f, hits[f], ref_hits[f])
        # a deterministic spread of initial hits (plus edge hits when the scene has edges)
        idx = np.unique(np.linspace(0, ref_hits["n"] - 1, n_tasks).astype(np.int64))
        edge_hits = np.nonzero(ref_hits["kind"] == abi.IE_EDGE)[0]
        if len(edge_hits) and n_edge:
            idx = np.unique(np.concatenate([idx, edge_hits[:: max(1, len(edge_hits) // n_edge)][:n_edge]]))
        sub = _subset(ref_hits, idx)
        with oracle.counting() as c:  # the reference's voxel_cone_trace calls on this sample
            crs = oracle.RefScene(scene)
            crg = oracle.build_grid(crs)
            c.read(reset=True)
            ref_c = oracle.propagate(crg, crs, tx, sub, tp)
            ref_cones, _ = c.read(reset=True)
            del crg, crs
        got_c = pcray.propagate(tx, sub, dg, ds, tp)
        st = pcray.last_trace_stats()
        assert st["cone_traces"] == ref_cones
        assert st["libm_unresolved"] == 0  # every knife-edge cone decision certified (trace.cuh libm_le)
        assert_paths_equal(got_c, ref_c)
        if ref_c["n"]:
            compare_outcomes(pcray.refine_paths(ref_c, dg, ds), oracle.refine_batch(rg, rs, ref_c))


@pytest.mark.parametrize("target", [1_000_000, 3_000_000])
@pytest.mark.parametrize("vs,dv", [(0.5, 2), (1.0, 4), (0.25, 1)])
def test_c5_grid_matches_oracle(oracle, gpu, target, vs, dv):
    base = scenes.config("C3")
    scene = scenes.scene_from_planar(base.planar, scenes.scaled_density(base, target), base.seed)
    params = abi.voxel_params(vs, dv)
    rg = oracle.build_grid(oracle.RefScene(scene), params)
    dg = pcray.build_grid(pcray.DeviceScene(scene), params)
    assert_grid_equal(dg.to_dict(), rg.to_dict())


def test_c5_properties_30m(gpu):
    base = scenes.config("C3")
    scene = scenes.scene_from_planar(base.planar, scenes.scaled_density(base, 30_000_000), base.seed)
    dg = pcray.build_grid(pcray.DeviceScene(scene))
    g = dg.to_dict()
    n = scene.n_points
    pidx = g["point_indices"]
    assert len(pidx) == n and np.array_equal(np.sort(pidx), np.arange(n, dtype=pidx.dtype))
    surf = g["ie_kind"] == abi.IE_SURFACE
    b, e = g["ie_point_begin"][surf].astype(np.int64), g["ie_point_end"][surf].astype(np.int64)
    assert b[0] == 0 and e[-1] == n and np.array_equal(b[1:], e[:-1]) and (e > b).all()
    # every point lies in its IE's voxel (voxel_grid.cpp:115-126)
    dims = g["dims"].astype(np.int64)
    vox = g["ie_voxel"][surf].astype(np.int64)
    owner = np.repeat(vox, e - b)
    p = scene.position[pidx.astype(np.int64)]
    v = np.clip(np.floor((p - g["origin"]) / (g["voxel_size"] / g["division_factor"])).astype(np.int64)
                // g["division_factor"], 0, dims - 1)
    lin = v[:, 0] + dims[0] * (v[:, 1] + dims[1] * v[:, 2])
    assert np.array_equal(lin, owner)
    # occupied cells tile the IE list in cell order; march == 0 exactly where IEs are
    cb, ce = g["cell_ie_begin"].astype(np.int64), g["cell_ie_end"].astype(np.int64)
    occupied = ce > cb
    ob, oe = cb[occupied], ce[occupied]
    assert ob[0] == 0 and oe[-1] == len(g["ie_kind"]) and np.array_equal(ob[1:], oe[:-1])
    assert np.array_equal(g["ie_voxel"][ob], np.nonzero(occupied)[0])
    assert np.array_equal(g["cell_march"] == 0, occupied)
