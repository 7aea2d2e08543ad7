"""Golden fixtures (tests/golden, generated from the oracle by make_golden.py).

CPU: the oracle still reproduces every fixture (pins fixtures <-> reference).
GPU: the CUDA path reproduces every fixture bit for bit — these run without the
oracle library, so they also cover a GPU box where oracle/_ref is absent."""
import json
import os

import numpy as np
import pytest

from conftest import assert_bitwise, assert_grid_equal
from golden.make_golden import GRID_SCENES, golden_scene
from paper_2402_13747_b200 import abi

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    z = np.load(os.path.join(GOLDEN, name))
    out = {}
    for k in z.files:
        if "." in k:
            a, b = k.split(".", 1)
            out.setdefault(a, {})[b] = z[k]
        else:
            out[k] = z[k]
    return out


def scalarize(d):
    for k, v in list(d.items()):
        if isinstance(v, dict):
            scalarize(v)
        elif isinstance(v, np.ndarray) and v.ndim == 0:
            d[k] = v.item()
    return d


@pytest.mark.parametrize("name", GRID_SCENES)
def test_oracle_reproduces_grid_fixture(oracle, name):
    want = scalarize(load(f"grid_{name}.npz"))
    got = oracle.build_grid(oracle.RefScene(golden_scene(name))).to_dict()
    assert_grid_equal(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("name", GRID_SCENES)
def test_gpu_grid_matches_fixture(gpu, name):
    from paper_2402_13747_b200 import pcray

    want = scalarize(load(f"grid_{name}.npz"))
    got = pcray.build_grid(pcray.DeviceScene(golden_scene(name))).to_dict()
    assert_grid_equal(got, want)


@pytest.mark.gpu
def test_gpu_trace_and_refine_match_fixture(gpu):
    from paper_2402_13747_b200 import pcray

    want = scalarize(load("trace_box_room_mi2.npz"))
    ds = pcray.DeviceScene(golden_scene("box_room"))
    dg = pcray.build_grid(ds)
    tp = abi.trace_params(max_interactions=2, max_diffractions=0)
    los, hits = pcray.transmission_phase(0, dg, ds, tp)
    for f in ["ie_index", "kind", "position", "normal", "incoming"]:
        assert_bitwise(f, hits[f], want["hits"][f])
    assert_bitwise("los_length", los["length"], want["los"]["length"])
    cands = pcray.propagate(0, hits, dg, ds, tp)
    c = want["cands"]
    assert cands["n"] == c["n"]
    for f in ["rx_id", "length", "n_inter"]:
        assert_bitwise(f, cands[f], c[f])
    for i in range(int(c["n"])):
        k = int(c["n_inter"][i])
        for f in ["kind", "position", "label", "normal", "ie_index"]:
            assert_bitwise(f, cands[f][i, :k], c[f][i, :k])
    out = pcray.refine_paths(cands, dg, ds)
    o = want["out"]
    assert_bitwise("reason", out["reason"], o["reason"])
    assert_bitwise("has_path", out["has_path"], o["has_path"])
    sel = np.nonzero(o["has_path"])[0]
    assert_bitwise("length", out["length"][sel], o["length"][sel])


@pytest.mark.gpu
def test_gpu_pipeline_c1_matches_fixture(gpu):
    from paper_2402_13747_b200 import pcray, scenes

    with open(os.path.join(GOLDEN, "smoke_c1.json")) as f:
        want = json.load(f)
    scene, cfg = scenes.build_scene("C1")
    got = pcray.run_pipeline_on_scene(scene, abi.default_run_config(**cfg.run))
    for k in ["point_count", "ie_count", "grid_dims", "coarse_paths", "refined_paths", "rejected", "exact_paths",
              "hash"]:
        assert got[k] == want[k], k
    assert np.allclose(got["paths"]["length"], want["paths"]["length"], rtol=1e-6, atol=1e-4)
    assert got["paths"]["rx_id"].tolist() == want["paths"]["rx_id"]
