"""C2-np: the C2 office with every normal tilted by up to 1 degree, so
no IE is planar and every march, projection and polish runs the Gaussian-weighted
SDF (estimate_surface, exp()). The device exp is the host libm's algorithm restated
(geom.cuh glibc_exp), checked here against the host's exp() bit for bit, so the
non-planar pipeline is bit-exact too (north-star tolerance asserted as the floor)."""
import ctypes
import math

import numpy as np
import pytest

from conftest import assert_grid_equal
from paper_2402_13747_b200 import abi, pcray, scenes

pytestmark = pytest.mark.gpu

TOL_ABS, TOL_REL = 1e-4, 1e-6


def test_device_exp_matches_host_libm(gpu):
    libm = ctypes.CDLL("libm.so.6")
    libm.exp.restype = ctypes.c_double
    libm.exp.argtypes = [ctypes.c_double]
    rng = np.random.default_rng(5)
    x = np.concatenate([
        -rng.uniform(0, 40, 400_000),             # the SDF's range: -d2/h^2
        rng.uniform(-745.2, 709.8, 200_000),      # the whole finite range
        rng.uniform(-745.2, -700, 50_000),        # scaled subnormal results
        rng.uniform(700, 709.8, 20_000),          # scaled results near overflow
        rng.uniform(-1e-15, 1e-15, 10_000),
        np.array([0.0, -0.0, 1e-300, -1e-300, 709.782712893384, 709.7827128933841, -745.1332191019411,
                  -745.1332191019412, -708.3964185322641, -1000.0, 1000.0, math.inf, -math.inf, 1.0, -1.0]),
    ])
    got = pcray.libm_exp(x)
    ref = np.array([libm.exp(float(v)) for v in x])
    bad = np.nonzero(got.view(np.uint64) != ref.view(np.uint64))[0]
    assert len(bad) == 0, f"{len(bad)} mismatches, first x={x[bad[0]]!r}: {got[bad[0]]!r} vs {ref[bad[0]]!r}"


@pytest.fixture(scope="module")
def c2np():
    scene, _ = scenes.build_scene("C2np")
    return scene


def test_c2np_grid_is_nonplanar_and_exact(oracle, gpu, c2np):
    rg = oracle.build_grid(oracle.RefScene(c2np)).to_dict()
    dg = pcray.build_grid(pcray.DeviceScene(c2np)).to_dict()
    assert_grid_equal(dg, rg)
    surf = dg["ie_kind"] == abi.IE_SURFACE
    assert not dg["ie_planar"][surf].any()


@pytest.mark.parametrize("mi,md", [(1, 0), (1, 1)])
def test_c2np_pipeline_within_tolerance(oracle, gpu, c2np, mi, md):
    kw = dict(max_interactions=mi, max_diffractions=md)
    ref = oracle.run_pipeline_on_scene(oracle.RefScene(c2np), oracle.default_run_config(**kw))
    got = pcray.run_pipeline_on_scene(c2np, abi.default_run_config(**kw))
    for k in ["ie_count", "coarse_paths", "refined_paths", "exact_paths"]:
        assert got[k] == ref[k], k
    assert list(got["rejected"]) == list(ref["rejected"])
    gp, rp = got["paths"], ref["paths"]
    for f in ["tx_id", "rx_id", "n_inter"]:
        assert np.array_equal(gp[f], rp[f]), f
    for i in range(rp["n"]):
        k = int(rp["n_inter"][i])
        assert np.array_equal(gp["label"][i, :k], rp["label"][i, :k])
        a, b = gp["position"][i, :k], rp["position"][i, :k]
        assert (np.abs(a - b) <= np.maximum(TOL_ABS, TOL_REL * np.abs(b))).all()
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), f"path {i} positions not bit-identical"
    assert (np.abs(gp["length"] - rp["length"]) <= np.maximum(TOL_ABS, TOL_REL * rp["length"])).all()
    assert np.array_equal(gp["length"].view(np.uint64), rp["length"].view(np.uint64))
