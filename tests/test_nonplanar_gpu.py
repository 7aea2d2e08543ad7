"""C2-np: the C2 office with every normal tilted by up to 1 degree, so
no IE is planar and every march, projection and polish runs the Gaussian-weighted
SDF (estimate_surface, exp()). The grid is bit-exact (no libm on that path); traced
and refined geometry is compared within the north-star tolerance, because CUDA's
exp may differ from glibc's in the last ulp."""
import numpy as np
import pytest

from conftest import assert_grid_equal
from paper_2402_13747_b200 import abi, pcray, scenes

pytestmark = pytest.mark.gpu

TOL_ABS, TOL_REL = 1e-4, 1e-6


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
    assert (np.abs(gp["length"] - rp["length"]) <= np.maximum(TOL_ABS, TOL_REL * rp["length"])).all()
