"""Stage-1 parity: the CUDA build_grid / compute_march_distances against the oracle,
bit for bit (dims, origin, every cell, every IE field, point_indices).

Cases follow proj/tests/test_voxel_grid.cpp:49-310 plus the synthetic configs."""
import numpy as np
import pytest

from conftest import assert_bitwise, assert_grid_equal
from fixtures import voxel_grid_scenes
from paper_2402_13747_b200 import abi, pcray, scenes

pytestmark = pytest.mark.gpu

SCENES = voxel_grid_scenes()


@pytest.mark.parametrize("name", sorted(SCENES))
@pytest.mark.parametrize("vs,dv", [(0.5, 2), (0.25, 1), (0.7, 3)])
def test_build_grid_matches_oracle(oracle, gpu, name, vs, dv):
    scene = SCENES[name]
    rs = oracle.RefScene(scene)
    params = abi.voxel_params(vs, dv)
    ref = oracle.build_grid(rs, params).to_dict()
    got = pcray.build_grid(pcray.DeviceScene(scene), params).to_dict()
    assert_grid_equal(got, ref)


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_config_grid_matches_oracle(oracle, gpu, cfg):
    scene, sc = scenes.build_scene(cfg)
    ref = oracle.build_grid(oracle.RefScene(scene)).to_dict()
    got = pcray.build_grid(pcray.DeviceScene(scene)).to_dict()
    assert_grid_equal(got, ref)
    # every IE of these rectangle scenes is planar
    surf = got["ie_kind"] == abi.IE_SURFACE
    assert got["ie_planar"][surf].all()


def test_wide_keys_split_label_sort(oracle, gpu):
    # labels near 2^32 force the two-pass (label, then voxel/subvoxel) sort
    scene = SCENES["big_labels"]
    for params in [abi.voxel_params(0.05, 8), abi.voxel_params(0.5, 2)]:
        ref = oracle.build_grid(oracle.RefScene(scene), params).to_dict()
        got = pcray.build_grid(pcray.DeviceScene(scene), params).to_dict()
        assert_grid_equal(got, ref)


def test_errors_match_reference_text(gpu):
    scene = SCENES["single_point"]
    ds = pcray.DeviceScene(scene)
    for params, msg in [(abi.voxel_params(0.0), "voxel_size must be > 0"),
                        (abi.voxel_params(0.5, 0), "division_factor must be >= 1")]:
        with pytest.raises(pcray.PcrError, match=msg):
            pcray.build_grid(ds, params)
    from fixtures import make_scene
    huge = make_scene([((0, 0, 0), (0, 0, 1), 0), ((1000, 1000, 1000), (0, 0, 1), 0)])
    with pytest.raises(pcray.PcrError, match="grid too large"):
        pcray.build_grid(pcray.DeviceScene(huge), abi.VoxelParams(0.5, 2, 1000))
    empty = abi.Scene()
    with pytest.raises(pcray.PcrError, match="empty scene"):
        pcray.build_grid(pcray.DeviceScene(empty))


def _random_grid(rng, dims):
    n = int(np.prod(dims))
    occ = rng.uniform(size=n) < 0.15
    begin = np.zeros(n, np.uint32)
    end = np.zeros(n, np.uint32)
    k = 0
    for i in range(n):
        if occ[i]:
            begin[i] = k
            k += 1
            end[i] = k
    ni = k
    g = {"origin": np.zeros(3), "dims": np.array(dims, np.int32), "voxel_size": 1.0, "division_factor": 2,
         "cell_ie_begin": begin, "cell_ie_end": end, "cell_march": np.full(n, abi.MARCH_NO_IES, np.int32)}
    for f, dt, w in [("ie_kind", np.uint8, 1), ("ie_label", np.uint32, 1), ("ie_reception_point", float, 3),
                     ("ie_sphere_center", float, 3), ("ie_sphere_radius", float, 1), ("ie_point_begin", np.uint32, 1),
                     ("ie_point_end", np.uint32, 1), ("ie_seg_start", float, 3), ("ie_seg_end", float, 3),
                     ("ie_edge_index", np.uint32, 1), ("ie_rx_id", np.uint32, 1), ("ie_planar", np.uint8, 1),
                     ("ie_plane_point", float, 3), ("ie_plane_normal", float, 3), ("ie_voxel", np.uint32, 1),
                     ("ie_subvoxel", np.uint32, 1)]:
        g[f] = np.zeros((ni, w) if w == 3 else ni, dt)
    g["point_indices"] = np.zeros(0, np.uint32)
    return g


def test_march_distances_random_grids(oracle, gpu):
    """test_voxel_grid.cpp:211-239 (20 random grids) + acceptance c5 (grids up to 16^3)."""
    rng = np.random.default_rng(42)
    for trial in range(40):
        dims = tuple(int(x) for x in rng.integers(1, 17 if trial >= 20 else 9, size=3))
        g = _random_grid(rng, dims)
        r = oracle.RefGrid.from_dict(g)
        r.compute_march_distances()
        d = pcray.DeviceGrid.from_dict(g)
        pcray.compute_march_distances(d)
        assert_bitwise(f"march {dims}", d.to_dict()["cell_march"], r.to_dict()["cell_march"])


def test_empty_grid_keeps_sentinel(gpu):
    g = _random_grid(np.random.default_rng(0), (3, 3, 3))
    g["cell_ie_end"][:] = 0
    g["cell_ie_begin"][:] = 0
    for k in list(g):
        if k.startswith("ie_"):
            g[k] = g[k][:0]
    d = pcray.DeviceGrid.from_dict(g)
    pcray.compute_march_distances(d)
    assert (d.to_dict()["cell_march"] == abi.MARCH_NO_IES).all()


def test_grid_roundtrip_upload_download(oracle, gpu):
    scene = SCENES["reception_points"]
    ref = oracle.build_grid(oracle.RefScene(scene)).to_dict()
    d = pcray.DeviceGrid.from_dict(ref)
    assert_grid_equal(d.to_dict(), ref)
