"""Stage-2 parity: transmission_phase, segment_visible, voxel_cone_trace and propagate
on the GPU against the oracle. Integer/index outputs and positions must be bit-exact
(the cone test's atan2/asin knife edges are the only tolerated source of divergence,
and none are expected on these inputs)."""
import numpy as np
import pytest

from conftest import assert_bitwise, assert_fp
from fixtures import add_wall, box_room, make_scene, voxel_grid_scenes
from paper_2402_13747_b200 import abi, pcray, scenes

pytestmark = pytest.mark.gpu

# scenes whose surface model calls exp() (the non-planar SDF); the device exp equals
# the host libm's bit for bit (geom.cuh glibc_exp), so these are bitwise too
NONPLANAR = set()

PATH_FIELDS = ["tx_id", "rx_id", "tx_position", "rx_position", "length", "n_inter", "kind", "position", "label",
               "normal", "ie_index", "edge_index"]


def assert_paths_equal(got, ref, fields=PATH_FIELDS):
    assert got["n"] == ref["n"], f"path count {got['n']} vs {ref['n']}"
    s = min(got["stride"], ref["stride"])
    for f in fields:
        a, b = got[f], ref[f]
        if a.ndim >= 2:
            # compare the used interaction slots only
            n_inter = ref["n_inter"]
            for i in range(ref["n"]):
                k = int(n_inter[i])
                assert_bitwise(f"{f}[{i}]", a[i, :k], b[i, :k])
        else:
            assert_bitwise(f, a, b)
    del s


def trace_scenes():
    out = {}
    out["box_room"] = make_scene(box_room((2, 2, 2), 0.05), tx=[(0.6, 0.7, 0.9)], rx=[(1.3, 1.2, 1.1)])
    pts = []
    add_wall(pts, (0, -1, -1), (0, 2, 0), (0, 0, 2), (1, 0, 0), 0, 0.04)
    out["wall_blocks_los"] = make_scene(pts, tx=[(0.8, 0, 0)], rx=[(-0.8, 0, 0)])
    pts = []
    add_wall(pts, (-2, 0, 0), (4, 0, 0), (0, 0, 1), (0, -1, 0), 0, 0.04)
    add_wall(pts, (-2, 0, 1), (4, 0, 0), (0, 1.5, 0), (0, 0, 1), 1, 0.04)
    out["screen_edge"] = make_scene(pts, tx=[(0.5, -1, 0.3)], rx=[(0.5, 2, 1.5)],
                                    edges=[((-2, 0, 1), (2, 0, 1), (0, -1, 0), (0, 0, 1), 7)])
    out["empty_los"] = make_scene([], tx=[(0, 0, 1)], rx=[(3, 2, 1)])
    out["nonplanar_patch"] = voxel_grid_scenes()["nonplanar_patch"]
    return out


TS = trace_scenes()


@pytest.fixture(scope="module")
def built(oracle, gpu):
    cache = {}

    def get(name, scene=None):
        if name not in cache:
            sc = scene if scene is not None else TS[name]
            rs = oracle.RefScene(sc)
            rg = oracle.build_grid(rs)
            ds = pcray.DeviceScene(sc)
            dg = pcray.build_grid(ds)
            cache[name] = (rs, rg, ds, dg)
        return cache[name]

    return get


@pytest.mark.parametrize("name", sorted(TS))
def test_transmission_phase(oracle, built, name):
    rs, rg, ds, dg = built(name)
    ref_los, ref_hits = oracle.transmission_phase(rg, rs, 0)
    los, hits = pcray.transmission_phase(0, dg, ds)
    assert_paths_equal(los, ref_los, ["tx_id", "rx_id", "tx_position", "rx_position", "length", "n_inter"])
    assert hits["n"] == ref_hits["n"]
    for f in ["ie_index", "kind", "position", "normal", "incoming"]:
        assert_fp(f, hits[f], ref_hits[f], exact=name not in NONPLANAR)


@pytest.mark.parametrize("name", ["box_room", "screen_edge", "wall_blocks_los", "nonplanar_patch"])
def test_segment_visible_random(oracle, built, name):
    rs, rg, ds, dg = built(name)
    g = dg.to_dict()
    rng = np.random.default_rng(1)
    lo = g["origin"]
    hi = lo + g["dims"] * g["voxel_size"]
    n = 4000
    o = rng.uniform(lo, hi, size=(n, 3))
    t = rng.uniform(lo, hi, size=(n, 3))
    # half of the targets are IE reception points with their own index exempt
    ni = len(g["ie_kind"])
    tie = np.full(n, abi.NO_IE, np.uint32)
    if ni:
        pick = rng.integers(0, ni, size=n // 2)
        t[: n // 2] = g["ie_reception_point"][pick]
        tie[: n // 2] = pick
    ref = oracle.segment_visible_batch(rg, rs, o, t, tie)
    got = pcray.segment_visible(o, t, tie, dg, ds)
    assert_bitwise("visible", got, ref)
    assert 0 < ref.sum() < n or name == "nonplanar_patch"


def _random_rays(g, rng, n, with_planes=True):
    lo = g["origin"]
    hi = lo + g["dims"] * g["voxel_size"]
    rays = []
    ni = len(g["ie_kind"])
    for k in range(n):
        o = rng.uniform(lo, hi)
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        planes = []
        if with_planes and k % 3 == 0:
            nrm = rng.standard_normal(3)
            nrm /= np.linalg.norm(nrm)
            planes = [(o, nrm)]
        oie, olab = abi.NO_IE, 0
        if ni and k % 2 == 0:
            oie = int(rng.integers(0, ni))
            olab = int(g["ie_label"][oie])
        rays.append(pcray.make_ray(o, d, np.pi / 180.0 * (1.0 + 4.0 * (k % 4)), planes, oie, olab))
    return rays


@pytest.mark.parametrize("name", ["box_room", "screen_edge", "nonplanar_patch"])
def test_voxel_cone_trace_batch(oracle, built, name):
    rs, rg, ds, dg = built(name)
    g = dg.to_dict()
    rays = _random_rays(g, np.random.default_rng(7), 300)
    ref = oracle.cone_trace_batch(rg, rs, rays, want_debug=True)
    got = pcray.voxel_cone_trace(rays, dg, ds, want_debug=True)
    for f in ["ray_offset", "ie_index", "reception_point", "hit_valid", "hit_position", "hit_normal", "hit_label",
              "hit_distance"]:
        assert_fp(f, got[f], ref[f], exact=name not in NONPLANAR)
    # TraceDebug.evaluated: same set per ray (and no duplicates)
    for k in range(len(rays)):
        a = got["evaluated"][got["evaluated_offset"][k]:got["evaluated_offset"][k + 1]]
        b = ref["evaluated"][ref["evaluated_offset"][k]:ref["evaluated_offset"][k + 1]]
        assert len(a) == len(set(a.tolist()))
        assert sorted(a.tolist()) == sorted(b.tolist()), f"ray {k}"
    # TraceDebug.visited: the walker's voxels in walk order (jumps included), exactly
    assert_bitwise("visited_offset", got["visited_offset"], ref["visited_offset"])
    assert_bitwise("visited", got["visited"], ref["visited"])


@pytest.mark.parametrize("name,mi,md", [("box_room", 1, 0), ("box_room", 2, 0), ("screen_edge", 2, 1),
                                        ("wall_blocks_los", 2, 0), ("nonplanar_patch", 2, 0)])
def test_propagate(oracle, built, name, mi, md):
    rs, rg, ds, dg = built(name)
    tp = abi.trace_params(max_interactions=mi, max_diffractions=md)
    _, ref_hits = oracle.transmission_phase(rg, rs, 0, tp)
    ref = oracle.propagate(rg, rs, 0, ref_hits, tp)
    got = pcray.propagate(0, ref_hits, dg, ds, tp)
    assert_paths_equal(got, ref)


@pytest.mark.parametrize("kappa", [1, 3])
def test_propagate_kappa(oracle, built, kappa):
    rs, rg, ds, dg = built("box_room")
    tp = abi.trace_params(max_interactions=2, kappa=kappa, max_diffractions=0)
    _, ref_hits = oracle.transmission_phase(rg, rs, 0, tp)
    ref = oracle.propagate(rg, rs, 0, ref_hits, tp)
    got = pcray.propagate(0, ref_hits, dg, ds, tp)
    assert_paths_equal(got, ref)


def test_propagate_c1(oracle, gpu):
    scene, cfg = scenes.build_scene("C1")
    rs = oracle.RefScene(scene)
    rg = oracle.build_grid(rs)
    ds = pcray.DeviceScene(scene)
    dg = pcray.build_grid(ds)
    tp = abi.trace_params(max_interactions=2, max_diffractions=0)
    _, ref_hits = oracle.transmission_phase(rg, rs, 0, tp)
    _, hits = pcray.transmission_phase(0, dg, ds, tp)
    for f in ["ie_index", "kind", "position", "normal", "incoming"]:
        assert_bitwise(f, hits[f], ref_hits[f])
    ref = oracle.propagate(rg, rs, 0, ref_hits, tp)
    got = pcray.propagate(0, hits, dg, ds, tp)
    assert_paths_equal(got, ref)
