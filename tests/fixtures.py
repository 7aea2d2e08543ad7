"""Scene fixtures restating the reference's test helpers (proj/tests/test_helpers.hpp:11-45)
and the small scenes its suites build, so parity tests read like the reference's own."""
from __future__ import annotations

import math

import numpy as np

from paper_2402_13747_b200.abi import Scene


def _lround(x):
    r = math.floor(abs(x))
    if abs(x) - r >= 0.5:
        r += 1
    return int(r if x >= 0 else -r)


def _norm(v):
    v = np.asarray(v, float)
    return math.sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2])


def _normalized(v):
    v = np.asarray(v, float)
    z = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]
    return v / math.sqrt(z) if z > 0 else v


def add_wall(pts, corner, e1, e2, normal, label, spacing):
    """test_helpers.hpp:13-25: lattice patch with inclusive ends."""
    corner, e1, e2 = (np.asarray(x, float) for x in (corner, e1, e2))
    n1 = max(1, _lround(_norm(e1) / spacing))
    n2 = max(1, _lround(_norm(e2) / spacing))
    n = _normalized(normal)
    for i in range(n1 + 1):
        for j in range(n2 + 1):
            p = (corner + (float(i) / n1) * e1) + (float(j) / n2) * e2
            pts.append((p, n, label))


def box_room(size, spacing):
    """test_helpers.hpp:28-38: closed box, inward normals, labels 0..5."""
    sx, sy, sz = size
    pts = []
    add_wall(pts, (0, 0, 0), (0, sy, 0), (0, 0, sz), (1, 0, 0), 0, spacing)
    add_wall(pts, (sx, 0, 0), (0, sy, 0), (0, 0, sz), (-1, 0, 0), 1, spacing)
    add_wall(pts, (0, 0, 0), (sx, 0, 0), (0, 0, sz), (0, 1, 0), 2, spacing)
    add_wall(pts, (0, sy, 0), (sx, 0, 0), (0, 0, sz), (0, -1, 0), 3, spacing)
    add_wall(pts, (0, 0, 0), (sx, 0, 0), (0, sy, 0), (0, 0, 1), 4, spacing)
    add_wall(pts, (0, 0, sz), (sx, 0, 0), (0, sy, 0), (0, 0, -1), 5, spacing)
    return pts


def make_scene(points=(), tx=((0.2, 0.2, 0.2),), rx=((0.3, 0.3, 0.3),), edges=()) -> Scene:
    """scene_with_radios (test_helpers.hpp:40-45) generalised to lists; edges as
    (start, end, normal_a, normal_b, label)."""
    pts = list(points)
    pos = np.array([p for p, _, _ in pts], float).reshape(-1, 3)
    nrm = np.array([n for _, n, _ in pts], float).reshape(-1, 3)
    lab = np.array([l for _, _, l in pts], np.uint32)
    eg = np.array([[*s, *e, *a, *b] for s, e, a, b, _ in edges], float).reshape(-1, 12)
    el = np.array([l for *_, l in edges], np.uint32)
    tx = np.asarray(tx, float).reshape(-1, 3)
    rx = np.asarray(rx, float).reshape(-1, 3)
    return Scene(pos, nrm, lab, eg, el, tx, np.arange(len(tx), dtype=np.uint32), rx,
                 np.arange(len(rx), dtype=np.uint32))


def random_points(seed, n, lo, hi, normal=(0, 0, 1), n_labels=1):
    rng = np.random.default_rng(seed)
    p = rng.uniform(lo, hi, size=(n, 3))
    return [(p[i], np.asarray(normal, float), i % n_labels) for i in range(n)]


# ---- the reference's test scenes (names point at the test that builds them) ------------------
def voxel_grid_scenes():
    """Scenes of proj/tests/test_voxel_grid.cpp plus a few edge cases."""
    out = {}
    out["single_point"] = make_scene([((0.1, 0.1, 0.1), (0, 0, 1), 0)], tx=[(0.1, 0.1, 0.1)], rx=[(0.1, 0.1, 0.1)])
    out["two_labels"] = make_scene([((0.10, 0.10, 0.10), (0, 0, 1), 1), ((0.11, 0.11, 0.11), (0, 0, 1), 2)])
    out["edge_clip"] = make_scene(edges=[((0, 0, 0), (1, 0, 0), (0, 0, 1), (0, -1, 0), 5)])
    out["reception_points"] = make_scene(
        [((1.00, 1.0, 1.0), (0, 0, 1), 0), ((1.05, 1.0, 1.0), (0, 0, 1), 0)], rx=[(3, 2, 1)],
        edges=[((2, 2, 2), (2, 2, 2.25), (1, 0, 0), (0, 1, 0), 5)])
    out["partition"] = make_scene(random_points(7, 500, -2.0, 2.0, n_labels=3))
    out["march_corner"] = make_scene([((0.25, 0.25, 0.25), (0, 0, 1), 0)], tx=[(0.25, 0.25, 0.25)],
                                     rx=[(1.25, 1.25, 1.25)])
    out["determinism"] = make_scene(random_points(3, 300, -1.0, 3.0, normal=(0, 1, 0), n_labels=4),
                                    edges=[((0, 0, 0), (2, 0, 0), (0, 0, 1), (0, -1, 0), 99)])
    out["distance_field"] = make_scene(random_points(11, 40, 0.0, 4.0))
    out["radios_only"] = make_scene()
    out["oblique_edge"] = make_scene(edges=[((0.13, -0.4, 0.2), (1.9, 1.1, 0.95), (0, 0, 1), (0.6, -0.8, 0), 7),
                                            ((1.0, 1.0, 0.0), (1.0, 1.0, 2.0), (1, 0, 0), (0, 1, 0), 8)])
    out["big_labels"] = make_scene([((0.1 * i, 0.05 * i, 0.0), (0, 0, 1), 4000000000 - i) for i in range(50)])
    out["dup_rx_ids"] = Scene(
        np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0, np.uint32), np.zeros((0, 12)), np.zeros(0, np.uint32),
        np.array([[0, 0, 0.0]]), np.array([0], np.uint32), np.array([[1, 1, 1.0], [1.05, 1, 1.0], [2, 2, 2.0]]),
        np.array([3, 3, 1], np.uint32))
    pts = box_room((2, 2, 2), 0.05)
    out["box_room"] = make_scene(pts, tx=[(0.6, 0.7, 0.9)], rx=[(1.3, 1.2, 1.1)])
    # non-planar: jittered normals on a tilted patch
    rng = np.random.default_rng(5)
    npts = []
    for i in range(-5, 6):
        for j in range(-5, 6):
            n = _normalized(np.array([0.05 * rng.standard_normal(), 0.05 * rng.standard_normal(), 1.0]))
            npts.append(((0.03 * i, 0.03 * j, 0.01 * i), n, 0))
    out["nonplanar_patch"] = make_scene(npts)
    return out
