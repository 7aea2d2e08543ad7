"""Synthetic labeled planar scenes for parity tests and the benchmark.

Every scene is a set of rectangles (corner, e1, e2, label; e1 x e2 is the outward
normal) plus optional diffraction edges, sampled into a labeled point cloud with
the reference's own stratified-jitter rule (proj/src/oracle.cpp:208-236):

    rng = std::mt19937(seed); jitter = uniform_real_distribution<double>(0, 1)
    per rectangle: nu = max(1, lround(|e1| sqrt(density))), nv likewise,
    n = normalize(e1 x e2), point(i, j) = (corner + u e1) + v e2,
    u = (i + jitter) / nu, v = (j + jitter) / nv   (u drawn before v)

`sample_planar_scene` reproduces that bit for bit in numpy: numpy's MT19937 with
legacy seeding is init_genrand (= std::mt19937(seed)), and libstdc++'s
generate_canonical<double, 53> consumes two 32-bit draws as
(lo + hi * 2^32) / 2^64 (clamped below 1). tests/test_scenes.py pins this
against the reference sampler compiled in oracle/_ref. The scene is input
synthesis, not part of the measured path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .abi import Scene

_TWO32 = 4294967296.0
_TWO64 = 18446744073709551616.0


@dataclass
class PlanarScene:
    """pcray::PlanarScene (proj/include/pcray/oracle.hpp:12-27)."""

    rects: list = field(default_factory=list)  # (corner, e1, e2, label)
    edges: list = field(default_factory=list)  # (start, end, normal_a, normal_b, label)
    tx: list = field(default_factory=list)
    rx: list = field(default_factory=list)

    def add_rect(self, corner, e1, e2, label):
        self.rects.append((np.asarray(corner, float), np.asarray(e1, float), np.asarray(e2, float), int(label)))
        return self

    def rect_array(self) -> np.ndarray:
        """n_rect x 10 doubles (corner, e1, e2, label) — the oracle's sampler input."""
        return np.array([[*c, *a, *b, float(l)] for c, a, b, l in self.rects], dtype=np.float64).reshape(-1, 10)


def _dot(a, b):
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]


def _norm(a):
    return math.sqrt(_dot(a, a))


def _cross(a, b):
    return np.array([a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]])


def _normalized(a):
    z = _dot(a, a)
    return a / math.sqrt(z) if z > 0 else a


def _lround(x: float) -> int:
    r = math.floor(abs(x))
    if abs(x) - r >= 0.5:
        r += 1
    return int(r if x >= 0 else -r)


def _canonical(raw: np.ndarray) -> np.ndarray:
    lo = raw[0::2].astype(np.float64)
    hi = raw[1::2].astype(np.float64)
    r = (lo + hi * _TWO32) / _TWO64
    r[r >= 1.0] = np.nextafter(1.0, 0.0)
    return r * (1.0 - 0.0) + 0.0


def sample_planar_scene(planar: PlanarScene, density: float, seed: int):
    """Bit-exact numpy restatement of pcray::sample_planar_scene (oracle.cpp:208-227)."""
    bg = np.random.MT19937(0)
    bg._legacy_seeding(int(seed) & 0xFFFFFFFF)
    sq = math.sqrt(density)
    pos, nrm, lab = [], [], []
    for corner, e1, e2, label in planar.rects:
        nu = max(1, _lround(_norm(e1) * sq))
        nv = max(1, _lround(_norm(e2) * sq))
        n = _normalized(_cross(e1, e2))
        m = nu * nv
        raw = bg.random_raw(4 * m).astype(np.uint64)
        jit = _canonical(raw).reshape(m, 2)
        i = np.repeat(np.arange(nu, dtype=np.float64), nv)
        j = np.tile(np.arange(nv, dtype=np.float64), nu)
        u = (i + jit[:, 0]) / nu
        v = (j + jit[:, 1]) / nv
        p = (corner[None, :] + u[:, None] * e1[None, :]) + v[:, None] * e2[None, :]
        pos.append(p)
        nrm.append(np.broadcast_to(n, (m, 3)))
        lab.append(np.full(m, label, dtype=np.uint32))
    if not pos:
        return np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0, np.uint32)
    return (np.ascontiguousarray(np.concatenate(pos)), np.ascontiguousarray(np.concatenate(nrm)),
            np.concatenate(lab))


def scene_from_planar(planar: PlanarScene, density: float, seed: int, carrier_frequency_hz=60e9) -> Scene:
    """pcray::scene_from_planar (oracle.cpp:229-236), generalised to radio lists (ids 0..n-1 as
    run_pipeline assigns them, pipeline.cpp:224-231)."""
    pos, nrm, lab = sample_planar_scene(planar, density, seed)
    edges = np.array([[*s, *e, *na, *nb] for s, e, na, nb, _ in planar.edges], dtype=np.float64).reshape(-1, 12)
    elab = np.array([l for *_, l in planar.edges], dtype=np.uint32)
    tx = np.asarray(planar.tx, dtype=np.float64).reshape(-1, 3)
    rx = np.asarray(planar.rx, dtype=np.float64).reshape(-1, 3)
    return Scene(pos, nrm, lab, edges, elab, tx, np.arange(len(tx), dtype=np.uint32), rx,
                 np.arange(len(rx), dtype=np.uint32), carrier_frequency_hz)


# ---------------------------------------------------------------------------------------------
# geometry builders
def box_planar(size, tx=None, rx=None) -> PlanarScene:
    """Six inward-facing rectangles, labels 0..5 (acceptance_main.cpp:68-80)."""
    sx, sy, sz = size
    s = PlanarScene()
    s.add_rect((0, 0, 0), (0, sy, 0), (0, 0, sz), 0)
    s.add_rect((sx, 0, 0), (0, 0, sz), (0, sy, 0), 1)
    s.add_rect((0, 0, 0), (0, 0, sz), (sx, 0, 0), 2)
    s.add_rect((0, sy, 0), (sx, 0, 0), (0, 0, sz), 3)
    s.add_rect((0, 0, 0), (sx, 0, 0), (0, sy, 0), 4)
    s.add_rect((0, 0, sz), (0, sy, 0), (sx, 0, 0), 5)
    if tx is not None:
        s.tx.append(list(tx))
    if rx is not None:
        s.rx.append(list(rx))
    return s


def _box_outward(s: PlanarScene, lo, hi, label0, top=True, bottom=False):
    """Axis-aligned solid box with outward-facing side faces (+ optional top/bottom)."""
    (x0, y0, z0), (x1, y1, z1) = lo, hi
    dx, dy, dz = x1 - x0, y1 - y0, z1 - z0
    lab = label0
    s.add_rect((x0, y0, z0), (0, 0, dz), (0, dy, 0), lab); lab += 1        # -x face: e1 x e2 = -x
    s.add_rect((x1, y0, z0), (0, dy, 0), (0, 0, dz), lab); lab += 1        # +x
    s.add_rect((x0, y0, z0), (dx, 0, 0), (0, 0, dz), lab); lab += 1        # -y
    s.add_rect((x0, y1, z0), (0, 0, dz), (dx, 0, 0), lab); lab += 1        # +y
    if top:
        s.add_rect((x0, y0, z1), (dx, 0, 0), (0, dy, 0), lab); lab += 1    # +z
    if bottom:
        s.add_rect((x0, y0, z0), (0, dy, 0), (dx, 0, 0), lab); lab += 1    # -z
    return lab


def office_planar() -> PlanarScene:
    """C2: 20 x 10 x 3 m office shell + 4 pillars (0.6 x 0.6 x 3) + 6 desks (2 x 1 x 0.75).

    Diffraction edges: the 4 vertical edges of every pillar and the 4 top edges of
    every desk (labels >= 1000, disjoint from the surface labels)."""
    s = box_planar((20.0, 10.0, 3.0))
    lab = 6
    pillars = [(5.0, 3.0), (15.0, 3.0), (5.0, 7.0), (15.0, 7.0)]
    desks = [(2.0, 1.0), (8.0, 1.0), (12.0, 1.0), (2.0, 8.0), (8.0, 8.0), (12.0, 8.0)]
    edge_label = 1000
    for (cx, cy) in pillars:
        lo, hi = (cx - 0.3, cy - 0.3, 0.0), (cx + 0.3, cy + 0.3, 3.0)
        lab = _box_outward(s, lo, hi, lab, top=False)
        for (ex, ey, na, nb) in [(lo[0], lo[1], (-1, 0, 0), (0, -1, 0)), (hi[0], lo[1], (1, 0, 0), (0, -1, 0)),
                                 (lo[0], hi[1], (-1, 0, 0), (0, 1, 0)), (hi[0], hi[1], (1, 0, 0), (0, 1, 0))]:
            s.edges.append(((ex, ey, 0.0), (ex, ey, 3.0), na, nb, edge_label)); edge_label += 1
    for (x0, y0) in desks:
        lo, hi = (x0, y0, 0.0), (x0 + 2.0, y0 + 1.0, 0.75)
        lab = _box_outward(s, lo, hi, lab, top=True)
        z = 0.75
        s.edges.append(((x0, y0, z), (x0 + 2.0, y0, z), (0, 0, 1), (0, -1, 0), edge_label)); edge_label += 1
        s.edges.append(((x0, y0 + 1.0, z), (x0 + 2.0, y0 + 1.0, z), (0, 0, 1), (0, 1, 0), edge_label)); edge_label += 1
        s.edges.append(((x0, y0, z), (x0, y0 + 1.0, z), (0, 0, 1), (-1, 0, 0), edge_label)); edge_label += 1
        s.edges.append(((x0 + 2.0, y0, z), (x0 + 2.0, y0 + 1.0, z), (0, 0, 1), (1, 0, 0), edge_label)); edge_label += 1
    s.tx.append([3.1, 4.3, 2.2])
    for i in range(8):
        for j in range(8):
            s.rx.append([1.3 + 2.4 * i, 0.7 + 1.2 * j, 1.2])
    return s


def canyon_planar(n_tx=4, n_rx=256) -> PlanarScene:
    """C3: street canyon — ground 200 x 20 m and two 200 x 30 m facade rows split into
    10 buildings each (labels 1..20), radios at street level."""
    s = PlanarScene()
    s.add_rect((0, 0, 0), (200.0, 0, 0), (0, 20.0, 0), 0)  # ground, +z
    lab = 1
    for b in range(10):
        x0 = 20.0 * b
        s.add_rect((x0, 0, 0), (0, 0, 30.0), (20.0, 0, 0), lab); lab += 1     # y=0 facade, +y
        s.add_rect((x0, 20.0, 0), (20.0, 0, 0), (0, 0, 30.0), lab); lab += 1  # y=20 facade, -y
    for t in range(n_tx):
        s.tx.append([25.0 + 50.0 * t + 0.37, 6.3 + 1.1 * t, 6.0 + 0.5 * t])
    per_lane = max(1, n_rx // 4)
    for lane in range(4):
        for i in range(per_lane):
            if len(s.rx) >= n_rx:
                break
            s.rx.append([1.0 + (198.0 / per_lane) * i + 0.13 * lane, 3.5 + 4.3 * lane, 1.5])
    return s


def dense_floor_planar(n_rx_per_room=64) -> PlanarScene:
    """C4: 40 x 40 x 3 m floor, 4 x 4 rooms of 10 x 10 m; 0.1 m thick partitions with a
    1 m door per room side; door jambs are diffraction edges (labels >= 10000)."""
    s = box_planar((40.0, 40.0, 3.0))
    lab = 6
    edge_label = 10000
    th = 0.1
    for axis in (0, 1):
        for k in (1, 2, 3):
            c = 10.0 * k
            for seg in range(4):
                a0, a1 = 10.0 * seg, 10.0 * seg + 10.0
                d0, d1 = a0 + 4.5, a0 + 5.5  # door opening
                for (p0, p1) in [(a0, d0), (d1, a1)]:
                    if axis == 0:  # wall at x = c, spanning y in [p0, p1]
                        lo, hi = (c - th / 2, p0, 0.0), (c + th / 2, p1, 3.0)
                        s.add_rect((lo[0], p0, 0), (0, 0, 3.0), (0, p1 - p0, 0), lab); lab += 1       # -x face
                        s.add_rect((hi[0], p0, 0), (0, p1 - p0, 0), (0, 0, 3.0), lab); lab += 1       # +x face
                    else:  # wall at y = c spanning x in [p0, p1]
                        lo, hi = (p0, c - th / 2, 0.0), (p1, c + th / 2, 3.0)
                        s.add_rect((p0, lo[1], 0), (p1 - p0, 0, 0), (0, 0, 3.0), lab); lab += 1       # -y face
                        s.add_rect((p0, hi[1], 0), (0, 0, 3.0), (p1 - p0, 0, 0), lab); lab += 1       # +y face
                for dz in (d0, d1):
                    if axis == 0:
                        for side, nx in ((c - th / 2, -1.0), (c + th / 2, 1.0)):
                            ny = 1.0 if dz == d0 else -1.0
                            s.edges.append(((side, dz, 0.0), (side, dz, 3.0), (nx, 0, 0), (0, ny, 0), edge_label))
                            edge_label += 1
                    else:
                        for side, ny in ((c - th / 2, -1.0), (c + th / 2, 1.0)):
                            nx = 1.0 if dz == d0 else -1.0
                            s.edges.append(((dz, side, 0.0), (dz, side, 3.0), (0, ny, 0), (nx, 0, 0), edge_label))
                            edge_label += 1
    for i in range(4):
        for j in range(4):
            s.tx.append([10.0 * i + 3.3, 10.0 * j + 6.1, 2.4])
            side = int(math.isqrt(n_rx_per_room))
            for a in range(side):
                for b in range(side):
                    s.rx.append([10.0 * i + 1.1 + 8.0 * a / max(1, side - 1) * 0.98,
                                 10.0 * j + 1.2 + 8.0 * b / max(1, side - 1) * 0.97, 1.3])
    return s


# ---------------------------------------------------------------------------------------------
@dataclass
class SceneConfig:
    name: str
    planar: PlanarScene
    density: float
    seed: int
    run: dict  # RunConfig overrides
    note: str = ""


def config(name: str) -> SceneConfig:
    """The BASELINE.json configs as concrete scenes."""
    if name == "C1":
        p = box_planar((4.0, 3.0, 2.5), (1.07, 0.83, 1.12), (2.71, 2.29, 1.57))
        return SceneConfig("C1", p, 1700.0, 7, dict(max_interactions=2, max_diffractions=0),
                           "synthetic labeled box room, 100k points, 1 TX / 1 RX, max 2 reflections")
    if name == "C2":
        # "3 reflections + 1 diffraction" = 4 interactions; the reference caps only the
        # total and the diffraction count (tracer.cpp:418-472), SURVEY.md §8.0
        return SceneConfig("C2", office_planar(), 1545.0, 11, dict(max_interactions=4, max_diffractions=1),
                           "synthetic indoor office, 1M points, 1 TX / 64 RX, 4 interactions incl. <= 1 diffraction")
    if name == "C2d3":
        return SceneConfig("C2d3", office_planar(), 1545.0, 11, dict(max_interactions=3, max_diffractions=1),
                           "C2 at depth 3 (secondary, shallower than the contract's 4 / 1)")
    if name == "C2np":
        return SceneConfig("C2np", office_planar(), 1545.0, 11, dict(max_interactions=4, max_diffractions=1),
                           "C2 with every normal tilted by up to 1 deg (seeded): non-planar IEs, exp() SDF path")
    if name == "C3":
        return SceneConfig("C3", canyon_planar(), 625.0, 3, dict(max_interactions=3, max_diffractions=0),
                           "synthetic street canyon, 10M points, 4 TX / 256 RX, 3 reflections")
    if name == "C4":
        return SceneConfig("C4", dense_floor_planar(), 1950.0, 5, dict(max_interactions=5, max_diffractions=1),
                           "dense synthetic floor, 10M points, 16 TX / 1024 RX, 5 interactions incl. <= 1 diffraction")
    raise KeyError(name)


def scaled_density(cfg: SceneConfig, target_points: int) -> float:
    """Density that gives ~target_points for cfg's rectangles (C5 sweep)."""
    area = sum(_norm(e1) * _norm(e2) for _, e1, e2, _ in cfg.planar.rects)
    return target_points / area


def jitter_normals(scene: Scene, max_deg: float, seed: int) -> Scene:
    """Tilt every normal by a random angle in [0, max_deg] about a random axis
    perpendicular to it; the result is renormalised."""
    rng = np.random.default_rng(seed)
    n = np.asarray(scene.normal, dtype=np.float64)
    a = rng.normal(size=n.shape)
    a -= (a * n).sum(1, keepdims=True) * n
    a /= np.linalg.norm(a, axis=1, keepdims=True)
    th = np.radians(rng.uniform(0.0, max_deg, size=(len(n), 1)))
    out = n * np.cos(th) + a * np.sin(th)
    out /= np.linalg.norm(out, axis=1, keepdims=True)
    return Scene(scene.position, out, scene.label, scene.edges, scene.edge_label, scene.tx, scene.tx_id, scene.rx,
                 scene.rx_id, scene.carrier_frequency_hz)


def build_scene(name: str, density: float | None = None) -> tuple[Scene, SceneConfig]:
    cfg = config(name)
    scene = scene_from_planar(cfg.planar, density or cfg.density, cfg.seed)
    if name == "C2np":
        scene = jitter_normals(scene, 1.0, cfg.seed)
    return scene, cfg
