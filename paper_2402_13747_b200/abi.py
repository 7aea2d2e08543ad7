"""ctypes mirror of include/pcray_b200.h (the C-ABI drop-in boundary).

Only struct layouts and numpy<->struct conversion live here; the loaders are in
``_lib.py`` (product library) and ``oracle/ref.py`` (test-only reference build).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

PCR_OK = 0
IE_SURFACE, IE_EDGE, IE_RECEIVER = 0, 1, 2
REFLECTION, DIFFRACTION = 0, 1
RAY_MISSED, NOT_CONVERGED, OCCLUDED, DEGENERATE = 0, 1, 2, 3
MARCH_NO_IES = 2147483647
NO_IE = 0xFFFFFFFF
MAX_STAGES = 16

_pd = C.POINTER(C.c_double)
_pu32 = C.POINTER(C.c_uint32)
_pi32 = C.POINTER(C.c_int32)
_pu8 = C.POINTER(C.c_uint8)
_pu64 = C.POINTER(C.c_uint64)


class SceneDesc(C.Structure):
    _fields_ = [
        ("point_position", _pd), ("point_normal", _pd), ("point_label", _pu32), ("n_points", C.c_uint64),
        ("edge_geometry", _pd), ("edge_label", _pu32), ("n_edges", C.c_uint32),
        ("tx_position", _pd), ("tx_id", _pu32), ("n_tx", C.c_uint32),
        ("rx_position", _pd), ("rx_id", _pu32), ("n_rx", C.c_uint32),
        ("carrier_frequency_hz", C.c_double),
    ]


class VoxelParams(C.Structure):
    _fields_ = [("voxel_size", C.c_double), ("division_factor", C.c_int32), ("max_cells", C.c_uint64)]


class TraceParams(C.Structure):
    _fields_ = [("max_interactions", C.c_int32), ("kappa", C.c_int32), ("cone_apex_angle", C.c_double),
                ("diffraction_ray_count", C.c_int32), ("max_diffractions", C.c_int32)]


class RefineParams(C.Structure):
    _fields_ = [("delta", C.c_double), ("rho", C.c_int32), ("step_size", C.c_double),
                ("fresnel_enabled", C.c_int32)]


class RunConfig(C.Structure):
    _fields_ = [
        ("carrier_frequency_hz", C.c_double), ("voxel_size_m", C.c_double), ("division_factor", C.c_int32),
        ("kappa", C.c_int32), ("max_interactions", C.c_int32), ("max_diffractions", C.c_int32),
        ("cone_apex_angle_deg", C.c_double), ("diffraction_ray_count", C.c_int32), ("delta", C.c_double),
        ("rho", C.c_int32), ("step_size", C.c_double), ("seed", C.c_uint32), ("thread_count", C.c_int32),
        ("fresnel_enabled", C.c_int32),
    ]


class GridHost(C.Structure):
    _fields_ = [
        ("origin", C.c_double * 3), ("dims", C.c_int32 * 3), ("voxel_size", C.c_double),
        ("division_factor", C.c_int32), ("n_cells", C.c_uint64), ("n_ies", C.c_uint64),
        ("n_point_indices", C.c_uint64),
        ("cell_ie_begin", _pu32), ("cell_ie_end", _pu32), ("cell_march", _pi32),
        ("ie_kind", _pu8), ("ie_label", _pu32), ("ie_reception_point", _pd), ("ie_sphere_center", _pd),
        ("ie_sphere_radius", _pd), ("ie_point_begin", _pu32), ("ie_point_end", _pu32),
        ("ie_seg_start", _pd), ("ie_seg_end", _pd), ("ie_edge_index", _pu32), ("ie_rx_id", _pu32),
        ("ie_planar", _pu8), ("ie_plane_point", _pd), ("ie_plane_normal", _pd), ("ie_voxel", _pu32),
        ("ie_subvoxel", _pu32), ("point_indices", _pu32),
    ]


class Paths(C.Structure):
    _fields_ = [
        ("n", C.c_uint64), ("stride", C.c_uint32), ("tx_id", _pu32), ("rx_id", _pu32),
        ("tx_position", _pd), ("rx_position", _pd), ("length", _pd), ("delay", _pd),
        ("converged", _pu8), ("gradient_norm", _pd), ("n_inter", _pu32), ("kind", _pu8),
        ("position", _pd), ("label", _pu32), ("normal", _pd), ("ie_index", _pu32), ("edge_index", _pu32),
    ]


class InitialHits(C.Structure):
    _fields_ = [("n", C.c_uint64), ("ie_index", _pu32), ("kind", _pu8), ("position", _pd),
                ("normal", _pd), ("incoming", _pd)]


class Outcomes(C.Structure):
    _fields_ = [("paths", Paths), ("has_path", _pu8), ("reason", _pi32)]


class Summary(C.Structure):
    _fields_ = [
        ("point_count", C.c_uint64), ("edge_count", C.c_uint64), ("ie_count", C.c_uint64),
        ("grid_dims", C.c_int32 * 3), ("coarse_paths", C.c_uint64), ("refined_paths", C.c_uint64),
        ("rejected", C.c_uint64 * 4), ("exact_paths", C.c_uint64), ("n_timings", C.c_uint32),
        ("timing_stage", (C.c_char * 16) * MAX_STAGES), ("timing_seconds", C.c_double * MAX_STAGES),
        ("hash", C.c_uint64), ("paths", Paths), ("transmission_rays", C.c_uint64),
        ("cone_traces", C.c_uint64), ("visibility_tests", C.c_uint64), ("refine_iterations", C.c_uint64),
        ("refine_trials", C.c_uint64), ("refine_marches", C.c_uint64), ("walk_cells", C.c_uint64),
        ("walk_ies", C.c_uint64), ("libm_unresolved", C.c_uint64), ("refine_trial_nodes", C.c_uint64),
        ("refine_iter_nodes", C.c_uint64),
    ]


class Edges(C.Structure):
    """pcr_edges: an edges file on the host (geometry n*12: start, end, normal_a, normal_b)."""
    _fields_ = [("n", C.c_uint32), ("geometry", C.POINTER(C.c_double)), ("label", C.POINTER(C.c_uint32))]


def edges_to_dict(e: Edges) -> dict:
    n = int(e.n)
    g = np.ctypeslib.as_array(e.geometry, (12 * n + 1,))[: 12 * n].reshape(n, 12).copy()
    return {"start": g[:, 0:3], "end": g[:, 3:6], "normal_a": g[:, 6:9], "normal_b": g[:, 9:12],
            "label": np.ctypeslib.as_array(e.label, (n + 1,))[:n].copy()}


class RunFiles(C.Structure):
    """pcr_run_files: RunConfig's file paths and radio lists (pipeline.hpp:12-32)."""
    _fields_ = [("scene_path", C.c_char_p), ("edges_path", C.c_char_p), ("output_path", C.c_char_p),
                ("tx_position", C.POINTER(C.c_double)), ("n_tx", C.c_uint32),
                ("rx_position", C.POINTER(C.c_double)), ("n_rx", C.c_uint32)]


class RunFilesKeepAlive:
    """A RunFiles plus the arrays its pointers reference."""

    def __init__(self, scene_path="", edges_path="", output_path="", transmitters=(), receivers=()):
        enc = lambda p: os.fsencode(p) if p else b""  # noqa: E731
        self.tx = np.ascontiguousarray(np.asarray(transmitters, dtype=np.float64).reshape(-1, 3))
        self.rx = np.ascontiguousarray(np.asarray(receivers, dtype=np.float64).reshape(-1, 3))
        self.files = RunFiles(enc(scene_path), enc(edges_path), enc(output_path),
                              self.tx.ctypes.data_as(C.POINTER(C.c_double)), len(self.tx),
                              self.rx.ctypes.data_as(C.POINTER(C.c_double)), len(self.rx))


SHARD_STATS_FIELDS = ("cone_traces", "visibility_tests", "walk_cells", "walk_ies", "refine_iterations",
                      "refine_trials", "refine_marches", "libm_unresolved", "refine_trial_nodes",
                      "refine_iter_nodes")


class ShardStats(C.Structure):
    """pcr_shard_stats: one shard's work counters (summed over shards by the caller)."""
    _fields_ = [(f, C.c_uint64) for f in SHARD_STATS_FIELDS]


class RayDesc(C.Structure):
    _fields_ = [
        ("origin", C.c_double * 3), ("direction", C.c_double * 3), ("apex_angle", C.c_double),
        ("n_planes", C.c_int32), ("plane_point", (C.c_double * 3) * 2), ("plane_normal", (C.c_double * 3) * 2),
        ("origin_ie", C.c_uint32), ("origin_label", C.c_uint32),
    ]


class PathNode(C.Structure):
    """pcr_path_node: PathNode (refine.hpp:19-45) flattened."""
    _fields_ = [("kind", C.c_int32), ("label", C.c_uint32), ("edge_index", C.c_uint32), ("pad", C.c_uint32),
                ("c", C.c_double * 3), ("u", C.c_double * 3), ("v", C.c_double * 3), ("normal", C.c_double * 3),
                ("r", C.c_double), ("s", C.c_double), ("t_min", C.c_double), ("t_max", C.c_double)]


class Receptions(C.Structure):
    _fields_ = [
        ("n_rays", C.c_uint64), ("n", C.c_uint64), ("ray_offset", _pu64), ("ie_index", _pu32),
        ("reception_point", _pd), ("hit_valid", _pu8), ("hit_position", _pd), ("hit_normal", _pd),
        ("hit_label", _pu32), ("hit_distance", _pd), ("evaluated_offset", _pu64), ("evaluated", _pu32),
        ("visited_offset", _pu64), ("visited", _pu32),
    ]


# ----------------------------------------------------------------------------------------------
# numpy views
def _arr(ptr, n, dtype, shape=None):
    n = int(n)
    if n == 0 or not ptr:
        out = np.zeros(n, dtype=dtype)
    else:
        out = np.ctypeslib.as_array(ptr, shape=(n,)).copy().astype(dtype, copy=False)
    return out.reshape(shape) if shape is not None else out


def grid_to_dict(h: GridHost) -> dict:
    nc, ni, npi = h.n_cells, h.n_ies, h.n_point_indices
    return {
        "origin": np.array(h.origin[:], dtype=np.float64),
        "dims": np.array(h.dims[:], dtype=np.int32),
        "voxel_size": float(h.voxel_size),
        "division_factor": int(h.division_factor),
        "cell_ie_begin": _arr(h.cell_ie_begin, nc, np.uint32),
        "cell_ie_end": _arr(h.cell_ie_end, nc, np.uint32),
        "cell_march": _arr(h.cell_march, nc, np.int32),
        "ie_kind": _arr(h.ie_kind, ni, np.uint8),
        "ie_label": _arr(h.ie_label, ni, np.uint32),
        "ie_reception_point": _arr(h.ie_reception_point, 3 * ni, np.float64, (-1, 3)),
        "ie_sphere_center": _arr(h.ie_sphere_center, 3 * ni, np.float64, (-1, 3)),
        "ie_sphere_radius": _arr(h.ie_sphere_radius, ni, np.float64),
        "ie_point_begin": _arr(h.ie_point_begin, ni, np.uint32),
        "ie_point_end": _arr(h.ie_point_end, ni, np.uint32),
        "ie_seg_start": _arr(h.ie_seg_start, 3 * ni, np.float64, (-1, 3)),
        "ie_seg_end": _arr(h.ie_seg_end, 3 * ni, np.float64, (-1, 3)),
        "ie_edge_index": _arr(h.ie_edge_index, ni, np.uint32),
        "ie_rx_id": _arr(h.ie_rx_id, ni, np.uint32),
        "ie_planar": _arr(h.ie_planar, ni, np.uint8),
        "ie_plane_point": _arr(h.ie_plane_point, 3 * ni, np.float64, (-1, 3)),
        "ie_plane_normal": _arr(h.ie_plane_normal, 3 * ni, np.float64, (-1, 3)),
        "ie_voxel": _arr(h.ie_voxel, ni, np.uint32),
        "ie_subvoxel": _arr(h.ie_subvoxel, ni, np.uint32),
        "point_indices": _arr(h.point_indices, npi, np.uint32),
    }


GRID_ARRAY_FIELDS = [f for f, _ in GridHost._fields_ if f.startswith(("cell_", "ie_", "point_indices"))]


class GridKeepAlive:
    """Holds numpy buffers referenced by a GridHost built from a dict."""

    def __init__(self, g: dict):
        self.bufs = {}
        h = GridHost()
        h.origin[:] = list(map(float, g["origin"]))
        h.dims[:] = list(map(int, g["dims"]))
        h.voxel_size = float(g["voxel_size"])
        h.division_factor = int(g["division_factor"])
        h.n_cells = len(g["cell_march"])
        h.n_ies = len(g["ie_kind"])
        h.n_point_indices = len(g["point_indices"])
        for name in GRID_ARRAY_FIELDS:
            ctype = dict(GridHost._fields_)[name]._type_
            dtype = {C.c_uint32: np.uint32, C.c_int32: np.int32, C.c_uint8: np.uint8,
                     C.c_double: np.float64}[ctype]
            a = np.ascontiguousarray(np.asarray(g[name], dtype=dtype).reshape(-1))
            if a.size == 0:
                a = np.zeros(1, dtype=dtype)
            self.bufs[name] = a
            setattr(h, name, a.ctypes.data_as(C.POINTER(ctype)))
        self.host = h


def paths_to_dict(p: Paths) -> dict:
    n, s = int(p.n), int(p.stride)
    m = n * s
    return {
        "n": n,
        "stride": s,
        "tx_id": _arr(p.tx_id, n, np.uint32),
        "rx_id": _arr(p.rx_id, n, np.uint32),
        "tx_position": _arr(p.tx_position, 3 * n, np.float64, (-1, 3)),
        "rx_position": _arr(p.rx_position, 3 * n, np.float64, (-1, 3)),
        "length": _arr(p.length, n, np.float64),
        "delay": _arr(p.delay, n, np.float64),
        "converged": _arr(p.converged, n, np.uint8),
        "gradient_norm": _arr(p.gradient_norm, n, np.float64),
        "n_inter": _arr(p.n_inter, n, np.uint32),
        "kind": _arr(p.kind, m, np.uint8, (n, s)),
        "position": _arr(p.position, 3 * m, np.float64, (n, s, 3)),
        "label": _arr(p.label, m, np.uint32, (n, s)),
        "normal": _arr(p.normal, 3 * m, np.float64, (n, s, 3)),
        "ie_index": _arr(p.ie_index, m, np.uint32, (n, s)),
        "edge_index": _arr(p.edge_index, m, np.uint32, (n, s)),
    }


class PathsKeepAlive:
    """Builds a Paths struct (input direction) from a dict produced by paths_to_dict."""

    def __init__(self, d: dict):
        n, s = int(d["n"]), max(1, int(d["stride"]))
        self.bufs = []
        p = Paths()
        p.n, p.stride = n, s

        def put(name, dtype, ctype, shape):
            a = np.asarray(d.get(name, np.zeros(shape, dtype)), dtype=dtype)
            if a.size != int(np.prod(shape)):
                full = np.zeros(shape, dtype)
                if a.ndim >= 2 and a.shape[0] == n:
                    full[:, : a.shape[1]] = a
                a = full
            a = np.ascontiguousarray(a.reshape(-1))
            if a.size == 0:
                a = np.zeros(1, dtype)
            self.bufs.append(a)
            setattr(p, name, a.ctypes.data_as(C.POINTER(ctype)))

        put("tx_id", np.uint32, C.c_uint32, (n,))
        put("rx_id", np.uint32, C.c_uint32, (n,))
        put("tx_position", np.float64, C.c_double, (n, 3))
        put("rx_position", np.float64, C.c_double, (n, 3))
        put("length", np.float64, C.c_double, (n,))
        put("delay", np.float64, C.c_double, (n,))
        put("converged", np.uint8, C.c_uint8, (n,))
        put("gradient_norm", np.float64, C.c_double, (n,))
        put("n_inter", np.uint32, C.c_uint32, (n,))
        put("kind", np.uint8, C.c_uint8, (n, s))
        put("position", np.float64, C.c_double, (n, s, 3))
        put("label", np.uint32, C.c_uint32, (n, s))
        put("normal", np.float64, C.c_double, (n, s, 3))
        put("ie_index", np.uint32, C.c_uint32, (n, s))
        put("edge_index", np.uint32, C.c_uint32, (n, s))
        self.paths = p


def hits_to_dict(h: InitialHits) -> dict:
    n = int(h.n)
    return {
        "n": n,
        "ie_index": _arr(h.ie_index, n, np.uint32),
        "kind": _arr(h.kind, n, np.uint8),
        "position": _arr(h.position, 3 * n, np.float64, (-1, 3)),
        "normal": _arr(h.normal, 3 * n, np.float64, (-1, 3)),
        "incoming": _arr(h.incoming, 3 * n, np.float64, (-1, 3)),
    }


class HitsKeepAlive:
    def __init__(self, d: dict):
        n = int(d["n"])
        self.bufs = []
        h = InitialHits()
        h.n = n
        for name, dtype, ctype in [("ie_index", np.uint32, C.c_uint32), ("kind", np.uint8, C.c_uint8),
                                   ("position", np.float64, C.c_double), ("normal", np.float64, C.c_double),
                                   ("incoming", np.float64, C.c_double)]:
            a = np.ascontiguousarray(np.asarray(d[name], dtype=dtype).reshape(-1))
            if a.size == 0:
                a = np.zeros(1, dtype)
            self.bufs.append(a)
            setattr(h, name, a.ctypes.data_as(C.POINTER(ctype)))
        self.hits = h


def outcomes_to_dict(o: Outcomes) -> dict:
    d = paths_to_dict(o.paths)
    n = d["n"]
    d["has_path"] = _arr(o.has_path, n, np.uint8)
    d["reason"] = _arr(o.reason, n, np.int32)
    return d


def summary_to_dict(s: Summary) -> dict:
    return {
        "point_count": int(s.point_count), "edge_count": int(s.edge_count), "ie_count": int(s.ie_count),
        "grid_dims": list(s.grid_dims[:]), "coarse_paths": int(s.coarse_paths),
        "refined_paths": int(s.refined_paths), "rejected": [int(x) for x in s.rejected],
        "exact_paths": int(s.exact_paths),
        "timings": [(s.timing_stage[i].value.decode(), float(s.timing_seconds[i])) for i in range(s.n_timings)],
        "hash": int(s.hash), "paths": paths_to_dict(s.paths),
        "transmission_rays": int(s.transmission_rays), "cone_traces": int(s.cone_traces),
        "visibility_tests": int(s.visibility_tests), "refine_iterations": int(s.refine_iterations),
        "refine_trials": int(s.refine_trials), "refine_marches": int(s.refine_marches),
        "walk_cells": int(s.walk_cells), "walk_ies": int(s.walk_ies), "libm_unresolved": int(s.libm_unresolved),
        "refine_trial_nodes": int(s.refine_trial_nodes), "refine_iter_nodes": int(s.refine_iter_nodes),
    }


def receptions_to_dict(r: Receptions) -> dict:
    n, nr = int(r.n), int(r.n_rays)
    off = _arr(r.ray_offset, nr + 1, np.uint64)
    eoff = _arr(r.evaluated_offset, nr + 1, np.uint64)
    voff = _arr(r.visited_offset, nr + 1, np.uint64)
    return {
        "n_rays": nr, "n": n, "ray_offset": off,
        "ie_index": _arr(r.ie_index, n, np.uint32),
        "reception_point": _arr(r.reception_point, 3 * n, np.float64, (-1, 3)),
        "hit_valid": _arr(r.hit_valid, n, np.uint8),
        "hit_position": _arr(r.hit_position, 3 * n, np.float64, (-1, 3)),
        "hit_normal": _arr(r.hit_normal, 3 * n, np.float64, (-1, 3)),
        "hit_label": _arr(r.hit_label, n, np.uint32),
        "hit_distance": _arr(r.hit_distance, n, np.float64),
        "evaluated_offset": eoff,
        "evaluated": _arr(r.evaluated, int(eoff[-1]) if nr else 0, np.uint32),
        "visited_offset": voff,
        "visited": _arr(r.visited, int(voff[-1]) if nr else 0, np.uint32),
    }


# ----------------------------------------------------------------------------------------------
@dataclass
class Scene:
    """pcray::Scene (proj/include/pcray/scene.hpp:38-46) as numpy arrays."""

    position: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    normal: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    label: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    edges: np.ndarray = field(default_factory=lambda: np.zeros((0, 12)))  # start, end, normal_a, normal_b
    edge_label: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    tx: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    tx_id: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    rx: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    rx_id: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    carrier_frequency_hz: float = 60e9

    def normalized(self) -> "Scene":
        f = lambda a, dt, shp: np.ascontiguousarray(np.asarray(a, dtype=dt).reshape(shp))
        return Scene(
            f(self.position, np.float64, (-1, 3)), f(self.normal, np.float64, (-1, 3)),
            f(self.label, np.uint32, (-1,)), f(self.edges, np.float64, (-1, 12)),
            f(self.edge_label, np.uint32, (-1,)), f(self.tx, np.float64, (-1, 3)),
            f(self.tx_id, np.uint32, (-1,)), f(self.rx, np.float64, (-1, 3)),
            f(self.rx_id, np.uint32, (-1,)), float(self.carrier_frequency_hz))

    @property
    def n_points(self) -> int:
        return int(np.asarray(self.label).shape[0])


class SceneKeepAlive:
    def __init__(self, scene: Scene):
        s = scene.normalized()
        self.scene = s
        self.bufs = []
        d = SceneDesc()

        def ptr(a, ctype):
            if a.size == 0:
                a = np.zeros(1, dtype=a.dtype)
            self.bufs.append(a)
            return a.ctypes.data_as(C.POINTER(ctype))

        d.point_position = ptr(s.position, C.c_double)
        d.point_normal = ptr(s.normal, C.c_double)
        d.point_label = ptr(s.label, C.c_uint32)
        d.n_points = s.label.shape[0]
        d.edge_geometry = ptr(s.edges, C.c_double)
        d.edge_label = ptr(s.edge_label, C.c_uint32)
        d.n_edges = s.edge_label.shape[0]
        d.tx_position = ptr(s.tx, C.c_double)
        d.tx_id = ptr(s.tx_id, C.c_uint32)
        d.n_tx = s.tx_id.shape[0]
        d.rx_position = ptr(s.rx, C.c_double)
        d.rx_id = ptr(s.rx_id, C.c_uint32)
        d.n_rx = s.rx_id.shape[0]
        d.carrier_frequency_hz = s.carrier_frequency_hz
        self.desc = d


def default_run_config(**overrides) -> RunConfig:
    """RunConfig defaults (proj/include/pcray/pipeline.hpp:12-32; paper Table 1)."""
    c = RunConfig(carrier_frequency_hz=60e9, voxel_size_m=0.5, division_factor=2, kappa=100,
                  max_interactions=5, max_diffractions=1, cone_apex_angle_deg=1.0, diffraction_ray_count=360,
                  delta=1e-4, rho=2000, step_size=0.5, seed=1, thread_count=0, fresnel_enabled=1)
    for k, v in overrides.items():
        setattr(c, k, int(v) if isinstance(v, bool) else v)
    return c


def trace_params(max_interactions=5, kappa=100, cone_apex_angle=None, diffraction_ray_count=360,
                 max_diffractions=1) -> TraceParams:
    """TraceParams defaults (proj/include/pcray/tracer.hpp:16-22)."""
    if cone_apex_angle is None:
        cone_apex_angle = 1.0 * np.pi / 180.0
    return TraceParams(max_interactions, kappa, cone_apex_angle, diffraction_ray_count, max_diffractions)


def refine_params(delta=1e-4, rho=2000, step_size=0.5, fresnel_enabled=True) -> RefineParams:
    """RefineParams defaults (proj/include/pcray/refine.hpp:10-15)."""
    return RefineParams(delta, rho, step_size, int(fresnel_enabled))


def voxel_params(voxel_size=0.5, division_factor=2, max_cells=1 << 27) -> VoxelParams:
    """VoxelizationParams defaults (proj/include/pcray/voxel_grid.hpp:13-17)."""
    return VoxelParams(voxel_size, division_factor, max_cells)
