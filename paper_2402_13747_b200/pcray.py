"""Python mirror of the reference's C++ API (namespace ``pcray``) over the B200 C ABI.

Each function forwards to one ``pcr_*`` entry point of libpcray_b200.so (see
include/pcray_b200.h) and keeps the reference's name, argument meaning, output
order and error text. There is no CPU path: if the CUDA library is missing or no
GPU is visible, calls raise ``PcrError`` — nothing falls back to the oracle.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import abi
from .abi import (RunConfig, Scene, TraceParams, RefineParams, VoxelParams, default_run_config, refine_params,
                  trace_params, voxel_params)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpcray_b200.so")

_lib = None


class PcrError(RuntimeError):
    """std::runtime_error of the reference; .code is the pcr_status."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def lib():
    """Load the in-tree CUDA library (fails loudly when it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise PcrError(2, f"CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        vp, pp = C.c_void_p, C.POINTER
        L.pcr_abi_version.restype = C.c_int
        L.pcr_create.argtypes = [C.c_int, pp(vp)]
        L.pcr_destroy.argtypes = [vp]
        L.pcr_last_error.restype = C.c_char_p
        L.pcr_last_error.argtypes = [vp]
        L.pcr_kernel_launches.restype = C.c_uint64
        L.pcr_scene_upload.argtypes = [vp, pp(abi.SceneDesc), pp(vp)]
        L.pcr_scene_free.argtypes = [vp]
        L.pcr_build_grid.argtypes = [vp, vp, pp(abi.VoxelParams), pp(vp)]
        L.pcr_grid_upload.argtypes = [vp, pp(abi.GridHost), pp(vp)]
        L.pcr_compute_march_distances.argtypes = [vp, vp]
        L.pcr_grid_download.argtypes = [vp, vp, pp(pp(abi.GridHost))]
        L.pcr_grid_free.argtypes = [vp]
        L.pcr_free_grid_host.argtypes = [pp(abi.GridHost)]
        L.pcr_transmission_phase.argtypes = [vp, vp, vp, C.c_uint32, pp(abi.TraceParams), pp(pp(abi.Paths)),
                                             pp(pp(abi.InitialHits))]
        L.pcr_propagate.argtypes = [vp, vp, vp, C.c_uint32, pp(abi.InitialHits), pp(abi.TraceParams),
                                    pp(pp(abi.Paths))]
        L.pcr_last_trace_stats.argtypes = [vp, pp(C.c_uint64)]
        L.pcr_grid_part_build.argtypes = [vp, vp, pp(abi.VoxelParams), C.c_uint32, C.c_uint32, pp(C.c_uint64)]
        L.pcr_grid_part_copy.argtypes = [vp, vp]
        L.pcr_grid_assemble.argtypes = [vp, vp, pp(C.c_uint64), pp(C.c_uint64), C.c_uint32, pp(vp)]
        pd, pu32, pu8 = pp(C.c_double), pp(C.c_uint32), pp(C.c_uint8)
        L.pcr_estimate_surface_batch.argtypes = [vp, vp, vp, pd, pu32, C.c_uint64, pd, pd, pd, pd]
        L.pcr_march_segment_batch.argtypes = [vp, vp, vp, pd, pd, pu32, pd, C.c_uint64, pu8, pd, pd, pu32, pd]
        L.pcr_project_to_surface_batch.argtypes = [vp, vp, vp, pd, pu32, C.c_uint64, pu8, pd, pd, pu32]
        L.pcr_local_frame_batch.argtypes = [vp, pd, C.c_uint64, pd, pd]
        L.pcr_reception_point_batch.argtypes = [vp, vp, vp, pu32, C.c_uint64, pd]
        L.pcr_cone_intersects_sphere_batch.argtypes = [vp, pd, pd, pd, pd, pd, C.c_uint64, pu8]
        L.pcr_reflect_ray_batch.argtypes = [vp, vp, pd, pd, pd, C.c_uint64, pp(abi.TraceParams), pu8,
                                            pp(abi.RayDesc)]
        L.pcr_diffract_rays.argtypes = [vp, vp, C.c_uint32, pd, pd, pp(abi.TraceParams), pp(pp(abi.RayDesc)),
                                        pp(C.c_uint64)]
        L.pcr_free_rays.argtypes = [pp(abi.RayDesc)]
        L.pcr_free_rays.restype = None
        L.pcr_make_path_state.argtypes = [vp, vp, pp(abi.Paths), pp(abi.PathNode)]
        L.pcr_path_eval_batch.argtypes = [vp, pd, pd, pu32, pp(abi.PathNode), C.c_uint32, C.c_uint64, pd, pd, pu8]
        L.pcr_cone_trace_batch.argtypes = [vp, vp, vp, pp(abi.RayDesc), C.c_uint64, C.c_int,
                                           pp(pp(abi.Receptions))]
        L.pcr_segment_visible_batch.argtypes = [vp, vp, vp, pp(C.c_double), pp(C.c_double), pp(C.c_uint32),
                                                C.c_uint64, pp(C.c_uint8)]
        L.pcr_refine_batch.argtypes = [vp, vp, vp, pp(abi.Paths), pp(abi.RefineParams), pp(pp(abi.Outcomes))]
        L.pcr_run_pipeline_on_scene.argtypes = [vp, pp(abi.SceneDesc), pp(abi.RunConfig), pp(pp(abi.Summary))]
        L.pcr_run_pipeline_device.argtypes = [vp, vp, pp(abi.RunConfig), pp(pp(abi.Summary))]
        L.pcr_scene_load_ply.argtypes = [vp, C.c_char_p, pp(abi.SceneDesc), pp(vp)]
        L.pcr_scene_points.argtypes = [vp, vp, pp(C.c_double), pp(C.c_double), pp(C.c_uint32), pp(C.c_uint64)]
        L.pcr_write_paths.argtypes = [vp, C.c_char_p, pp(abi.Paths), C.c_uint64]
        L.pcr_load_edges.argtypes = [vp, C.c_char_p, pp(pp(abi.Edges))]
        L.pcr_free_edges.argtypes = [pp(abi.Edges)]
        L.pcr_free_edges.restype = None
        L.pcr_run_pipeline.argtypes = [vp, pp(abi.RunFiles), pp(abi.RunConfig), pp(pp(abi.Summary))]
        L.pcr_shard_trace.argtypes = [vp, vp, pp(abi.RunConfig), C.c_uint32, C.c_uint32, pp(C.c_uint64),
                                      pp(C.c_uint64)]
        L.pcr_shard_rows.argtypes = [vp, vp]
        L.pcr_shard_trace_grid.argtypes = [vp, vp, vp, pp(abi.RunConfig), C.c_uint32, C.c_uint32, pp(C.c_uint64),
                                           pp(C.c_uint64)]
        L.pcr_shard_refine.argtypes = [vp, vp, vp, C.c_uint64, pp(C.c_uint64), pp(C.c_uint64)]
        L.pcr_shard_outcomes.argtypes = [vp, vp]
        L.pcr_shard_stats_get.argtypes = [vp, pp(abi.ShardStats)]
        L.pcr_shard_finish.argtypes = [vp, vp, C.c_uint64, pp(abi.ShardStats), pp(pp(abi.Summary))]
        L.pcr_stream.restype = vp
        L.pcr_stream.argtypes = [vp]
        L.pcr_set_profiling.argtypes = [vp, C.c_int]
        L.pcr_kernel_times.argtypes = [vp, vp, pp(C.c_double), pp(C.c_uint64), C.c_int, C.c_int]
        L.pcr_transfer_bytes.argtypes = [pp(C.c_uint64), pp(C.c_uint64)]
        L.pcr_fp64_probe.argtypes = [vp, pp(C.c_double)]
        L.pcr_libm_exp_batch.argtypes = [vp, pp(C.c_double), pp(C.c_double), C.c_uint64]
        L.pcr_config_hash.restype = C.c_uint64
        L.pcr_config_hash.argtypes = [pp(abi.RunConfig)]
        L.pcr_run_config_defaults.argtypes = [pp(abi.RunConfig)]
        for name, t in [("pcr_free_paths", abi.Paths), ("pcr_free_initial_hits", abi.InitialHits),
                        ("pcr_free_outcomes", abi.Outcomes), ("pcr_free_summary", abi.Summary),
                        ("pcr_free_receptions", abi.Receptions)]:
            getattr(L, name).argtypes = [pp(t)]
        if L.pcr_abi_version() != 1:
            raise PcrError(1, "ABI version mismatch")
        _lib = L
    return _lib


EXPORTED_SYMBOLS = [
    "pcr_abi_version", "pcr_create", "pcr_destroy", "pcr_last_error", "pcr_scene_upload", "pcr_scene_free",
    "pcr_build_grid", "pcr_grid_upload", "pcr_compute_march_distances", "pcr_grid_download", "pcr_grid_free",
    "pcr_free_grid_host", "pcr_transmission_phase", "pcr_propagate", "pcr_cone_trace_batch",
    "pcr_segment_visible_batch", "pcr_refine_batch", "pcr_run_pipeline_on_scene", "pcr_config_hash",
    "pcr_run_config_defaults", "pcr_free_paths", "pcr_free_initial_hits", "pcr_free_outcomes",
    "pcr_free_summary", "pcr_free_receptions", "pcr_run_pipeline_device", "pcr_shard_trace", "pcr_shard_rows",
    "pcr_shard_refine", "pcr_shard_outcomes", "pcr_shard_stats_get", "pcr_shard_finish", "pcr_scene_load_ply",
    "pcr_scene_points", "pcr_write_paths", "pcr_libm_exp_batch", "pcr_load_edges", "pcr_free_edges",
    "pcr_run_pipeline", "pcr_last_trace_stats", "pcr_estimate_surface_batch", "pcr_march_segment_batch",
    "pcr_project_to_surface_batch", "pcr_local_frame_batch", "pcr_cone_intersects_sphere_batch",
    "pcr_reflect_ray_batch", "pcr_diffract_rays", "pcr_free_rays", "pcr_make_path_state", "pcr_path_eval_batch",
    "pcr_reception_point_batch", "pcr_grid_part_build", "pcr_grid_part_copy", "pcr_grid_assemble",
    "pcr_shard_trace_grid",
]


class Context:
    """One device context (pcr_create). Calls on one context are serialised."""

    _default = None

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        rc = lib().pcr_create(device, C.byref(h))
        if rc != 0:
            raise PcrError(rc, f"pcr_create(device={device}) failed (no CUDA device?)")
        self.handle = h

    @classmethod
    def default(cls) -> "Context":
        if cls._default is None:
            cls._default = Context(int(os.environ.get("PCR_DEVICE", "0")))
        return cls._default

    def check(self, rc: int):
        if rc != 0:
            raise PcrError(rc, lib().pcr_last_error(self.handle).decode())

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.pcr_destroy(self.handle)
            self.handle = None


def kernel_launches() -> int:
    """Number of library kernel launches so far in this process."""
    return int(lib().pcr_kernel_launches())


class DeviceScene:
    """Scene resident on the GPU (pcr_scene_upload)."""

    def __init__(self, scene: Scene, ctx: Context | None = None):
        self.ctx = ctx or Context.default()
        self.keep = abi.SceneKeepAlive(scene)
        self.scene = self.keep.scene
        h = C.c_void_p()
        self.ctx.check(lib().pcr_scene_upload(self.ctx.handle, C.byref(self.keep.desc), C.byref(h)))
        self.handle = h

    @classmethod
    def from_ply(cls, path: str, rest: Scene | None = None, ctx: Context | None = None,
                 host_mirror: bool = True) -> "DeviceScene":
        """pcray::load_point_cloud (io.hpp:15) straight into HBM (pcr_scene_load_ply); `rest`
        supplies edges, radios and the carrier frequency (its points are ignored).
        host_mirror=False skips reading the points back into `.scene`."""
        self = cls.__new__(cls)
        self.ctx = ctx or Context.default()
        self.keep = abi.SceneKeepAlive(rest or Scene())
        h = C.c_void_p()
        self.ctx.check(lib().pcr_scene_load_ply(self.ctx.handle, os.fsencode(path), C.byref(self.keep.desc),
                                                C.byref(h)))
        self.handle = h
        r = self.keep.scene
        if not host_mirror:
            self.scene = r
            return self
        pts = self.points()
        self.scene = Scene(pts["position"], pts["normal"], pts["label"], r.edges, r.edge_label, r.tx, r.tx_id,
                           r.rx, r.rx_id, r.carrier_frequency_hz)
        return self

    def points(self) -> dict:
        """The resident points back on the host (pcr_scene_points)."""
        n = C.c_uint64()
        self.ctx.check(lib().pcr_scene_points(self.ctx.handle, self.handle, None, None, None, C.byref(n)))
        k = n.value
        pos, nrm, lab = np.zeros((k, 3)), np.zeros((k, 3)), np.zeros(k, np.uint32)
        dp = C.POINTER(C.c_double)
        self.ctx.check(lib().pcr_scene_points(self.ctx.handle, self.handle, pos.ctypes.data_as(dp),
                                              nrm.ctypes.data_as(dp), lab.ctypes.data_as(C.POINTER(C.c_uint32)),
                                              C.byref(n)))
        return {"position": pos, "normal": nrm, "label": lab}

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.pcr_scene_free(self.handle)
            self.handle = None


class DeviceGrid:
    """VoxelGrid resident on the GPU; .to_dict() is the host VoxelGrid mirror."""

    def __init__(self, handle, ctx: Context):
        self.handle = handle
        self.ctx = ctx

    @classmethod
    def from_dict(cls, g: dict, ctx: Context | None = None) -> "DeviceGrid":
        ctx = ctx or Context.default()
        keep = abi.GridKeepAlive(g)
        h = C.c_void_p()
        ctx.check(lib().pcr_grid_upload(ctx.handle, C.byref(keep.host), C.byref(h)))
        return cls(h, ctx)

    def to_dict(self) -> dict:
        out = C.POINTER(abi.GridHost)()
        self.ctx.check(lib().pcr_grid_download(self.ctx.handle, self.handle, C.byref(out)))
        try:
            return abi.grid_to_dict(out.contents)
        finally:
            lib().pcr_free_grid_host(out)

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.pcr_grid_free(self.handle)
            self.handle = None


def _as_dev_scene(scene) -> DeviceScene:
    return scene if isinstance(scene, DeviceScene) else DeviceScene(scene)


# ---- stage 1 -----------------------------------------------------------------------------------
def build_grid(scene, params: VoxelParams | None = None) -> DeviceGrid:
    """pcray::build_grid (voxel_grid.hpp:99)."""
    ds = _as_dev_scene(scene)
    params = params or voxel_params()
    h = C.c_void_p()
    ds.ctx.check(lib().pcr_build_grid(ds.ctx.handle, ds.handle, C.byref(params), C.byref(h)))
    return DeviceGrid(h, ds.ctx)


def grid_part_build(scene: DeviceScene, shard: int, n_shards: int, params: VoxelParams | None = None) -> int:
    """Sharded build_grid: this shard's part on the scene's context; its size in bytes."""
    params = params or voxel_params()
    nb = C.c_uint64()
    scene.ctx.check(lib().pcr_grid_part_build(scene.ctx.handle, scene.handle, C.byref(params), shard, n_shards,
                                              C.byref(nb)))
    return int(nb.value)


def grid_part_copy(ctx: Context, dst_ptr: int) -> None:
    ctx.check(lib().pcr_grid_part_copy(ctx.handle, C.c_void_p(dst_ptr)))


def grid_assemble(ctx: Context, parts_ptr: int, offsets, sizes) -> DeviceGrid:
    """The grid from every shard's part (device bytes at parts_ptr + offsets[r], shard order)."""
    off = (C.c_uint64 * len(offsets))(*[int(x) for x in offsets])
    nb = (C.c_uint64 * len(sizes))(*[int(x) for x in sizes])
    h = C.c_void_p()
    ctx.check(lib().pcr_grid_assemble(ctx.handle, C.c_void_p(parts_ptr), off, nb, len(sizes), C.byref(h)))
    return DeviceGrid(h, ctx)


def compute_march_distances(grid: DeviceGrid) -> None:
    """pcray::compute_march_distances (voxel_grid.hpp:103), in place."""
    grid.ctx.check(lib().pcr_compute_march_distances(grid.ctx.handle, grid.handle))


# ---- stage 2 -----------------------------------------------------------------------------------
def transmission_phase(tx_index: int, grid: DeviceGrid, scene: DeviceScene, params: TraceParams | None = None):
    """pcray::transmission_phase (tracer.hpp:94-95) -> (los_paths, initial_hits)."""
    params = params or trace_params()
    los = C.POINTER(abi.Paths)()
    hits = C.POINTER(abi.InitialHits)()
    grid.ctx.check(lib().pcr_transmission_phase(grid.ctx.handle, grid.handle, scene.handle, tx_index,
                                                C.byref(params), C.byref(los), C.byref(hits)))
    try:
        return abi.paths_to_dict(los.contents), abi.hits_to_dict(hits.contents)
    finally:
        lib().pcr_free_paths(los)
        lib().pcr_free_initial_hits(hits)


def propagate(tx_index: int, hits: dict, grid: DeviceGrid, scene: DeviceScene, params: TraceParams | None = None):
    """pcray::propagate (tracer.hpp:122-124) -> candidates in (task, DFS) order after kappa."""
    params = params or trace_params()
    keep = abi.HitsKeepAlive(hits)
    out = C.POINTER(abi.Paths)()
    grid.ctx.check(lib().pcr_propagate(grid.ctx.handle, grid.handle, scene.handle, tx_index, C.byref(keep.hits),
                                       C.byref(params), C.byref(out)))
    try:
        return abi.paths_to_dict(out.contents)
    finally:
        lib().pcr_free_paths(out)


def last_trace_stats(ctx: Context | None = None) -> dict:
    """Work counters of the last propagate on ctx (cone traces = the reference's
    voxel_cone_trace / dfs_trace calls, visibility tests, cells and IEs walked)."""
    ctx = ctx or Context.default()
    a = (C.c_uint64 * 5)()
    ctx.check(lib().pcr_last_trace_stats(ctx.handle, a))
    return dict(zip(["cone_traces", "visibility_tests", "walk_cells", "walk_ies", "libm_unresolved"],
                    (int(x) for x in a)))


def make_ray(origin, direction, apex_angle, planes=(), origin_ie=abi.NO_IE, origin_label=0) -> abi.RayDesc:
    r = abi.RayDesc()
    r.origin[:] = [float(x) for x in origin]
    r.direction[:] = [float(x) for x in direction]
    r.apex_angle = float(apex_angle)
    r.n_planes = len(planes)
    for k, (p, n) in enumerate(planes):
        r.plane_point[k][:] = [float(x) for x in p]
        r.plane_normal[k][:] = [float(x) for x in n]
    r.origin_ie = origin_ie
    r.origin_label = origin_label
    return r


def voxel_cone_trace(rays, grid: DeviceGrid, scene: DeviceScene, want_debug: bool = False) -> dict:
    """pcray::voxel_cone_trace (tracer.hpp:118-120) over a batch of rays (CSR receptions)."""
    arr = (abi.RayDesc * max(1, len(rays)))(*rays)
    out = C.POINTER(abi.Receptions)()
    grid.ctx.check(lib().pcr_cone_trace_batch(grid.ctx.handle, grid.handle, scene.handle, arr, len(rays),
                                              int(want_debug), C.byref(out)))
    try:
        return abi.receptions_to_dict(out.contents)
    finally:
        lib().pcr_free_receptions(out)


def segment_visible(origin, target, target_ie, grid: DeviceGrid, scene: DeviceScene) -> np.ndarray:
    """pcray::segment_visible (tracer.hpp:88-89), batched."""
    o = np.ascontiguousarray(origin, dtype=np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(target, dtype=np.float64).reshape(-1, 3)
    ti = np.ascontiguousarray(np.broadcast_to(np.asarray(target_ie, dtype=np.uint32), (len(o),)))
    out = np.zeros(len(o), dtype=np.uint8)
    dp = C.POINTER(C.c_double)
    grid.ctx.check(lib().pcr_segment_visible_batch(grid.ctx.handle, grid.handle, scene.handle, o.ctypes.data_as(dp),
                                                   t.ctypes.data_as(dp), ti.ctypes.data_as(C.POINTER(C.c_uint32)),
                                                   len(o), out.ctypes.data_as(C.POINTER(C.c_uint8))))
    return out


# ---- stage 3 -----------------------------------------------------------------------------------
def refine_paths(candidates: dict, grid: DeviceGrid, scene: DeviceScene, params: RefineParams | None = None) -> dict:
    """pcray::refine_path (refine.hpp:77-78) for every candidate (LOS rows pass through)."""
    params = params or refine_params()
    keep = abi.PathsKeepAlive(candidates)
    out = C.POINTER(abi.Outcomes)()
    grid.ctx.check(lib().pcr_refine_batch(grid.ctx.handle, grid.handle, scene.handle, C.byref(keep.paths),
                                          C.byref(params), C.byref(out)))
    try:
        return abi.outcomes_to_dict(out.contents)
    finally:
        lib().pcr_free_outcomes(out)


# ---- pipeline ----------------------------------------------------------------------------------
def run_pipeline_on_scene(scene: Scene, config: RunConfig | None = None, ctx: Context | None = None) -> dict:
    """pcray::run_pipeline_on_scene (pipeline.hpp:61) -> RunSummary as a dict."""
    ctx = ctx or Context.default()
    config = config or default_run_config()
    keep = abi.SceneKeepAlive(scene)
    out = C.POINTER(abi.Summary)()
    ctx.check(lib().pcr_run_pipeline_on_scene(ctx.handle, C.byref(keep.desc), C.byref(config), C.byref(out)))
    try:
        return abi.summary_to_dict(out.contents)
    finally:
        lib().pcr_free_summary(out)


def run_pipeline_device(scene: DeviceScene, config: RunConfig | None = None) -> dict:
    """run_pipeline_on_scene over a scene already resident in HBM (pcr_run_pipeline_device)."""
    config = config or default_run_config()
    out = C.POINTER(abi.Summary)()
    scene.ctx.check(lib().pcr_run_pipeline_device(scene.ctx.handle, scene.handle, C.byref(config), C.byref(out)))
    try:
        return abi.summary_to_dict(out.contents)
    finally:
        lib().pcr_free_summary(out)


def load_point_cloud(path: str, rest: Scene | None = None, ctx: Context | None = None) -> DeviceScene:
    """pcray::load_point_cloud (io.hpp:15), device-resident result."""
    return DeviceScene.from_ply(path, rest, ctx)


def write_paths(path: str, paths: dict, config_hash: int, ctx: Context | None = None) -> None:
    """pcray::write_paths (io.hpp:33-34): the paths JSONL artifact."""
    ctx = ctx or Context.default()
    keep = abi.PathsKeepAlive(paths)
    ctx.check(lib().pcr_write_paths(ctx.handle, os.fsencode(path), C.byref(keep.paths), config_hash))


def load_edges(path: str, ctx: Context | None = None) -> dict:
    """pcray::load_edges (io.hpp:19-21) -> {start, end, normal_a, normal_b, label}."""
    ctx = ctx or Context.default()
    out = C.POINTER(abi.Edges)()
    ctx.check(lib().pcr_load_edges(ctx.handle, os.fsencode(path), C.byref(out)))
    try:
        return abi.edges_to_dict(out.contents)
    finally:
        lib().pcr_free_edges(out)


def run_pipeline(scene_path: str = "", edges_path: str = "", output_path: str = "", transmitters=(),
                 receivers=(), config: RunConfig | None = None, ctx: Context | None = None) -> dict:
    """pcray::run_pipeline (pipeline.hpp:63-64): files in, RunSummary (+ JSONL) out."""
    ctx = ctx or Context.default()
    config = config or default_run_config()
    keep = abi.RunFilesKeepAlive(scene_path, edges_path, output_path, transmitters, receivers)
    out = C.POINTER(abi.Summary)()
    ctx.check(lib().pcr_run_pipeline(ctx.handle, C.byref(keep.files), C.byref(config), C.byref(out)))
    try:
        return abi.summary_to_dict(out.contents)
    finally:
        lib().pcr_free_summary(out)


# ---- sharded pipeline (one process per GPU; orchestration in shard.py) ---------------------------
def shard_trace(scene: DeviceScene, config: RunConfig, shard: int, n_shards: int) -> tuple[int, int]:
    """pcr_shard_trace: validate, build_grid, transmission, this shard's propagate -> (rows, row bytes)."""
    n, b = C.c_uint64(), C.c_uint64()
    scene.ctx.check(lib().pcr_shard_trace(scene.ctx.handle, scene.handle, C.byref(config), shard, n_shards,
                                          C.byref(n), C.byref(b)))
    return n.value, b.value


def shard_rows(ctx: Context, dst_ptr: int) -> None:
    ctx.check(lib().pcr_shard_rows(ctx.handle, C.c_void_p(dst_ptr)))


def shard_refine(scene: DeviceScene, rows_ptr: int, n_rows: int) -> tuple[int, int]:
    """pcr_shard_refine: global kappa over every shard's rows, refine this shard's share -> (rows, bytes)."""
    n, b = C.c_uint64(), C.c_uint64()
    scene.ctx.check(lib().pcr_shard_refine(scene.ctx.handle, scene.handle, C.c_void_p(rows_ptr or None), n_rows,
                                           C.byref(n), C.byref(b)))
    return n.value, b.value


def shard_outcomes(ctx: Context, dst_ptr: int) -> None:
    ctx.check(lib().pcr_shard_outcomes(ctx.handle, C.c_void_p(dst_ptr)))


def shard_stats(ctx: Context) -> np.ndarray:
    st = abi.ShardStats()
    ctx.check(lib().pcr_shard_stats_get(ctx.handle, C.byref(st)))
    return np.array([getattr(st, f) for f in abi.SHARD_STATS_FIELDS], dtype=np.uint64)


def shard_finish(ctx: Context, rows_ptr: int, n_rows: int, totals) -> dict:
    """pcr_shard_finish: every shard's outcome rows + summed stats -> the RunSummary."""
    st = abi.ShardStats(*[int(x) for x in totals])
    out = C.POINTER(abi.Summary)()
    ctx.check(lib().pcr_shard_finish(ctx.handle, C.c_void_p(rows_ptr or None), n_rows, C.byref(st), C.byref(out)))
    try:
        return abi.summary_to_dict(out.contents)
    finally:
        lib().pcr_free_summary(out)


def stream_ptr(ctx: Context | None = None) -> int:
    """cudaStream_t the library launches on (for caller-side CUDA events)."""
    ctx = ctx or Context.default()
    return int(lib().pcr_stream(ctx.handle) or 0)


def set_profiling(on: bool, ctx: Context | None = None) -> None:
    ctx = ctx or Context.default()
    ctx.check(lib().pcr_set_profiling(ctx.handle, int(on)))


def kernel_times(reset: bool = True, ctx: Context | None = None) -> dict:
    """Per-kernel CUDA-event totals since the last reset: {name: (ms, launches)}."""
    ctx = ctx or Context.default()
    cap = 64
    names = (C.c_char * 32 * cap)()
    ms = (C.c_double * cap)()
    launches = (C.c_uint64 * cap)()
    n = lib().pcr_kernel_times(ctx.handle, names, ms, launches, cap, int(reset))
    if n < 0:
        ctx.check(-n)
    return {names[i].value.decode(): (float(ms[i]), int(launches[i])) for i in range(n)}


def transfer_bytes() -> tuple[int, int]:
    """(host->device, device->host) bytes the library copied so far in this process."""
    a, b = C.c_uint64(), C.c_uint64()
    lib().pcr_transfer_bytes(C.byref(a), C.byref(b))
    return int(a.value), int(b.value)


def fp64_probe(ctx: Context | None = None) -> float:
    """Measured non-FMA FP64 throughput of the device, TFLOP/s."""
    ctx = ctx or Context.default()
    v = C.c_double()
    ctx.check(lib().pcr_fp64_probe(ctx.handle, C.byref(v)))
    return float(v.value)


def config_hash(config: RunConfig) -> int:
    """pcray::config_hash (pipeline.hpp:39)."""
    return int(lib().pcr_config_hash(C.byref(config)))


def libm_exp(x, ctx: Context | None = None) -> np.ndarray:
    """The device exp() of the non-planar SDF (pcr_libm_exp_batch), elementwise."""
    ctx = ctx or Context.default()
    a = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    out = np.zeros_like(a)
    dp = C.POINTER(C.c_double)
    ctx.check(lib().pcr_libm_exp_batch(ctx.handle, a.ctypes.data_as(dp), out.ctypes.data_as(dp), len(a)))
    return out
