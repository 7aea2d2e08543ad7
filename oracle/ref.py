"""Python handle on the ORACLE — TEST INFRASTRUCTURE ONLY.

Loads oracle/_ref/libpcray_ref.so: the unmodified reference library
(/root/reference/proj/src/*.cpp) built by oracle/Makefile against the Eigen
subset shim, wrapped by oracle/ref_capi.cpp. Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline leg may import this module; the product package
never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2402_13747_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libpcray_ref.so")
REFERENCE_SRC = "/root/reference/proj"

COUNT_LIB_PATH = os.path.join(HERE, "_ref", "libpcray_ref_count.so")

_lib = None          # the library the module functions currently use
_libs = {}           # path -> loaded CDLL


def build(force: bool = False) -> None:
    """Compile the oracle (needs /root/reference; the GPU box uses the prebuilt .so)."""
    if os.path.isdir(REFERENCE_SRC):
        subprocess.check_call(["make", "-s", "-j8", "all"] + (["-B"] if force else []), cwd=HERE)


def available() -> bool:
    return os.path.exists(LIB_PATH)


class counting:
    """Context manager: route calls to the counting build (voxel_cone_trace /
    segment_visible entry counters; slower, never timed). Objects created inside
    must be used and freed inside."""

    def __enter__(self):
        global _lib
        self.prev = lib()
        _lib = _load(COUNT_LIB_PATH)
        _lib.pcrref_counters.argtypes = [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_int]
        return self

    def read(self, reset=True):
        a, b = C.c_uint64(), C.c_uint64()
        _lib.pcrref_counters(C.byref(a), C.byref(b), int(reset))
        return int(a.value), int(b.value)

    def __exit__(self, *exc):
        global _lib
        import gc

        gc.collect()
        _lib = self.prev
        return False


def lib():
    global _lib
    if _lib is None:
        _lib = _load(LIB_PATH)
    return _lib


def _load(path):
    if path not in _libs:
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        vp = C.c_void_p
        pp = C.POINTER
        L.pcrref_last_error.restype = C.c_char_p
        L.pcrref_scene_create.restype = vp
        L.pcrref_scene_create.argtypes = [pp(abi.SceneDesc)]
        L.pcrref_scene_free.argtypes = [vp]
        L.pcrref_validate_scene.argtypes = [vp, C.c_char_p, C.c_size_t]
        L.pcrref_build_grid.argtypes = [vp, pp(abi.VoxelParams), pp(vp)]
        L.pcrref_grid_free.argtypes = [vp]
        L.pcrref_compute_march_distances.argtypes = [vp]
        L.pcrref_grid_download.argtypes = [vp, pp(pp(abi.GridHost))]
        L.pcrref_grid_from_host.argtypes = [pp(abi.GridHost), pp(vp)]
        L.pcrref_free_grid_host.argtypes = [pp(abi.GridHost)]
        L.pcrref_transmission_phase.argtypes = [vp, vp, C.c_uint32, pp(abi.TraceParams),
                                                pp(pp(abi.Paths)), pp(pp(abi.InitialHits))]
        L.pcrref_propagate.argtypes = [vp, vp, C.c_uint32, pp(abi.InitialHits), pp(abi.TraceParams),
                                       C.c_int, pp(pp(abi.Paths))]
        L.pcrref_cone_trace_batch.argtypes = [vp, vp, pp(abi.RayDesc), C.c_uint64, C.c_int,
                                              pp(pp(abi.Receptions))]
        L.pcrref_free_receptions.argtypes = [pp(abi.Receptions)]
        L.pcrref_segment_visible_batch.argtypes = [vp, vp, pp(C.c_double), pp(C.c_double),
                                                   pp(C.c_uint32), C.c_uint64, pp(C.c_uint8)]
        L.pcrref_march_segment_batch.argtypes = [vp, vp, pp(C.c_double), pp(C.c_double), pp(C.c_uint32),
                                                 pp(C.c_double), C.c_uint64, pp(C.c_uint8), pp(C.c_double),
                                                 pp(C.c_double), pp(C.c_double)]
        L.pcrref_refine_batch.argtypes = [vp, vp, pp(abi.Paths), pp(abi.RefineParams), C.c_int,
                                          pp(pp(abi.Outcomes))]
        L.pcrref_free_outcomes.argtypes = [pp(abi.Outcomes)]
        L.pcrref_refine_dedup_batch.argtypes = [vp, vp, pp(abi.Paths), pp(abi.RefineParams), C.c_int, C.c_double,
                                                pp(C.c_uint64), pp(pp(abi.Outcomes))]
        L.pcrref_run_pipeline_on_scene.argtypes = [vp, pp(abi.RunConfig), pp(pp(abi.Summary))]
        L.pcrref_free_summary.argtypes = [pp(abi.Summary)]
        L.pcrref_free_paths.argtypes = [pp(abi.Paths)]
        L.pcrref_free_initial_hits.argtypes = [pp(abi.InitialHits)]
        L.pcrref_config_hash.restype = C.c_uint64
        L.pcrref_config_hash.argtypes = [pp(abi.RunConfig)]
        L.pcrref_run_config_defaults.argtypes = [pp(abi.RunConfig)]
        L.pcrref_sample_planar_scene.restype = C.c_uint64
        L.pcrref_sample_planar_scene.argtypes = [pp(C.c_double), C.c_uint32, C.c_double, C.c_uint32,
                                                 pp(C.c_double), pp(C.c_double), pp(C.c_uint32)]
        L.pcrref_image_method_paths.argtypes = [pp(C.c_double), C.c_uint32, pp(C.c_double), pp(C.c_double),
                                                C.c_int, pp(pp(abi.Paths))]
        L.pcrref_save_point_cloud.argtypes = [C.c_char_p, vp, C.c_int]
        L.pcrref_load_point_cloud.argtypes = [C.c_char_p, pp(pp(C.c_double)), pp(pp(C.c_double)),
                                              pp(pp(C.c_uint32)), pp(C.c_uint64)]
        L.pcrref_free.argtypes = [vp]
        L.pcrref_write_paths.argtypes = [C.c_char_p, pp(abi.Paths), C.c_uint64]
        L.pcrref_load_edges.argtypes = [C.c_char_p, pp(pp(abi.Edges))]
        L.pcrref_run_pipeline.argtypes = [pp(abi.RunFiles), pp(abi.RunConfig), pp(pp(abi.Summary))]
        _libs[path] = L
    return _libs[path]


class RefError(RuntimeError):
    pass


def _check(rc: int):
    if rc != 0:
        raise RefError(lib().pcrref_last_error().decode())


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class RefScene:
    def __init__(self, scene: abi.Scene):
        self.keep = abi.SceneKeepAlive(scene)
        self.scene = self.keep.scene
        self.L = lib()
        self.handle = self.L.pcrref_scene_create(C.byref(self.keep.desc))

    def __del__(self):
        if getattr(self, "handle", None):
            self.L.pcrref_scene_free(self.handle)
            self.handle = None

    def validate(self):
        buf = C.create_string_buffer(512)
        n = lib().pcrref_validate_scene(self.handle, buf, 512)
        return n, buf.value.decode()


class RefGrid:
    def __init__(self, handle):
        self.handle = handle
        self.L = lib()

    @classmethod
    def build(cls, scene: RefScene, params: abi.VoxelParams | None = None) -> "RefGrid":
        params = params or abi.voxel_params()
        h = C.c_void_p()
        _check(lib().pcrref_build_grid(scene.handle, C.byref(params), C.byref(h)))
        return cls(h)

    @classmethod
    def from_dict(cls, g: dict) -> "RefGrid":
        keep = abi.GridKeepAlive(g)
        h = C.c_void_p()
        _check(lib().pcrref_grid_from_host(C.byref(keep.host), C.byref(h)))
        return cls(h)

    def compute_march_distances(self):
        _check(lib().pcrref_compute_march_distances(self.handle))

    def to_dict(self) -> dict:
        out = C.POINTER(abi.GridHost)()
        _check(lib().pcrref_grid_download(self.handle, C.byref(out)))
        try:
            return abi.grid_to_dict(out.contents)
        finally:
            lib().pcrref_free_grid_host(out)

    def __del__(self):
        if getattr(self, "handle", None):
            self.L.pcrref_grid_free(self.handle)
            self.handle = None


def build_grid(scene: RefScene, params=None) -> RefGrid:
    return RefGrid.build(scene, params)


def transmission_phase(grid: RefGrid, scene: RefScene, tx_index: int, params=None):
    params = params or abi.trace_params()
    los = C.POINTER(abi.Paths)()
    hits = C.POINTER(abi.InitialHits)()
    _check(lib().pcrref_transmission_phase(grid.handle, scene.handle, tx_index, C.byref(params),
                                           C.byref(los), C.byref(hits)))
    try:
        return abi.paths_to_dict(los.contents), abi.hits_to_dict(hits.contents)
    finally:
        lib().pcrref_free_paths(los)
        lib().pcrref_free_initial_hits(hits)


def propagate(grid: RefGrid, scene: RefScene, tx_index: int, hits: dict, params=None, thread_count=0):
    params = params or abi.trace_params()
    keep = abi.HitsKeepAlive(hits)
    out = C.POINTER(abi.Paths)()
    _check(lib().pcrref_propagate(grid.handle, scene.handle, tx_index, C.byref(keep.hits), C.byref(params),
                                  thread_count, C.byref(out)))
    try:
        return abi.paths_to_dict(out.contents)
    finally:
        lib().pcrref_free_paths(out)


def cone_trace_batch(grid: RefGrid, scene: RefScene, rays, want_debug=False):
    arr = (abi.RayDesc * max(1, len(rays)))(*rays)
    out = C.POINTER(abi.Receptions)()
    _check(lib().pcrref_cone_trace_batch(grid.handle, scene.handle, arr, len(rays), int(want_debug),
                                         C.byref(out)))
    try:
        return abi.receptions_to_dict(out.contents)
    finally:
        lib().pcrref_free_receptions(out)


def segment_visible_batch(grid: RefGrid, scene: RefScene, origin, target, target_ie):
    o = np.ascontiguousarray(origin, dtype=np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(target, dtype=np.float64).reshape(-1, 3)
    ti = np.ascontiguousarray(target_ie, dtype=np.uint32).reshape(-1)
    out = np.zeros(len(ti), dtype=np.uint8)
    _check(lib().pcrref_segment_visible_batch(grid.handle, scene.handle, _dp(o), _dp(t),
                                              ti.ctypes.data_as(C.POINTER(C.c_uint32)), len(ti),
                                              out.ctypes.data_as(C.POINTER(C.c_uint8))))
    return out


def march_segment_batch(grid: RefGrid, scene: RefScene, origin, direction, ie, t_max=None):
    o = np.ascontiguousarray(origin, dtype=np.float64).reshape(-1, 3)
    d = np.ascontiguousarray(direction, dtype=np.float64).reshape(-1, 3)
    ie = np.ascontiguousarray(ie, dtype=np.uint32).reshape(-1)
    n = len(ie)
    tm = np.full(n, np.inf) if t_max is None else np.ascontiguousarray(t_max, dtype=np.float64)
    hit = np.zeros(n, np.uint8)
    pos = np.zeros((n, 3))
    nrm = np.zeros((n, 3))
    dist = np.zeros(n)
    _check(lib().pcrref_march_segment_batch(grid.handle, scene.handle, _dp(o), _dp(d),
                                            ie.ctypes.data_as(C.POINTER(C.c_uint32)), _dp(tm), n,
                                            hit.ctypes.data_as(C.POINTER(C.c_uint8)), _dp(pos), _dp(nrm),
                                            _dp(dist)))
    return hit, pos, nrm, dist


def refine_batch(grid: RefGrid, scene: RefScene, candidates: dict, params=None, thread_count=0):
    params = params or abi.refine_params()
    keep = abi.PathsKeepAlive(candidates)
    out = C.POINTER(abi.Outcomes)()
    _check(lib().pcrref_refine_batch(grid.handle, scene.handle, C.byref(keep.paths), C.byref(params),
                                     thread_count, C.byref(out)))
    try:
        return abi.outcomes_to_dict(out.contents)
    finally:
        lib().pcrref_free_outcomes(out)


def refine_dedup_count(grid: RefGrid, scene: RefScene, candidates: dict, params=None, thread_count=0,
                       carrier_frequency_hz=60e9) -> int:
    """refine_path on every candidate, then the pipeline's dedup_by_label ->
    dedup_by_fresnel (pipeline.cpp:181-208): the number RunSummary::exact_paths counts."""
    params = params or abi.refine_params()
    keep = abi.PathsKeepAlive(candidates)
    n = C.c_uint64()
    _check(lib().pcrref_refine_dedup_batch(grid.handle, scene.handle, C.byref(keep.paths), C.byref(params),
                                           thread_count, carrier_frequency_hz, C.byref(n), None))
    return int(n.value)


def run_pipeline_on_scene(scene: RefScene, config: abi.RunConfig | None = None):
    config = config or default_run_config()
    out = C.POINTER(abi.Summary)()
    _check(lib().pcrref_run_pipeline_on_scene(scene.handle, C.byref(config), C.byref(out)))
    try:
        return abi.summary_to_dict(out.contents)
    finally:
        lib().pcrref_free_summary(out)


def default_run_config(**overrides) -> abi.RunConfig:
    c = abi.RunConfig()
    lib().pcrref_run_config_defaults(C.byref(c))
    for k, v in overrides.items():
        setattr(c, k, int(v) if isinstance(v, bool) else v)
    return c


def config_hash(config: abi.RunConfig) -> int:
    return int(lib().pcrref_config_hash(C.byref(config)))


def sample_planar_scene(rect_array: np.ndarray, density: float, seed: int):
    r = np.ascontiguousarray(rect_array, dtype=np.float64)
    n = int(lib().pcrref_sample_planar_scene(_dp(r), r.shape[0], density, seed, None, None, None))
    pos = np.zeros((n, 3))
    nrm = np.zeros((n, 3))
    lab = np.zeros(n, np.uint32)
    lib().pcrref_sample_planar_scene(_dp(r), r.shape[0], density, seed, _dp(pos), _dp(nrm),
                                     lab.ctypes.data_as(C.POINTER(C.c_uint32)))
    return pos, nrm, lab


def image_method_paths(rect_array, tx, rx, max_order):
    r = np.ascontiguousarray(rect_array, dtype=np.float64)
    t = np.ascontiguousarray(tx, dtype=np.float64)
    x = np.ascontiguousarray(rx, dtype=np.float64)
    out = C.POINTER(abi.Paths)()
    _check(lib().pcrref_image_method_paths(_dp(r), r.shape[0], _dp(t), _dp(x), max_order, C.byref(out)))
    try:
        return abi.paths_to_dict(out.contents)
    finally:
        lib().pcrref_free_paths(out)


# ---- io.hpp (point clouds, paths artifact) ----------------------------------------------------
def save_point_cloud(path: str, scene: RefScene, binary: bool = True) -> None:
    """pcray::save_point_cloud (io.hpp:16-17)."""
    _check(lib().pcrref_save_point_cloud(path.encode(), scene.handle, int(binary)))


def load_point_cloud(path: str) -> dict:
    """pcray::load_point_cloud (io.hpp:15) -> {position, normal, label}."""
    pos, nrm, lab, n = C.POINTER(C.c_double)(), C.POINTER(C.c_double)(), C.POINTER(C.c_uint32)(), C.c_uint64()
    _check(lib().pcrref_load_point_cloud(path.encode(), C.byref(pos), C.byref(nrm), C.byref(lab), C.byref(n)))
    try:
        k = n.value
        return {"position": np.ctypeslib.as_array(pos, (max(k, 1) * 3,))[: 3 * k].reshape(-1, 3).copy(),
                "normal": np.ctypeslib.as_array(nrm, (max(k, 1) * 3,))[: 3 * k].reshape(-1, 3).copy(),
                "label": np.ctypeslib.as_array(lab, (max(k, 1),))[:k].copy()}
    finally:
        for p in (pos, nrm, lab):
            lib().pcrref_free(C.cast(p, C.c_void_p))


def write_paths(path: str, paths: dict, config_hash: int) -> None:
    """pcray::write_paths (io.hpp:33-34)."""
    keep = abi.PathsKeepAlive(paths)
    _check(lib().pcrref_write_paths(path.encode(), C.byref(keep.paths), config_hash))


def load_edges(path: str) -> dict:
    """pcray::load_edges (io.hpp:19-21) -> {start, end, normal_a, normal_b, label}."""
    out = C.POINTER(abi.Edges)()
    _check(lib().pcrref_load_edges(path.encode(), C.byref(out)))
    try:
        return abi.edges_to_dict(out.contents)
    finally:
        e = out.contents
        lib().pcrref_free(C.cast(e.geometry, C.c_void_p))
        lib().pcrref_free(C.cast(e.label, C.c_void_p))
        lib().pcrref_free(C.cast(out, C.c_void_p))


def run_pipeline(scene_path: str = "", edges_path: str = "", output_path: str = "", transmitters=(),
                 receivers=(), config: abi.RunConfig | None = None) -> dict:
    """pcray::run_pipeline (pipeline.hpp:63-64): files in, RunSummary (+ JSONL) out."""
    config = config or default_run_config()
    keep = abi.RunFilesKeepAlive(scene_path, edges_path, output_path, transmitters, receivers)
    out = C.POINTER(abi.Summary)()
    _check(lib().pcrref_run_pipeline(C.byref(keep.files), C.byref(config), C.byref(out)))
    try:
        return abi.summary_to_dict(out.contents)
    finally:
        lib().pcrref_free_summary(out)
