// device_state.cuh — owning device containers behind the C-ABI handles.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "geom.cuh"

namespace pcr {

// Device-resident scene (pcr_scene). Edges and radios are also kept on the host:
// they are tiny and the bounds / radio bookkeeping reads them there.
inline uint64_t next_scene_uid() {
  static std::atomic<uint64_t> n{0};
  return ++n;
}

struct SceneDev {
  const uint64_t uid = next_scene_uid();  // identity for caches keyed on the scene (GridDev payloads)
  uint64_t n_points = 0;
  DBuf<double> pos, nrm;  // n*3
  DBuf<uint32_t> label;
  uint32_t n_edges = 0;
  DBuf<double> edges;  // n_edges*12
  DBuf<uint32_t> edge_label;
  std::vector<double> h_edges;
  std::vector<uint32_t> h_edge_label;
  std::vector<double> h_tx, h_rx;  // n*3
  std::vector<uint32_t> h_tx_id, h_rx_id;
  DBuf<double> rx_pos;  // n_rx*3
  DBuf<uint32_t> rx_id;
  double carrier_frequency_hz = 60e9;

  SceneView view() const {
    SceneView v;
    v.pos = pos.get();
    v.nrm = nrm.get();
    v.label = label.get();
    v.n_points = n_points;
    v.edges = edges.get();
    v.edge_label = edge_label.get();
    v.n_edges = n_edges;
    return v;
  }
};

// Device-resident VoxelGrid (pcr_grid).
struct GridDev {
  V3 origin{0, 0, 0};
  int dims[3] = {0, 0, 0};
  double voxel_size = 0.5;
  int dv = 2;
  double sub_edge = 0, sub_radius = 0, voxel_radius = 0, hit_eps = 0;
  uint64_t n_cells = 0, n_ies = 0, n_pidx = 0;
  bool march_ok = false;  // cells[].z holds compute_march_distances' values (set by it)
  uint32_t part_voxel_lo = 0, part_voxel_hi = 0;  // a sharded build's part: its voxel range
  // staged non-planar payloads (GridView::pay_pos): built for the scene they came from
  mutable int has_nonplanar = -1;  // unknown until first asked
  mutable uint64_t pay_for = 0;  // SceneDev::uid the payloads were gathered from
  mutable DBuf<double> pay_pos, pay_nrm;
  GridView view_for(struct Ctx& ctx, const SceneDev& scene) const;
  DBuf<int4> cells;
  DBuf<uint32_t> meta, label, edge, rx, voxel, sub, pidx;
  DBuf<double4> sc, rp, pp, pn, seg_s, seg_e;
  DBuf<uint2> range;

  void set_geometry(const V3& o, const int d[3], double vs, int dvv) {
    origin = o;
    dims[0] = d[0];
    dims[1] = d[1];
    dims[2] = d[2];
    voxel_size = vs;
    dv = dvv;
    // voxel_grid.hpp:68-71
    sub_edge = voxel_size / dv;
    sub_radius = 0.5 * std::sqrt(3.0) * sub_edge;
    voxel_radius = 0.5 * std::sqrt(3.0) * voxel_size;
    hit_eps = 1e-4 * voxel_size;
  }

  GridView view() const {
    GridView v;
    v.origin = origin;
    v.dims[0] = dims[0];
    v.dims[1] = dims[1];
    v.dims[2] = dims[2];
    v.voxel_size = voxel_size;
    v.dv = dv;
    v.sub_edge = sub_edge;
    v.sub_radius = sub_radius;
    v.voxel_radius = voxel_radius;
    v.hit_eps = hit_eps;
    v.n_cells = static_cast<uint32_t>(n_cells);
    v.n_ies = static_cast<uint32_t>(n_ies);
    v.cells = cells.get();
    v.ie_meta = meta.get();
    v.ie_label = label.get();
    v.ie_sc = sc.get();
    v.ie_rp = rp.get();
    v.ie_pp = pp.get();
    v.ie_pn = pn.get();
    v.ie_range = range.get();
    v.ie_edge = edge.get();
    v.ie_rx = rx.get();
    v.point_indices = pidx.get();
    v.march_ok = march_ok ? 1 : 0;
    return v;
  }
  void alloc_ies(uint64_t n, cudaStream_t s) {
    n_ies = n;
    const size_t m = n ? n : 1;
    meta.alloc(m, s);
    label.alloc(m, s);
    edge.alloc(m, s);
    rx.alloc(m, s);
    voxel.alloc(m, s);
    sub.alloc(m, s);
    sc.alloc(m, s);
    rp.alloc(m, s);
    pp.alloc(m, s);
    pn.alloc(m, s);
    seg_s.alloc(m, s);
    seg_e.alloc(m, s);
    range.alloc(m, s);
  }
};

struct ShardState;  // pipeline.cu: state between the pcr_shard_* calls

struct Ctx {
  int device = 0;
  std::shared_ptr<ShardState> shard;
  cudaStream_t stream = nullptr;
  std::string last_error;
  std::mutex mu;
  // sin/cos table of the Keller fan azimuths, keyed by ray count (tracer.cpp:288-301)
  int fan_n = 0;
  DBuf<double> fan_table;  // n*6: cos phi, sin phi, sin(phi+dphi/2), cos(phi+dphi/2), sin(phi-dphi/2), cos(phi-dphi/2)
  int sm_count = 148;
  // pinned host scratch for the per-chunk counter round trips of the trace loop: a
  // device->host copy into pageable memory makes the driver wait for it inside
  // cudaMemcpyAsync (measured: 0.1-1.6 s of host gaps per C2 trace stage, varying run to
  // run); into pinned memory the copy is asynchronous and stream_wait spins on it
  uint64_t* pin = nullptr;  // kPinWords words, [0, 8) host->device, [8, 16) device->host
  static constexpr int kPinWords = 16;
  std::unique_ptr<GridDev> grid_part;  // the last pcr_grid_part_build's part
  std::shared_ptr<void> trace_ws;      // trace.cu's persistent node arena / candidate / task buffers
  // work counters of the last pcr_propagate call (cone traces, visibility tests, cells, IEs)
  uint64_t last_trace[5] = {0, 0, 0, 0, 0};
  // per-kernel CUDA-event timing (pcr_set_profiling); resolved lazily
  int profiling = 0;  // 0 off, 1 every kernel, 2 only the refine kernel (one launch per call)
  struct Pending {
    const char* name;
    cudaEvent_t a, b;
    double units;  // algorithmic work of the launch (bytes or flops, kernel-specific)
  };
  std::vector<Pending> pending;
  struct Total {
    double ms = 0, units = 0;
    uint64_t launches = 0;
  };
  std::vector<std::pair<std::string, Total>> totals;
  void resolve_timers();
};

// Scoped timer around one kernel launch on ctx.stream (no-op unless profiling).
struct KTimer {
  Ctx& c;
  const char* name;
  cudaEvent_t a = nullptr, b = nullptr;
  double units;
  KTimer(Ctx& ctx, const char* n, double u = 0) : c(ctx), name(n), units(u) {
    if (c.profiling == 2 && std::strcmp(n, "refine") != 0) c_skip = true;
    if (!c.profiling || c_skip) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, c.stream);
  }
  bool c_skip = false;
  ~KTimer() {
    if (!c.profiling || c_skip) return;
    cudaEventRecord(b, c.stream);
    c.pending.push_back({name, a, b, units});
  }
};

inline void Ctx::resolve_timers() {
  if (pending.empty()) return;
  cudaStreamSynchronize(stream);
  for (auto& p : pending) {
    float ms = 0;
    cudaEventElapsedTime(&ms, p.a, p.b);
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
    Total* t = nullptr;
    for (auto& kv : totals)
      if (kv.first == p.name) t = &kv.second;
    if (!t) {
      totals.emplace_back(p.name, Total{});
      t = &totals.back().second;
    }
    t->ms += ms;
    t->units += p.units;
    t->launches += 1;
  }
  pending.clear();
}

// stage 1 (voxelize.cu)
// one shard of a sharded build_grid: the shard's voxel range, its points'
// surface IEs and its edge pieces / receivers; the part has no cells (assembled grid)
struct VoxelShard {
  uint32_t index, n_shards;
};
void build_grid_device(Ctx& ctx, const SceneDev& scene, double voxel_size, int division_factor,
                       uint64_t max_cells, GridDev& out, const VoxelShard* shard = nullptr);
void compute_march_distances_device(Ctx& ctx, GridDev& grid);
// grid parts (one per shard, in shard order) as bytes -> the whole grid
uint64_t grid_part_bytes(const GridDev& part);
void grid_part_serialize(Ctx& ctx, const GridDev& part, void* dst_device);
void grid_assemble(Ctx& ctx, const uint8_t* parts_device, const uint64_t* offset, const uint64_t* bytes,
                   uint32_t n_parts, GridDev& out);

}  // namespace pcr
