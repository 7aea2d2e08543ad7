// capi.cu — the extern "C" boundary (include/pcray_b200.h). Every entry point
// catches C++/CUDA errors and reports them through pcr_last_error(ctx).
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "device_state.cuh"
#include "handles.cuh"
#include "host_alloc.hpp"
#include "pipeline.hpp"

namespace {

template <typename F>
int guarded(pcr_ctx* ctx, F&& f) {
  if (!ctx) return PCR_ERR_INVALID;
  std::lock_guard<std::mutex> lock(ctx->c.mu);
  try {
    PCR_CUDA(cudaSetDevice(ctx->c.device));
    f();
    ctx->c.last_error.clear();
    return PCR_OK;
  } catch (const pcr::Error& e) {
    ctx->c.last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    ctx->c.last_error = "host allocation failed";
    return PCR_ERR_NOMEM;
  } catch (const std::exception& e) {
    ctx->c.last_error = e.what();
    return PCR_ERR_RUNTIME;
  }
}

double4 pack4(const double* p, double w = 0.0) { return make_double4(p[0], p[1], p[2], w); }
void unpack4(double* d, const double4& v) {
  d[0] = v.x;
  d[1] = v.y;
  d[2] = v.z;
}

}  // namespace

extern "C" {

int pcr_abi_version(void) { return PCR_ABI_VERSION; }

int pcr_create(int device, pcr_ctx** out) {
  if (!out) return PCR_ERR_INVALID;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return PCR_ERR_CUDA;
  if (device < 0 || device >= n) return PCR_ERR_INVALID;
  auto* ctx = new pcr_ctx();
  ctx->c.device = device;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return PCR_ERR_CUDA;
  }
  cudaDeviceGetAttribute(&ctx->c.sm_count, cudaDevAttrMultiProcessorCount, device);
  if (cudaHostAlloc(reinterpret_cast<void**>(&ctx->c.pin), pcr::Ctx::kPinWords * sizeof(uint64_t), cudaHostAllocDefault) !=
      cudaSuccess) {
    cudaStreamDestroy(ctx->c.stream);
    delete ctx;
    return PCR_ERR_CUDA;
  }
  // keep freed pool memory cached across calls (stream-ordered allocator)
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = ctx;
  return PCR_OK;
}

void pcr_destroy(pcr_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->c.device);
  ctx->c.fan_table.release();
  ctx->c.shard.reset();      // its buffers are freed on the context's stream
  ctx->c.grid_part.reset();  // likewise the last sharded-voxelization part
  ctx->c.trace_ws.reset();   // and the trace workspace
  cudaStreamSynchronize(ctx->c.stream);
  cudaStreamDestroy(ctx->c.stream);
  if (ctx->c.pin) cudaFreeHost(ctx->c.pin);
  delete ctx;
}

const char* pcr_last_error(const pcr_ctx* ctx) { return ctx ? ctx->c.last_error.c_str() : "null context"; }

uint64_t pcr_kernel_launches(void) { return pcr::g_launch_count; }

void pcr_transfer_bytes(uint64_t* h2d, uint64_t* d2h) {
  if (h2d) *h2d = pcr::g_h2d_bytes;
  if (d2h) *d2h = pcr::g_d2h_bytes;
}

int pcr_scene_upload(pcr_ctx* ctx, const pcr_scene_desc* d, pcr_scene** out) {
  return guarded(ctx, [&] {
    if (!d || !out) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    auto* sc = new pcr_scene();
    try {
      pcr::upload_scene(ctx->c, *d, sc->s);
    } catch (...) {
      delete sc;
      throw;
    }
    *out = sc;
  });
}

void pcr_scene_free(pcr_scene* scene) { delete scene; }

int pcr_build_grid(pcr_ctx* ctx, const pcr_scene* scene, const pcr_voxel_params* p, pcr_grid** out) {
  return guarded(ctx, [&] {
    if (!scene || !p || !out) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    auto* g = new pcr_grid();
    try {
      pcr::build_grid_device(ctx->c, scene->s, p->voxel_size, p->division_factor, p->max_cells, g->g);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int pcr_compute_march_distances(pcr_ctx* ctx, pcr_grid* grid) {
  return guarded(ctx, [&] {
    if (!grid) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    pcr::compute_march_distances_device(ctx->c, grid->g);
    PCR_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

int pcr_grid_upload(pcr_ctx* ctx, const pcr_grid_host* h, pcr_grid** out) {
  return guarded(ctx, [&] {
    if (!h || !out) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    cudaStream_t s = ctx->c.stream;
    auto* gg = new pcr_grid();
    try {
      pcr::GridDev& G = gg->g;
      G.set_geometry(pcr::V3{h->origin[0], h->origin[1], h->origin[2]}, h->dims, h->voxel_size,
                     h->division_factor);
      G.n_cells = h->n_cells;
      std::vector<int4> cells(h->n_cells ? h->n_cells : 1);
      for (size_t i = 0; i < h->n_cells; ++i)
        cells[i] = make_int4(static_cast<int>(h->cell_ie_begin[i]), static_cast<int>(h->cell_ie_end[i]),
                             h->cell_march[i], 0);
      G.cells.alloc(cells.size(), s);
      pcr::h2d(G.cells.get(), cells.data(), cells.size(), s);
      const size_t ni = h->n_ies;
      G.alloc_ies(ni, s);
      std::vector<uint32_t> meta(ni), rx(ni), edge(ni), label(ni), vox(ni), sub(ni);
      std::vector<double4> sc(ni), rp(ni), pp(ni), pn(ni), ss(ni), se(ni);
      std::vector<uint2> range(ni);
      for (size_t i = 0; i < ni; ++i) {
        meta[i] = h->ie_kind[i] | (h->ie_planar[i] ? 4u : 0u);
        rx[i] = h->ie_rx_id[i];
        edge[i] = h->ie_edge_index[i];
        label[i] = h->ie_label[i];
        vox[i] = h->ie_voxel[i];
        sub[i] = h->ie_subvoxel[i];
        sc[i] = pack4(h->ie_sphere_center + 3 * i, h->ie_sphere_radius[i]);
        rp[i] = pack4(h->ie_reception_point + 3 * i);
        pp[i] = pack4(h->ie_plane_point + 3 * i);
        pn[i] = pack4(h->ie_plane_normal + 3 * i);
        ss[i] = pack4(h->ie_seg_start + 3 * i);
        se[i] = pack4(h->ie_seg_end + 3 * i);
        range[i] = make_uint2(h->ie_point_begin[i], h->ie_point_end[i]);
      }
      pcr::h2d(G.meta.get(), meta.data(), ni, s);
      pcr::h2d(G.rx.get(), rx.data(), ni, s);
      pcr::h2d(G.edge.get(), edge.data(), ni, s);
      pcr::h2d(G.label.get(), label.data(), ni, s);
      pcr::h2d(G.voxel.get(), vox.data(), ni, s);
      pcr::h2d(G.sub.get(), sub.data(), ni, s);
      pcr::h2d(G.sc.get(), sc.data(), ni, s);
      pcr::h2d(G.rp.get(), rp.data(), ni, s);
      pcr::h2d(G.pp.get(), pp.data(), ni, s);
      pcr::h2d(G.pn.get(), pn.data(), ni, s);
      pcr::h2d(G.seg_s.get(), ss.data(), ni, s);
      pcr::h2d(G.seg_e.get(), se.data(), ni, s);
      pcr::h2d(G.range.get(), range.data(), ni, s);
      G.n_pidx = h->n_point_indices;
      G.pidx.alloc(G.n_pidx ? G.n_pidx : 1, s);
      pcr::h2d(G.pidx.get(), h->point_indices, G.n_pidx, s);
      pcr::stream_wait(s);
    } catch (...) {
      delete gg;
      throw;
    }
    *out = gg;
  });
}

int pcr_grid_download(pcr_ctx* ctx, const pcr_grid* grid, pcr_grid_host** out) {
  return guarded(ctx, [&] {
    if (!grid || !out) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    cudaStream_t s = ctx->c.stream;
    const pcr::GridDev& G = grid->g;
    pcr_grid_host* h = pcr::alloc_grid_host(G.n_cells, G.n_ies, G.n_pidx);
    try {
      h->origin[0] = G.origin.x;
      h->origin[1] = G.origin.y;
      h->origin[2] = G.origin.z;
      for (int a = 0; a < 3; ++a) h->dims[a] = G.dims[a];
      h->voxel_size = G.voxel_size;
      h->division_factor = G.dv;
      const size_t nc = G.n_cells, ni = G.n_ies;
      std::vector<int4> cells(nc);
      pcr::d2h(cells.data(), G.cells.get(), nc, s);
      std::vector<uint32_t> meta(ni);
      std::vector<double4> sc(ni), rp(ni), pp(ni), pn(ni), ss(ni), se(ni);
      std::vector<uint2> range(ni);
      pcr::d2h(meta.data(), G.meta.get(), ni, s);
      pcr::d2h(sc.data(), G.sc.get(), ni, s);
      pcr::d2h(rp.data(), G.rp.get(), ni, s);
      pcr::d2h(pp.data(), G.pp.get(), ni, s);
      pcr::d2h(pn.data(), G.pn.get(), ni, s);
      pcr::d2h(ss.data(), G.seg_s.get(), ni, s);
      pcr::d2h(se.data(), G.seg_e.get(), ni, s);
      pcr::d2h(range.data(), G.range.get(), ni, s);
      pcr::d2h(h->ie_label, G.label.get(), ni, s);
      pcr::d2h(h->ie_edge_index, G.edge.get(), ni, s);
      pcr::d2h(h->ie_rx_id, G.rx.get(), ni, s);
      pcr::d2h(h->ie_voxel, G.voxel.get(), ni, s);
      pcr::d2h(h->ie_subvoxel, G.sub.get(), ni, s);
      pcr::d2h(h->point_indices, G.pidx.get(), G.n_pidx, s);
      pcr::stream_wait(s);
      for (size_t i = 0; i < nc; ++i) {
        h->cell_ie_begin[i] = static_cast<uint32_t>(cells[i].x);
        h->cell_ie_end[i] = static_cast<uint32_t>(cells[i].y);
        h->cell_march[i] = cells[i].z;
      }
      for (size_t i = 0; i < ni; ++i) {
        h->ie_kind[i] = static_cast<uint8_t>(meta[i] & 3u);
        h->ie_planar[i] = static_cast<uint8_t>((meta[i] >> 2) & 1u);
        unpack4(h->ie_sphere_center + 3 * i, sc[i]);
        h->ie_sphere_radius[i] = sc[i].w;
        unpack4(h->ie_reception_point + 3 * i, rp[i]);
        unpack4(h->ie_plane_point + 3 * i, pp[i]);
        unpack4(h->ie_plane_normal + 3 * i, pn[i]);
        unpack4(h->ie_seg_start + 3 * i, ss[i]);
        unpack4(h->ie_seg_end + 3 * i, se[i]);
        h->ie_point_begin[i] = range[i].x;
        h->ie_point_end[i] = range[i].y;
      }
    } catch (...) {
      pcr::free_grid_host(h);
      throw;
    }
    *out = h;
  });
}

void pcr_grid_free(pcr_grid* grid) { delete grid; }
void pcr_free_grid_host(pcr_grid_host* h) { pcr::free_grid_host(h); }

void pcr_free_paths(pcr_paths* p) {
  if (!p) return;
  pcr::free_paths_arrays(p);
  std::free(p);
}

void pcr_free_initial_hits(pcr_initial_hits* h) {
  if (!h) return;
  std::free(h->ie_index);
  std::free(h->kind);
  std::free(h->position);
  std::free(h->normal);
  std::free(h->incoming);
  std::free(h);
}

void pcr_free_outcomes(pcr_outcomes* o) {
  if (!o) return;
  pcr::free_paths_arrays(&o->paths);
  std::free(o->has_path);
  std::free(o->reason);
  std::free(o);
}

void pcr_free_summary(pcr_summary* s) {
  if (!s) return;
  pcr::free_paths_arrays(&s->paths);
  std::free(s);
}

void pcr_free_receptions(pcr_receptions* r) {
  if (!r) return;
  void* a[] = {r->ray_offset, r->ie_index,   r->reception_point,  r->hit_valid, r->hit_position,
               r->hit_normal, r->hit_label,  r->hit_distance,     r->evaluated_offset, r->evaluated,
               r->visited_offset, r->visited};
  for (void* x : a) std::free(x);
  std::free(r);
}

// ---- stage 2 / stage 3 / pipeline entry points (trace.cu, refine.cu, pipeline.cu)
int pcr_transmission_phase(pcr_ctx* ctx, const pcr_grid* grid, const pcr_scene* scene, uint32_t tx_index,
                           const pcr_trace_params* params, pcr_paths** los_out, pcr_initial_hits** hits_out) {
  return guarded(ctx, [&] {
    if (!grid || !scene || !params || !los_out || !hits_out) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    pcr::api_transmission(ctx->c, grid->g, scene->s, tx_index, *params, los_out, hits_out);
  });
}

int pcr_propagate(pcr_ctx* ctx, const pcr_grid* grid, const pcr_scene* scene, uint32_t tx_index,
                  const pcr_initial_hits* hits, const pcr_trace_params* params, pcr_paths** out) {
  return guarded(ctx, [&] {
    if (!grid || !scene || !hits || !params || !out) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    pcr::api_propagate(ctx->c, grid->g, scene->s, tx_index, *hits, *params, out);
  });
}

// ---- sharded voxelization (gridparts.cu) -----------------------------------
int pcr_grid_part_build(pcr_ctx* ctx, const pcr_scene* scene, const pcr_voxel_params* p, uint32_t shard,
                        uint32_t n_shards, uint64_t* part_bytes) {
  return guarded(ctx, [&] {
    if (!scene || !p || !part_bytes) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    auto part = std::make_unique<pcr::GridDev>();
    const pcr::VoxelShard vs{shard, n_shards};
    try {
      pcr::build_grid_device(ctx->c, scene->s, p->voxel_size, p->division_factor, p->max_cells, *part, &vs);
    } catch (const pcr::Error& e) {
      throw pcr::Error(e.code, std::string(e.what()));
    }
    *part_bytes = pcr::grid_part_bytes(*part);
    ctx->c.grid_part = std::move(part);
  });
}

int pcr_grid_part_copy(pcr_ctx* ctx, void* dst_device) {
  return guarded(ctx, [&] {
    if (!ctx->c.grid_part) throw pcr::Error(PCR_ERR_INVALID, "voxelize: no grid part built on this context");
    if (!dst_device) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    pcr::grid_part_serialize(ctx->c, *ctx->c.grid_part, dst_device);
  });
}

int pcr_grid_assemble(pcr_ctx* ctx, const void* parts_device, const uint64_t* part_offset, const uint64_t* part_bytes,
                      uint32_t n_parts, pcr_grid** out) {
  return guarded(ctx, [&] {
    if (!parts_device || !part_offset || !part_bytes || !out) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    auto g = std::make_unique<pcr_grid>();
    pcr::grid_assemble(ctx->c, static_cast<const uint8_t*>(parts_device), part_offset, part_bytes, n_parts, g->g);
    *out = g.release();
  });
}

int pcr_last_trace_stats(pcr_ctx* ctx, uint64_t* out5) {
  return guarded(ctx, [&] {
    uint64_t* out4 = out5;
    if (!out4) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    for (int i = 0; i < 5; ++i) out4[i] = ctx->c.last_trace[i];
  });
}

int pcr_cone_trace_batch(pcr_ctx* ctx, const pcr_grid* grid, const pcr_scene* scene, const pcr_ray_desc* rays,
                         uint64_t n_rays, int want_debug, pcr_receptions** out) {
  return guarded(ctx, [&] {
    if (!grid || !scene || (!rays && n_rays) || !out) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    pcr::api_cone_trace_batch(ctx->c, grid->g, scene->s, rays, n_rays, want_debug != 0, out);
  });
}

int pcr_segment_visible_batch(pcr_ctx* ctx, const pcr_grid* grid, const pcr_scene* scene, const double* origin,
                              const double* target, const uint32_t* target_ie, uint64_t n, uint8_t* visible_out) {
  return guarded(ctx, [&] {
    if (!grid || !scene || (n && (!origin || !target || !target_ie || !visible_out)))
      throw pcr::Error(PCR_ERR_INVALID, "null argument");
    pcr::api_segment_visible_batch(ctx->c, grid->g, scene->s, origin, target, target_ie, n, visible_out);
  });
}

int pcr_refine_batch(pcr_ctx* ctx, const pcr_grid* grid, const pcr_scene* scene, const pcr_paths* candidates,
                     const pcr_refine_params* params, pcr_outcomes** out) {
  return guarded(ctx, [&] {
    if (!grid || !scene || !candidates || !params || !out) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    pcr::api_refine_batch(ctx->c, grid->g, scene->s, *candidates, *params, out);
  });
}

int pcr_run_pipeline_on_scene(pcr_ctx* ctx, const pcr_scene_desc* scene, const pcr_run_config* config,
                              pcr_summary** out) {
  return guarded(ctx, [&] {
    if (!scene || !config || !out) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    pcr::api_run_pipeline_on_scene(ctx->c, *scene, *config, out);
  });
}

int pcr_run_pipeline_device(pcr_ctx* ctx, const pcr_scene* scene, const pcr_run_config* config,
                            pcr_summary** out) {
  return guarded(ctx, [&] {
    if (!scene || !config || !out) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    pcr::api_run_pipeline_device(ctx->c, scene->s, *config, out);
  });
}

int pcr_scene_load_ply(pcr_ctx* ctx, const char* path, const pcr_scene_desc* rest, pcr_scene** out) {
  return guarded(ctx, [&] {
    if (!path || !rest || !out) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    auto* sc = new pcr_scene();
    try {
      pcr::api_scene_load_ply(ctx->c, path, *rest, sc->s);
    } catch (...) {
      delete sc;
      throw;
    }
    *out = sc;
  });
}

int pcr_scene_points(pcr_ctx* ctx, const pcr_scene* scene, double* position, double* normal, uint32_t* label,
                     uint64_t* n) {
  return guarded(ctx, [&] {
    if (!scene) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    if (n) *n = scene->s.n_points;
    pcr::api_scene_points(ctx->c, scene->s, position, normal, label);
  });
}

int pcr_write_paths(pcr_ctx* ctx, const char* path, const pcr_paths* paths, uint64_t config_hash) {
  return guarded(ctx, [&] {
    if (!path || !paths) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    pcr::api_write_paths(path, *paths, config_hash);
  });
}

int pcr_load_edges(pcr_ctx* ctx, const char* path, pcr_edges** out) {
  return guarded(ctx, [&] {
    if (!path || !out) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    std::vector<double> g;
    std::vector<uint32_t> l;
    pcr::api_load_edges(path, g, l);
    pcr_edges* e = pcr::halloc<pcr_edges>(1);
    e->n = static_cast<uint32_t>(l.size());
    e->geometry = pcr::halloc<double>(g.size() + 1);
    e->label = pcr::halloc<uint32_t>(l.size() + 1);
    if (!g.empty()) std::memcpy(e->geometry, g.data(), g.size() * sizeof(double));
    if (!l.empty()) std::memcpy(e->label, l.data(), l.size() * sizeof(uint32_t));
    *out = e;
  });
}

void pcr_free_edges(pcr_edges* e) {
  if (!e) return;
  std::free(e->geometry);
  std::free(e->label);
  std::free(e);
}

int pcr_run_pipeline(pcr_ctx* ctx, const pcr_run_files* files, const pcr_run_config* config, pcr_summary** out) {
  return guarded(ctx, [&] {
    if (!files || !config || !out) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    if ((files->n_tx && !files->tx_position) || (files->n_rx && !files->rx_position))
      throw pcr::Error(PCR_ERR_INVALID, "null argument");
    pcr::api_run_pipeline(ctx->c, *files, *config, out);
  });
}

int pcr_shard_trace(pcr_ctx* ctx, const pcr_scene* scene, const pcr_run_config* config, uint32_t shard,
                    uint32_t n_shards, uint64_t* n_rows, uint64_t* row_bytes) {
  return guarded(ctx, [&] {
    if (!scene || !config || !n_rows || !row_bytes) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    pcr::api_shard_trace(ctx->c, scene->s, *config, shard, n_shards, n_rows, row_bytes);
  });
}

int pcr_shard_trace_grid(pcr_ctx* ctx, const pcr_scene* scene, const pcr_grid* grid, const pcr_run_config* config,
                         uint32_t shard, uint32_t n_shards, uint64_t* n_rows, uint64_t* row_bytes) {
  return guarded(ctx, [&] {
    if (!scene || !grid || !config || !n_rows || !row_bytes) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    pcr::api_shard_trace(ctx->c, scene->s, *config, shard, n_shards, n_rows, row_bytes, &grid->g);
  });
}

int pcr_shard_rows(pcr_ctx* ctx, void* dst_device) {
  return guarded(ctx, [&] { pcr::api_shard_rows(ctx->c, dst_device); });
}

int pcr_shard_refine(pcr_ctx* ctx, const pcr_scene* scene, const void* rows_device, uint64_t n_rows,
                     uint64_t* n_out, uint64_t* out_row_bytes) {
  return guarded(ctx, [&] {
    if (!scene || !n_out || !out_row_bytes || (n_rows && !rows_device))
      throw pcr::Error(PCR_ERR_INVALID, "null argument");
    pcr::api_shard_refine(ctx->c, scene->s, rows_device, n_rows, n_out, out_row_bytes);
  });
}

int pcr_shard_outcomes(pcr_ctx* ctx, void* dst_device) {
  return guarded(ctx, [&] { pcr::api_shard_outcomes(ctx->c, dst_device); });
}

int pcr_shard_stats_get(pcr_ctx* ctx, pcr_shard_stats* out) {
  return guarded(ctx, [&] {
    if (!out) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    pcr::api_shard_stats(ctx->c, out);
  });
}

int pcr_shard_finish(pcr_ctx* ctx, const void* outcome_rows_device, uint64_t n_rows, const pcr_shard_stats* totals,
                     pcr_summary** out) {
  return guarded(ctx, [&] {
    if (!totals || !out || (n_rows && !outcome_rows_device)) throw pcr::Error(PCR_ERR_INVALID, "null argument");
    pcr::api_shard_finish(ctx->c, outcome_rows_device, n_rows, *totals, out);
  });
}

void* pcr_stream(pcr_ctx* ctx) { return ctx ? static_cast<void*>(ctx->c.stream) : nullptr; }

int pcr_set_profiling(pcr_ctx* ctx, int on) {
  return guarded(ctx, [&] {
    ctx->c.resolve_timers();
    ctx->c.profiling = on == 2 ? 2 : on != 0 ? 1 : 0;
  });
}

int pcr_kernel_times(pcr_ctx* ctx, char (*names)[32], double* ms, uint64_t* launches, int cap, int reset) {
  int n = 0;
  const int rc = guarded(ctx, [&] {
    ctx->c.resolve_timers();
    for (const auto& kv : ctx->c.totals) {
      if (n >= cap) break;
      std::snprintf(names[n], 32, "%s", kv.first.c_str());
      ms[n] = kv.second.ms;
      launches[n] = kv.second.launches;
      ++n;
    }
    if (reset) ctx->c.totals.clear();
  });
  return rc == PCR_OK ? n : -rc;
}

uint64_t pcr_config_hash(const pcr_run_config* c) { return pcr::config_hash(*c); }

void pcr_run_config_defaults(pcr_run_config* c) { pcr::run_config_defaults(c); }

}  // extern "C"
