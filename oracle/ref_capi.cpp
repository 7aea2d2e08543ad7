// ref_capi.cpp — TEST INFRASTRUCTURE ONLY: C-ABI wrapper around the UNMODIFIED
// reference library (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile
// against oracle/shim). It fills the same result structs as the product library
// (include/pcray_b200.h) so parity tests compare them field by field, and it is
// the CPU baseline arm of bench.py (cpu_baseline.kind = "reference").
//
// Nothing in the product (paper_2402_13747_b200/) links, loads or calls this.
// Every function forwards to the reference entry point cited beside it.

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <map>
#include <string>
#include <vector>

#include "pcray/io.hpp"
#include "pcray/oracle.hpp"
#include "pcray/parallel.hpp"
#include "pcray/pipeline.hpp"
#include "pcray/refine.hpp"
#include "pcray/surface.hpp"
#include "pcray/tracer.hpp"
#include "pcray/voxel_grid.hpp"
#include "pcray_b200.h"

using namespace pcray;

namespace {

thread_local std::string g_err;

template <typename T>
T* alloc(std::size_t n) {
  return static_cast<T*>(std::calloc(n ? n : 1, sizeof(T)));
}

void put3(double* dst, const Vec3& v) {
  dst[0] = v.x();
  dst[1] = v.y();
  dst[2] = v.z();
}
Vec3 get3(const double* s) { return Vec3(s[0], s[1], s[2]); }

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return PCR_OK;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PCR_ERR_RUNTIME;
  } catch (...) {
    g_err = "unknown error";
    return PCR_ERR_RUNTIME;
  }
}

Scene scene_from_desc(const pcr_scene_desc* d) {
  Scene s;
  s.points.resize(d->n_points);
  for (std::uint64_t i = 0; i < d->n_points; ++i) {
    s.points[i].position = get3(d->point_position + 3 * i);
    s.points[i].normal = get3(d->point_normal + 3 * i);
    s.points[i].label = d->point_label[i];
  }
  s.edges.resize(d->n_edges);
  for (std::uint32_t e = 0; e < d->n_edges; ++e) {
    const double* g = d->edge_geometry + 12 * e;
    s.edges[e] = DiffractionEdge{get3(g), get3(g + 3), get3(g + 6), get3(g + 9), d->edge_label[e]};
  }
  for (std::uint32_t i = 0; i < d->n_tx; ++i)
    s.transmitters.push_back(Radio{RadioKind::Tx, get3(d->tx_position + 3 * i), d->tx_id[i]});
  for (std::uint32_t i = 0; i < d->n_rx; ++i)
    s.receivers.push_back(Radio{RadioKind::Rx, get3(d->rx_position + 3 * i), d->rx_id[i]});
  s.carrier_frequency_hz = d->carrier_frequency_hz;
  return s;
}

TraceParams trace_params(const pcr_trace_params* p) {
  TraceParams t;
  t.max_interactions = p->max_interactions;
  t.kappa = p->kappa;
  t.cone_apex_angle = p->cone_apex_angle;
  t.diffraction_ray_count = p->diffraction_ray_count;
  t.max_diffractions = p->max_diffractions;
  return t;
}

RunConfig run_config(const pcr_run_config* c) {
  RunConfig r;
  r.carrier_frequency_hz = c->carrier_frequency_hz;
  r.voxel_size_m = c->voxel_size_m;
  r.division_factor = c->division_factor;
  r.kappa = c->kappa;
  r.max_interactions = c->max_interactions;
  r.max_diffractions = c->max_diffractions;
  r.cone_apex_angle_deg = c->cone_apex_angle_deg;
  r.diffraction_ray_count = c->diffraction_ray_count;
  r.delta = c->delta;
  r.rho = c->rho;
  r.step_size = c->step_size;
  r.seed = c->seed;
  r.thread_count = c->thread_count;
  r.fresnel_enabled = c->fresnel_enabled != 0;
  return r;
}

pcr_paths* alloc_paths(std::uint64_t n, std::uint32_t stride) {
  pcr_paths* p = alloc<pcr_paths>(1);
  p->n = n;
  p->stride = stride;
  p->tx_id = alloc<std::uint32_t>(n);
  p->rx_id = alloc<std::uint32_t>(n);
  p->tx_position = alloc<double>(3 * n);
  p->rx_position = alloc<double>(3 * n);
  p->length = alloc<double>(n);
  p->delay = alloc<double>(n);
  p->converged = alloc<std::uint8_t>(n);
  p->gradient_norm = alloc<double>(n);
  p->n_inter = alloc<std::uint32_t>(n);
  const std::size_t m = static_cast<std::size_t>(n) * stride;
  p->kind = alloc<std::uint8_t>(m);
  p->position = alloc<double>(3 * m);
  p->label = alloc<std::uint32_t>(m);
  p->normal = alloc<double>(3 * m);
  p->ie_index = alloc<std::uint32_t>(m);
  p->edge_index = alloc<std::uint32_t>(m);
  return p;
}

void free_paths_arrays(pcr_paths* p) {
  std::free(p->tx_id);
  std::free(p->rx_id);
  std::free(p->tx_position);
  std::free(p->rx_position);
  std::free(p->length);
  std::free(p->delay);
  std::free(p->converged);
  std::free(p->gradient_norm);
  std::free(p->n_inter);
  std::free(p->kind);
  std::free(p->position);
  std::free(p->label);
  std::free(p->normal);
  std::free(p->ie_index);
  std::free(p->edge_index);
}

void put_interactions(pcr_paths* p, std::size_t row, const std::vector<Interaction>& its) {
  p->n_inter[row] = static_cast<std::uint32_t>(its.size());
  for (std::size_t k = 0; k < its.size(); ++k) {
    const std::size_t j = row * p->stride + k;
    p->kind[j] = static_cast<std::uint8_t>(its[k].kind);
    put3(p->position + 3 * j, its[k].position);
    p->label[j] = its[k].label;
    put3(p->normal + 3 * j, its[k].normal);
    p->ie_index[j] = its[k].ie_index;
    p->edge_index[j] = its[k].edge_index;
  }
}

std::uint32_t max_inter(const std::vector<PathCandidate>& v) {
  std::size_t m = 1;
  for (const auto& c : v) m = std::max(m, c.interactions.size());
  return static_cast<std::uint32_t>(m);
}

pcr_paths* paths_from_candidates(const std::vector<PathCandidate>& v) {
  pcr_paths* p = alloc_paths(v.size(), max_inter(v));
  for (std::size_t i = 0; i < v.size(); ++i) {
    p->tx_id[i] = v[i].tx_id;
    p->rx_id[i] = v[i].rx_id;
    put3(p->tx_position + 3 * i, v[i].tx_position);
    put3(p->rx_position + 3 * i, v[i].rx_position);
    p->length[i] = v[i].coarse_length;
    put_interactions(p, i, v[i].interactions);
  }
  return p;
}

void put_exact(pcr_paths* p, std::size_t i, const ExactPath& e) {
  p->tx_id[i] = e.tx_id;
  p->rx_id[i] = e.rx_id;
  put3(p->tx_position + 3 * i, e.tx_position);
  put3(p->rx_position + 3 * i, e.rx_position);
  p->length[i] = e.total_length;
  p->delay[i] = e.delay;
  p->converged[i] = e.converged ? 1 : 0;
  p->gradient_norm[i] = e.gradient_norm;
  put_interactions(p, i, e.interactions);
}

std::vector<PathCandidate> candidates_from_paths(const pcr_paths* p) {
  std::vector<PathCandidate> out(p->n);
  for (std::uint64_t i = 0; i < p->n; ++i) {
    PathCandidate& c = out[i];
    c.tx_id = p->tx_id[i];
    c.rx_id = p->rx_id[i];
    c.tx_position = get3(p->tx_position + 3 * i);
    c.rx_position = get3(p->rx_position + 3 * i);
    c.coarse_length = p->length[i];
    for (std::uint32_t k = 0; k < p->n_inter[i]; ++k) {
      const std::size_t j = i * p->stride + k;
      Interaction it;
      it.kind = static_cast<InteractionKind>(p->kind[j]);
      it.position = get3(p->position + 3 * j);
      it.label = p->label[j];
      it.normal = get3(p->normal + 3 * j);
      it.ie_index = p->ie_index[j];
      it.edge_index = p->edge_index[j];
      c.interactions.push_back(it);
    }
  }
  return out;
}

}  // namespace

extern "C" {

const char* pcrref_last_error(void) { return g_err.c_str(); }

// ---- scene -------------------------------------------------------------------
void* pcrref_scene_create(const pcr_scene_desc* desc) { return new Scene(scene_from_desc(desc)); }
void pcrref_scene_free(void* s) { delete static_cast<Scene*>(s); }

// validate_scene (scene.cpp:31-91): returns the violation count, first rule in buf.
int pcrref_validate_scene(const void* scene, char* first_rule, size_t cap) {
  const auto v = validate_scene(*static_cast<const Scene*>(scene));
  if (!v.empty() && first_rule && cap) {
    std::snprintf(first_rule, cap, "%s", (v.front().rule + " (" + v.front().detail + ")").c_str());
  }
  return static_cast<int>(v.size());
}

// ---- stage 1 -------------------------------------------------------------------
// build_grid (voxel_grid.cpp:82-227)
int pcrref_build_grid(const void* scene, const pcr_voxel_params* vp, void** out) {
  return guarded([&] {
    VoxelizationParams p;
    p.voxel_size = vp->voxel_size;
    p.division_factor = vp->division_factor;
    p.max_cells = vp->max_cells;
    *out = new VoxelGrid(build_grid(*static_cast<const Scene*>(scene), p));
  });
}

void pcrref_grid_free(void* g) { delete static_cast<VoxelGrid*>(g); }

// compute_march_distances (voxel_grid.cpp:229-268)
int pcrref_compute_march_distances(void* g) {
  return guarded([&] { compute_march_distances(*static_cast<VoxelGrid*>(g)); });
}

int pcrref_grid_download(const void* gp, pcr_grid_host** out) {
  return guarded([&] {
    const VoxelGrid& g = *static_cast<const VoxelGrid*>(gp);
    pcr_grid_host* h = alloc<pcr_grid_host>(1);
    put3(h->origin, g.origin);
    for (int a = 0; a < 3; ++a) h->dims[a] = g.dims[a];
    h->voxel_size = g.voxel_size;
    h->division_factor = g.division_factor;
    const std::size_t nc = g.cells.size(), ni = g.ies.size(), np = g.point_indices.size();
    h->n_cells = nc;
    h->n_ies = ni;
    h->n_point_indices = np;
    h->cell_ie_begin = alloc<std::uint32_t>(nc);
    h->cell_ie_end = alloc<std::uint32_t>(nc);
    h->cell_march = alloc<std::int32_t>(nc);
    for (std::size_t i = 0; i < nc; ++i) {
      h->cell_ie_begin[i] = g.cells[i].ie_begin;
      h->cell_ie_end[i] = g.cells[i].ie_end;
      h->cell_march[i] = g.cells[i].march;
    }
    h->ie_kind = alloc<std::uint8_t>(ni);
    h->ie_label = alloc<std::uint32_t>(ni);
    h->ie_reception_point = alloc<double>(3 * ni);
    h->ie_sphere_center = alloc<double>(3 * ni);
    h->ie_sphere_radius = alloc<double>(ni);
    h->ie_point_begin = alloc<std::uint32_t>(ni);
    h->ie_point_end = alloc<std::uint32_t>(ni);
    h->ie_seg_start = alloc<double>(3 * ni);
    h->ie_seg_end = alloc<double>(3 * ni);
    h->ie_edge_index = alloc<std::uint32_t>(ni);
    h->ie_rx_id = alloc<std::uint32_t>(ni);
    h->ie_planar = alloc<std::uint8_t>(ni);
    h->ie_plane_point = alloc<double>(3 * ni);
    h->ie_plane_normal = alloc<double>(3 * ni);
    h->ie_voxel = alloc<std::uint32_t>(ni);
    h->ie_subvoxel = alloc<std::uint32_t>(ni);
    for (std::size_t i = 0; i < ni; ++i) {
      const IntersectableEntity& e = g.ies[i];
      h->ie_kind[i] = static_cast<std::uint8_t>(e.kind);
      h->ie_label[i] = e.label;
      put3(h->ie_reception_point + 3 * i, e.reception_point);
      put3(h->ie_sphere_center + 3 * i, e.sphere_center);
      h->ie_sphere_radius[i] = e.sphere_radius;
      h->ie_point_begin[i] = e.point_begin;
      h->ie_point_end[i] = e.point_end;
      put3(h->ie_seg_start + 3 * i, e.seg_start);
      put3(h->ie_seg_end + 3 * i, e.seg_end);
      h->ie_edge_index[i] = e.edge_index;
      h->ie_rx_id[i] = e.rx_id;
      h->ie_planar[i] = e.planar ? 1 : 0;
      put3(h->ie_plane_point + 3 * i, e.plane_point);
      put3(h->ie_plane_normal + 3 * i, e.plane_normal);
      h->ie_voxel[i] = e.voxel;
      h->ie_subvoxel[i] = e.subvoxel;
    }
    h->point_indices = alloc<std::uint32_t>(np);
    if (np) std::memcpy(h->point_indices, g.point_indices.data(), np * sizeof(std::uint32_t));
    *out = h;
  });
}

int pcrref_grid_from_host(const pcr_grid_host* h, void** out) {
  return guarded([&] {
    auto* g = new VoxelGrid();
    g->origin = get3(h->origin);
    g->dims = Eigen::Vector3i(h->dims[0], h->dims[1], h->dims[2]);
    g->voxel_size = h->voxel_size;
    g->division_factor = h->division_factor;
    g->cells.resize(h->n_cells);
    for (std::size_t i = 0; i < h->n_cells; ++i)
      g->cells[i] = VoxelCell{h->cell_ie_begin[i], h->cell_ie_end[i], h->cell_march[i]};
    g->ies.resize(h->n_ies);
    for (std::size_t i = 0; i < h->n_ies; ++i) {
      IntersectableEntity& e = g->ies[i];
      e.kind = static_cast<IeKind>(h->ie_kind[i]);
      e.label = h->ie_label[i];
      e.reception_point = get3(h->ie_reception_point + 3 * i);
      e.sphere_center = get3(h->ie_sphere_center + 3 * i);
      e.sphere_radius = h->ie_sphere_radius[i];
      e.point_begin = h->ie_point_begin[i];
      e.point_end = h->ie_point_end[i];
      e.seg_start = get3(h->ie_seg_start + 3 * i);
      e.seg_end = get3(h->ie_seg_end + 3 * i);
      e.edge_index = h->ie_edge_index[i];
      e.rx_id = h->ie_rx_id[i];
      e.planar = h->ie_planar[i] != 0;
      e.plane_point = get3(h->ie_plane_point + 3 * i);
      e.plane_normal = get3(h->ie_plane_normal + 3 * i);
      e.voxel = h->ie_voxel[i];
      e.subvoxel = h->ie_subvoxel[i];
    }
    g->point_indices.assign(h->point_indices, h->point_indices + h->n_point_indices);
    *out = g;
  });
}

void pcrref_free_grid_host(pcr_grid_host* h) {
  if (!h) return;
  void* arrays[] = {h->cell_ie_begin,   h->cell_ie_end,        h->cell_march,     h->ie_kind,
                    h->ie_label,        h->ie_reception_point, h->ie_sphere_center, h->ie_sphere_radius,
                    h->ie_point_begin,  h->ie_point_end,       h->ie_seg_start,   h->ie_seg_end,
                    h->ie_edge_index,   h->ie_rx_id,           h->ie_planar,      h->ie_plane_point,
                    h->ie_plane_normal, h->ie_voxel,           h->ie_subvoxel,    h->point_indices};
  for (void* a : arrays) std::free(a);
  std::free(h);
}

// ---- stage 2 -------------------------------------------------------------------
// transmission_phase (tracer.cpp:207-255)
int pcrref_transmission_phase(const void* grid, const void* scene, uint32_t tx_index,
                              const pcr_trace_params* tp, pcr_paths** los_out,
                              pcr_initial_hits** hits_out) {
  return guarded([&] {
    const Scene& s = *static_cast<const Scene*>(scene);
    const TransmissionResult tr = transmission_phase(
        s.transmitters.at(tx_index), *static_cast<const VoxelGrid*>(grid), s, trace_params(tp));
    *los_out = paths_from_candidates(tr.los_paths);
    pcr_initial_hits* h = alloc<pcr_initial_hits>(1);
    const std::size_t n = tr.initial_hits.size();
    h->n = n;
    h->ie_index = alloc<std::uint32_t>(n);
    h->kind = alloc<std::uint8_t>(n);
    h->position = alloc<double>(3 * n);
    h->normal = alloc<double>(3 * n);
    h->incoming = alloc<double>(3 * n);
    for (std::size_t i = 0; i < n; ++i) {
      const InitialHit& ih = tr.initial_hits[i];
      h->ie_index[i] = ih.ie_index;
      h->kind[i] = static_cast<std::uint8_t>(ih.kind);
      put3(h->position + 3 * i, ih.position);
      put3(h->normal + 3 * i, ih.normal);
      put3(h->incoming + 3 * i, ih.incoming);
    }
    *hits_out = h;
  });
}

// propagate (tracer.cpp:476-533)
int pcrref_propagate(const void* grid, const void* scene, uint32_t tx_index,
                     const pcr_initial_hits* hits, const pcr_trace_params* tp, int thread_count,
                     pcr_paths** out) {
  return guarded([&] {
    const Scene& s = *static_cast<const Scene*>(scene);
    std::vector<InitialHit> ih(hits->n);
    for (std::size_t i = 0; i < hits->n; ++i) {
      ih[i].ie_index = hits->ie_index[i];
      ih[i].kind = static_cast<IeKind>(hits->kind[i]);
      ih[i].position = get3(hits->position + 3 * i);
      ih[i].normal = get3(hits->normal + 3 * i);
      ih[i].incoming = get3(hits->incoming + 3 * i);
    }
    const auto cands = propagate(s.transmitters.at(tx_index), ih,
                                 *static_cast<const VoxelGrid*>(grid), s, trace_params(tp),
                                 thread_count);
    *out = paths_from_candidates(cands);
  });
}

static ConicalRay ray_from_desc(const pcr_ray_desc& d) {
  ConicalRay r;
  r.origin = get3(d.origin);
  r.direction = get3(d.direction);
  r.apex_angle = d.apex_angle;
  for (int k = 0; k < d.n_planes; ++k)
    r.separation_planes.push_back(SeparationPlane{get3(d.plane_point[k]), get3(d.plane_normal[k])});
  if (d.origin_ie != PCR_NO_IE) {
    Interaction it;
    it.ie_index = d.origin_ie;
    it.label = d.origin_label;
    r.provenance.push_back(it);
  }
  return r;
}

// voxel_cone_trace (tracer.cpp:313-403), one call per ray, TraceDebug optional
int pcrref_cone_trace_batch(const void* grid, const void* scene, const pcr_ray_desc* rays,
                            uint64_t n_rays, int want_debug, pcr_receptions** out) {
  return guarded([&] {
    const VoxelGrid& g = *static_cast<const VoxelGrid*>(grid);
    const Scene& s = *static_cast<const Scene*>(scene);
    std::vector<std::vector<Reception>> recs(n_rays);
    std::vector<TraceDebug> dbg(n_rays);
    parallel_for(n_rays, 0, [&](std::size_t i) {
      recs[i] = voxel_cone_trace(ray_from_desc(rays[i]), g, s, TraceParams{},
                                 want_debug ? &dbg[i] : nullptr);
    });
    std::size_t total = 0, total_ev = 0, total_vi = 0;
    for (std::size_t i = 0; i < n_rays; ++i) {
      total += recs[i].size();
      total_ev += dbg[i].evaluated.size();
      total_vi += dbg[i].visited.size();
    }
    pcr_receptions* r = alloc<pcr_receptions>(1);
    r->n_rays = n_rays;
    r->n = total;
    r->ray_offset = alloc<std::uint64_t>(n_rays + 1);
    r->ie_index = alloc<std::uint32_t>(total);
    r->reception_point = alloc<double>(3 * total);
    r->hit_valid = alloc<std::uint8_t>(total);
    r->hit_position = alloc<double>(3 * total);
    r->hit_normal = alloc<double>(3 * total);
    r->hit_label = alloc<std::uint32_t>(total);
    r->hit_distance = alloc<double>(total);
    r->evaluated_offset = alloc<std::uint64_t>(n_rays + 1);
    r->evaluated = alloc<std::uint32_t>(total_ev);
    r->visited_offset = alloc<std::uint64_t>(n_rays + 1);
    r->visited = alloc<std::uint32_t>(total_vi);
    std::size_t k = 0, ke = 0, kv = 0;
    for (std::size_t i = 0; i < n_rays; ++i) {
      r->ray_offset[i] = k;
      r->evaluated_offset[i] = ke;
      r->visited_offset[i] = kv;
      for (std::uint32_t c : dbg[i].visited) r->visited[kv++] = c;
      for (const Reception& rc : recs[i]) {
        r->ie_index[k] = rc.ie_index;
        put3(r->reception_point + 3 * k, rc.reception_point);
        r->hit_valid[k] = rc.hit_valid ? 1 : 0;
        put3(r->hit_position + 3 * k, rc.surface_hit.position);
        put3(r->hit_normal + 3 * k, rc.surface_hit.normal);
        r->hit_label[k] = rc.surface_hit.label;
        r->hit_distance[k] = rc.surface_hit.distance_along_ray;
        ++k;
      }
      for (std::uint32_t c : dbg[i].evaluated) r->evaluated[ke++] = c;
    }
    r->ray_offset[n_rays] = k;
    r->evaluated_offset[n_rays] = ke;
    r->visited_offset[n_rays] = kv;
    *out = r;
  });
}

void pcrref_free_receptions(pcr_receptions* r) {
  if (!r) return;
  void* arrays[] = {r->ray_offset, r->ie_index,   r->reception_point, r->hit_valid,
                    r->hit_position, r->hit_normal, r->hit_label,     r->hit_distance,
                    r->evaluated_offset, r->evaluated, r->visited_offset, r->visited};
  for (void* a : arrays) std::free(a);
  std::free(r);
}

// segment_visible (tracer.cpp:138-205)
int pcrref_segment_visible_batch(const void* grid, const void* scene, const double* origin,
                                 const double* target, const uint32_t* target_ie, uint64_t n,
                                 uint8_t* visible_out) {
  return guarded([&] {
    const VoxelGrid& g = *static_cast<const VoxelGrid*>(grid);
    const Scene& s = *static_cast<const Scene*>(scene);
    parallel_for(n, 0, [&](std::size_t i) {
      visible_out[i] =
          segment_visible(get3(origin + 3 * i), get3(target + 3 * i), target_ie[i], g, s) ? 1 : 0;
    });
  });
}

// march_segment (surface.cpp:64-134) per (origin, direction, ie, t_max)
int pcrref_march_segment_batch(const void* grid, const void* scene, const double* origin,
                               const double* direction, const uint32_t* ie, const double* t_max,
                               uint64_t n, uint8_t* hit, double* position, double* normal,
                               double* distance) {
  return guarded([&] {
    const VoxelGrid& g = *static_cast<const VoxelGrid*>(grid);
    const Scene& s = *static_cast<const Scene*>(scene);
    for (std::size_t i = 0; i < n; ++i) {
      const auto h = march_segment(get3(origin + 3 * i), get3(direction + 3 * i), g.ies.at(ie[i]),
                                   g, s, t_max[i]);
      hit[i] = h ? 1 : 0;
      if (h) {
        put3(position + 3 * i, h->position);
        put3(normal + 3 * i, h->normal);
        distance[i] = h->distance_along_ray;
      }
    }
  });
}

// ---- stage 3 -------------------------------------------------------------------
// refine_path (refine.cpp:189-286) per candidate; LOS rows pass through as in
// run_pipeline_on_scene (pipeline.cpp:160-170).
static int refine_batch_impl(const void* grid, const void* scene, const pcr_paths* cands,
                             const pcr_refine_params* rp, int thread_count, pcr_outcomes** out,
                             double carrier_frequency_hz, uint64_t* n_dedup) {
  return guarded([&] {
    const VoxelGrid& g = *static_cast<const VoxelGrid*>(grid);
    const Scene& s = *static_cast<const Scene*>(scene);
    const auto cv = candidates_from_paths(cands);
    RefineParams p;
    p.delta = rp->delta;
    p.rho = rp->rho;
    p.step_size = rp->step_size;
    p.fresnel_enabled = rp->fresnel_enabled != 0;
    std::vector<RefineOutcome> oc(cv.size());
    parallel_for(cv.size(), thread_count, [&](std::size_t i) {
      if (cv[i].interactions.empty()) {
        ExactPath los;
        los.tx_id = cv[i].tx_id;
        los.rx_id = cv[i].rx_id;
        los.tx_position = cv[i].tx_position;
        los.rx_position = cv[i].rx_position;
        los.total_length = cv[i].coarse_length;
        los.delay = los.total_length / kSpeedOfLight;
        los.converged = true;
        oc[i] = {los, RejectReason::not_converged};
      } else {
        oc[i] = refine_path(cv[i], g, s, p);
      }
    });
    if (n_dedup) {
      // the pipeline's post-refine step (pipeline.cpp:181-208): exact paths, then
      // dedup_by_label -> dedup_by_fresnel (refine.cpp:324-372) -> final sort
      std::vector<ExactPath> exact;
      for (const RefineOutcome& r : oc)
        if (r.path) exact.push_back(*r.path);
      exact = dedup_by_label(std::move(exact));
      if (p.fresnel_enabled) exact = dedup_by_fresnel(std::move(exact), carrier_frequency_hz);
      std::sort(exact.begin(), exact.end(), [](const ExactPath& a, const ExactPath& b) {
        if (a.tx_id != b.tx_id) return a.tx_id < b.tx_id;
        if (a.rx_id != b.rx_id) return a.rx_id < b.rx_id;
        return a.delay < b.delay;
      });
      *n_dedup = exact.size();
    }
    if (!out) return;
    pcr_outcomes* o = alloc<pcr_outcomes>(1);
    pcr_paths* pp = alloc_paths(cv.size(), std::max<std::uint32_t>(1, cands->stride));
    o->paths = *pp;
    std::free(pp);
    o->has_path = alloc<std::uint8_t>(cv.size());
    o->reason = alloc<std::int32_t>(cv.size());
    for (std::size_t i = 0; i < cv.size(); ++i) {
      o->reason[i] = static_cast<std::int32_t>(oc[i].reason);
      o->has_path[i] = oc[i].path ? 1 : 0;
      if (oc[i].path) put_exact(&o->paths, i, *oc[i].path);
    }
    *out = o;
  });
}

int pcrref_refine_batch(const void* grid, const void* scene, const pcr_paths* cands,
                        const pcr_refine_params* rp, int thread_count, pcr_outcomes** out) {
  return refine_batch_impl(grid, scene, cands, rp, thread_count, out, 0.0, nullptr);
}

// refine_path per candidate + the pipeline's dedup (bench CPU arm: exact paths counted
// the way RunSummary::exact_paths counts them); outcomes optional (out may be null)
int pcrref_refine_dedup_batch(const void* grid, const void* scene, const pcr_paths* cands,
                              const pcr_refine_params* rp, int thread_count, double carrier_frequency_hz,
                              uint64_t* n_exact, pcr_outcomes** out) {
  return refine_batch_impl(grid, scene, cands, rp, thread_count, out, carrier_frequency_hz, n_exact);
}

void pcrref_free_outcomes(pcr_outcomes* o) {
  if (!o) return;
  free_paths_arrays(&o->paths);
  std::free(o->has_path);
  std::free(o->reason);
  std::free(o);
}

// ---- whole pipeline ----------------------------------------------------------------
// RunSummary (pipeline.hpp:40-58) into the pcr_summary layout
static pcr_summary* summary_of(const RunSummary& rs) {
  pcr_summary* s = alloc<pcr_summary>(1);
  s->point_count = rs.point_count;
  s->edge_count = rs.edge_count;
  s->ie_count = rs.ie_count;
  for (int a = 0; a < 3; ++a) s->grid_dims[a] = rs.grid_dims[a];
  s->coarse_paths = rs.coarse_paths;
  s->refined_paths = rs.refined_paths;
  for (int r = 0; r < 4; ++r) s->rejected[r] = rs.rejected[r];
  s->exact_paths = rs.exact_paths;
  s->n_timings = static_cast<std::uint32_t>(std::min<std::size_t>(rs.timings.size(), PCR_MAX_STAGES));
  for (std::uint32_t t = 0; t < s->n_timings; ++t) {
    std::snprintf(s->timing_stage[t], sizeof(s->timing_stage[t]), "%s", rs.timings[t].stage.c_str());
    s->timing_seconds[t] = rs.timings[t].seconds;
  }
  s->hash = rs.hash;
  std::size_t stride = 1;
  for (const auto& p : rs.paths) stride = std::max(stride, p.interactions.size());
  pcr_paths* pp = alloc_paths(rs.paths.size(), static_cast<std::uint32_t>(stride));
  for (std::size_t i = 0; i < rs.paths.size(); ++i) put_exact(pp, i, rs.paths[i]);
  s->paths = *pp;
  std::free(pp);
  return s;
}

// run_pipeline_on_scene (pipeline.cpp:99-212)
int pcrref_run_pipeline_on_scene(const void* scene, const pcr_run_config* cfg, pcr_summary** out) {
  return guarded([&] { *out = summary_of(run_pipeline_on_scene(*static_cast<const Scene*>(scene), run_config(cfg))); });
}

// run_pipeline (pipeline.hpp:63-64): the file-level run, paths and radios from `files`
int pcrref_run_pipeline(const pcr_run_files* f, const pcr_run_config* cfg, pcr_summary** out) {
  return guarded([&] {
    RunConfig rc = run_config(cfg);
    if (f->scene_path) rc.scene_path = f->scene_path;
    if (f->edges_path) rc.edges_path = f->edges_path;
    if (f->output_path) rc.output_path = f->output_path;
    for (std::uint32_t i = 0; i < f->n_tx; ++i) rc.transmitters.push_back(get3(f->tx_position + 3 * i));
    for (std::uint32_t i = 0; i < f->n_rx; ++i) rc.receivers.push_back(get3(f->rx_position + 3 * i));
    *out = summary_of(run_pipeline(rc));
  });
}

// load_edges (io.hpp:19-21) into the pcr_edges layout
int pcrref_load_edges(const char* path, pcr_edges** out) {
  return guarded([&] {
    const auto edges = load_edges(path);
    pcr_edges* e = alloc<pcr_edges>(1);
    e->n = static_cast<std::uint32_t>(edges.size());
    e->geometry = alloc<double>(12 * edges.size() + 1);
    e->label = alloc<std::uint32_t>(edges.size() + 1);
    for (std::size_t i = 0; i < edges.size(); ++i) {
      put3(e->geometry + 12 * i, edges[i].start);
      put3(e->geometry + 12 * i + 3, edges[i].end);
      put3(e->geometry + 12 * i + 6, edges[i].normal_a);
      put3(e->geometry + 12 * i + 9, edges[i].normal_b);
      e->label[i] = edges[i].label;
    }
    *out = e;
  });
}

void pcrref_free_summary(pcr_summary* s) {
  if (!s) return;
  free_paths_arrays(&s->paths);
  std::free(s);
}

void pcrref_free_paths(pcr_paths* p) {
  if (!p) return;
  free_paths_arrays(p);
  std::free(p);
}

void pcrref_free_initial_hits(pcr_initial_hits* h) {
  if (!h) return;
  std::free(h->ie_index);
  std::free(h->kind);
  std::free(h->position);
  std::free(h->normal);
  std::free(h->incoming);
  std::free(h);
}

uint64_t pcrref_config_hash(const pcr_run_config* cfg) { return config_hash(run_config(cfg)); }

void pcrref_run_config_defaults(pcr_run_config* c) {
  const RunConfig r;
  c->carrier_frequency_hz = r.carrier_frequency_hz;
  c->voxel_size_m = r.voxel_size_m;
  c->division_factor = r.division_factor;
  c->kappa = r.kappa;
  c->max_interactions = r.max_interactions;
  c->max_diffractions = r.max_diffractions;
  c->cone_apex_angle_deg = r.cone_apex_angle_deg;
  c->diffraction_ray_count = r.diffraction_ray_count;
  c->delta = r.delta;
  c->rho = r.rho;
  c->step_size = r.step_size;
  c->seed = r.seed;
  c->thread_count = r.thread_count;
  c->fresnel_enabled = r.fresnel_enabled ? 1 : 0;
}

// ---- planar-scene sampler and image method (oracle.cpp:208-236, 55-117) ----------
// rects: n_rect*10 doubles (corner, e1, e2, label-as-double). Returns the point
// count; fills the arrays when they are non-null (call twice: size, then fill).
uint64_t pcrref_sample_planar_scene(const double* rects, uint32_t n_rect, double density,
                                    uint32_t seed, double* pos, double* nrm, uint32_t* label) {
  PlanarScene ps;
  for (std::uint32_t r = 0; r < n_rect; ++r) {
    const double* q = rects + 10 * r;
    ps.rectangles.push_back(PlanarRect{get3(q), get3(q + 3), get3(q + 6), static_cast<Label>(q[9])});
  }
  const auto pts = sample_planar_scene(ps, density, seed);
  if (pos) {
    for (std::size_t i = 0; i < pts.size(); ++i) {
      put3(pos + 3 * i, pts[i].position);
      put3(nrm + 3 * i, pts[i].normal);
      label[i] = pts[i].label;
    }
  }
  return pts.size();
}

int pcrref_image_method_paths(const double* rects, uint32_t n_rect, const double* tx,
                              const double* rx, int max_order, pcr_paths** out) {
  return guarded([&] {
    PlanarScene ps;
    for (std::uint32_t r = 0; r < n_rect; ++r) {
      const double* q = rects + 10 * r;
      ps.rectangles.push_back(PlanarRect{get3(q), get3(q + 3), get3(q + 6), static_cast<Label>(q[9])});
    }
    ps.tx = get3(tx);
    ps.rx = get3(rx);
    const auto paths = image_method_paths(ps, max_order);
    std::size_t stride = 1;
    for (const auto& p : paths) stride = std::max(stride, p.interactions.size());
    pcr_paths* pp = alloc_paths(paths.size(), static_cast<std::uint32_t>(stride));
    for (std::size_t i = 0; i < paths.size(); ++i) put_exact(pp, i, paths[i]);
    *out = pp;
  });
}

// save_point_cloud (io.hpp:16-17): the scene's points as a PLY file
int pcrref_save_point_cloud(const char* path, const void* scene, int binary) {
  return guarded([&] { save_point_cloud(path, static_cast<const Scene*>(scene)->points, binary != 0); });
}

// load_point_cloud (io.hpp:15): points into library-allocated arrays (pcrref_free)
int pcrref_load_point_cloud(const char* path, double** pos, double** nrm, uint32_t** label, uint64_t* n) {
  return guarded([&] {
    const auto pts = load_point_cloud(path);
    *n = pts.size();
    *pos = alloc<double>(3 * pts.size());
    *nrm = alloc<double>(3 * pts.size());
    *label = alloc<uint32_t>(pts.size());
    for (std::size_t i = 0; i < pts.size(); ++i) {
      put3(*pos + 3 * i, pts[i].position);
      put3(*nrm + 3 * i, pts[i].normal);
      (*label)[i] = pts[i].label;
    }
  });
}

void pcrref_free(void* p) { std::free(p); }

// write_paths (io.hpp:33-34) over exact paths given as a pcr_paths table
int pcrref_write_paths(const char* path, const pcr_paths* p, uint64_t config_hash) {
  return guarded([&] {
    std::vector<ExactPath> v(p->n);
    for (std::uint64_t i = 0; i < p->n; ++i) {
      ExactPath& e = v[i];
      e.tx_id = p->tx_id[i];
      e.rx_id = p->rx_id[i];
      e.tx_position = get3(p->tx_position + 3 * i);
      e.rx_position = get3(p->rx_position + 3 * i);
      e.total_length = p->length[i];
      e.delay = p->delay[i];
      e.converged = p->converged[i] != 0;
      e.gradient_norm = p->gradient_norm[i];
      for (std::uint32_t k = 0; k < p->n_inter[i]; ++k) {
        const std::size_t j = i * p->stride + k;
        Interaction it;
        it.kind = static_cast<InteractionKind>(p->kind[j]);
        it.position = get3(p->position + 3 * j);
        it.label = p->label[j];
        it.normal = get3(p->normal + 3 * j);
        it.ie_index = p->ie_index[j];
        it.edge_index = p->edge_index[j];
        e.interactions.push_back(it);
      }
    }
    write_paths(path, v, config_hash);
  });
}

}  // extern "C"
