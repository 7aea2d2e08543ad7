// helpers.cu — the reference's scalar public helpers as device batch primitives, so the
// C++ drop-in (adapter/pcray_gpu.cpp) answers every pcray:: call on the GPU with the same
// device functions the stage kernels use (one source, no host re-implementation):
//
//   estimate_surface, march_segment, project_to_surface, local_frame (surface.hpp:37-55)
//   cone_intersects_sphere, reflect_ray, diffract_rays                (tracer.hpp:91-113)
//   make_path_state, path_length, local_gradients                     (refine.hpp:69-75)
//
// One thread per item; inputs and outputs are host arrays copied through the context
// stream (these are API-surface calls: a test or a caller asks for a few items at a
// time; the pipeline itself never goes through them).
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "handles.cuh"
#include "host_alloc.hpp"
#include "pipeline.hpp"
#include "trace.cuh"

namespace pcr {
namespace {

constexpr unsigned kHT = 128;
unsigned hb(uint64_t n) { return static_cast<unsigned>(n ? (n + kHT - 1) / kHT : 1); }

template <typename T>
DBuf<T> up(const T* h, size_t n, cudaStream_t s) {
  DBuf<T> d(n ? n : 1, s);
  if (n) h2d(d.get(), h, n, s);
  return d;
}

__global__ void estimate_surface_kernel(GridView g, SceneView s, const double* __restrict__ x,
                                        const uint32_t* __restrict__ ie, uint64_t n, double* p_bar, double* n_bar,
                                        double* sdf, double* wsum) {
  const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  const SurfaceEstimate e = estimate_surface(load3(x + 3 * k), ie[k], g, s);
  store3(p_bar + 3 * k, e.p_bar);
  store3(n_bar + 3 * k, e.n_bar);
  sdf[k] = e.sdf;
  wsum[k] = e.weight_sum;
}

__global__ void march_segment_kernel(GridView g, SceneView s, const double* __restrict__ o,
                                     const double* __restrict__ d, const uint32_t* __restrict__ ie,
                                     const double* __restrict__ t_max, uint64_t n, uint8_t* hit, double* pos,
                                     double* nrm, uint32_t* label, double* dist) {
  const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  SurfaceHit h;
  const bool ok = march_segment(load3(o + 3 * k), load3(d + 3 * k), ie[k], g, s, t_max[k], &h);
  hit[k] = ok ? 1 : 0;
  if (!ok) return;
  store3(pos + 3 * k, h.position);
  store3(nrm + 3 * k, h.normal);
  label[k] = h.label;
  dist[k] = h.distance;
}

__global__ void project_kernel(GridView g, SceneView s, const double* __restrict__ x, const uint32_t* __restrict__ ie,
                               uint64_t n, uint8_t* hit, double* pos, double* nrm, uint32_t* label) {
  const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  SurfaceHit h;
  const bool ok = project_to_surface(load3(x + 3 * k), ie[k], g, s, &h);
  hit[k] = ok ? 1 : 0;
  if (!ok) return;
  store3(pos + 3 * k, h.position);
  store3(nrm + 3 * k, h.normal);
  label[k] = h.label;
}

__global__ void local_frame_kernel(const double* __restrict__ nrm, uint64_t n, double* u, double* v) {
  const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  V3 a, b;
  local_frame(load3(nrm + 3 * k), a, b);
  store3(u + 3 * k, a);
  store3(v + 3 * k, b);
}

// cone_intersects_sphere (tracer.cpp:129-136): the cone walk's test (trace.cuh
// cone_test, certified against glibc at the knife edge)
__global__ void cone_sphere_kernel(const double* __restrict__ o, const double* __restrict__ d,
                                   const double* __restrict__ alpha, const double* __restrict__ c,
                                   const double* __restrict__ r, uint64_t n, uint8_t* out) {
  const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  const V3 dd = load3(d + 3 * k);
  out[k] = cone_test(load3(o + 3 * k), dd, cone_consts(alpha[k], dd), load3(c + 3 * k), r[k]) ? 1 : 0;
}

__device__ void put_ray(pcr_ray_desc& r, const V3& o, const V3& d, double apex, int np, const V3* pn) {
  store3(r.origin, o);
  store3(r.direction, d);
  r.apex_angle = apex;
  r.n_planes = np;
  for (int q = 0; q < 2; ++q) {
    store3(r.plane_point[q], q < np ? o : V3{0, 0, 0});
    store3(r.plane_normal[q], q < np ? pn[q] : V3{0, 0, 1});
  }
  r.origin_ie = kNoIe;
  r.origin_label = 0;
}

// reflect_ray (tracer.cpp:257-267); spawn_apex_angle is the identity (:110-114)
__global__ void reflect_kernel(GridView g, const double* __restrict__ pos, const double* __restrict__ nrm,
                               const double* __restrict__ inc, uint64_t n, double apex, uint8_t* ok,
                               pcr_ray_desc* out) {
  const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  const V3 nn = load3(nrm + 3 * k), in = load3(inc + 3 * k);
  const double dn = dot(in, nn);
  ok[k] = dn < 0.0;
  if (dn >= 0.0) return;
  const V3 o = load3(pos + 3 * k) + g.hit_eps * nn;
  put_ray(out[k], o, normalized(in - (2.0 * dn) * nn), apex, 1, &nn);
}

// diffract_rays (tracer.cpp:269-311): ray j of the Keller fan, the stage kernels' fan
// frame and host sin/cos table
__global__ void diffract_kernel(SceneView s, uint32_t edge, V3 point, V3 inc, double apex, FanTable fan,
                                uint8_t* ok, pcr_ray_desc* out) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= static_cast<uint32_t>(fan.n)) return;
  V3 w, e1, e2, na, nb;
  double cos_b, sin_b;
  ok[j] = 0;
  if (!fan_frame(s.edges + 12ull * edge, inc, w, e1, e2, cos_b, sin_b, na, nb)) return;
  const double* t = fan.t + 6ull * j;
  const V3 dir = cos_b * w + sin_b * (t[0] * e1 + t[1] * e2);
  if (dot(dir, na) < 0.0 && dot(dir, nb) < 0.0) return;
  const V3 tp = (-t[2]) * e1 + t[3] * e2;
  const V3 pn[2] = {-tp, (-t[4]) * e1 + t[5] * e2};
  ok[j] = 1;
  put_ray(out[j], point, dir, apex, 2, pn);
}

// reception_point_of (voxel_grid.cpp:61-80): payload centroid summed in point_indices
// order, segment midpoint, RX position by id (the IE's own point when no radio matches)
__global__ void reception_point_kernel(GridView g, SceneView s, const double4* __restrict__ seg_s,
                                       const double4* __restrict__ seg_e, const double* __restrict__ rx_pos,
                                       const uint32_t* __restrict__ rx_id, uint32_t n_rx, const uint32_t* __restrict__ ie,
                                       uint64_t n, double* out) {
  const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  const uint32_t i = ie[k];
  V3 p = ld3(g.ie_rp[i]);
  const uint32_t kind = ie_kind(g, i);
  if (kind == kSurface) {
    const uint2 r = g.ie_range[i];
    V3 sum{0, 0, 0};
    for (uint32_t j = r.x; j < r.y; ++j) sum = sum + load3(s.pos + 3ull * g.point_indices[j]);
    p = sum / static_cast<double>(r.y - r.x);
  } else if (kind == kEdge) {
    p = 0.5 * (ld3(seg_s[i]) + ld3(seg_e[i]));
  } else {
    for (uint32_t q = 0; q < n_rx; ++q)
      if (rx_id[q] == g.ie_rx[i]) {
        p = load3(rx_pos + 3ull * q);
        break;
      }
  }
  store3(out + 3 * k, p);
}

// PathNode::point (refine.hpp:40-44)
__device__ __forceinline__ V3 pnode_point(const pcr_path_node& x) {
  return x.kind == 0 ? (load3(x.c) + x.r * load3(x.u)) + x.s * load3(x.v) : load3(x.c) + x.r * load3(x.u);
}

// make_path_state (refine.cpp:134-161)
__global__ void make_state_kernel(SceneView s, uint64_t n, uint32_t stride, const uint32_t* __restrict__ n_inter,
                                  const uint8_t* __restrict__ kind, const double* __restrict__ pos,
                                  const double* __restrict__ nrm, const uint32_t* __restrict__ label,
                                  const uint32_t* __restrict__ edge, pcr_path_node* out) {
  const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  for (uint32_t q = 0; q < n_inter[k]; ++q) {
    const uint64_t j = k * stride + q;
    pcr_path_node x;
    memset(&x, 0, sizeof(x));
    x.kind = kind[j];
    x.label = label[j];
    store3(x.c, load3(pos + 3 * j));
    if (x.kind == 0) {
      const V3 nn = load3(nrm + 3 * j);
      V3 u, v;
      local_frame(nn, u, v);
      store3(x.normal, nn);
      store3(x.u, u);
      store3(x.v, v);
    } else {
      x.edge_index = edge[j];
      const double* e = s.edges + 12ull * x.edge_index;
      const V3 es = load3(e), ee = load3(e + 3), c = load3(pos + 3 * j);
      const V3 w = normalized(ee - es);
      store3(x.u, w);
      x.t_min = dot(es - c, w);
      x.t_max = dot(ee - c, w);
    }
    out[j] = x;
  }
}

// path_length (refine.cpp:163-165) and local_gradients (:167-187)
__global__ void path_eval_kernel(uint64_t n, uint32_t stride, const double* __restrict__ tx,
                                 const double* __restrict__ rx, const uint32_t* __restrict__ n_nodes,
                                 const pcr_path_node* __restrict__ nodes, double* length, double* grads,
                                 uint8_t* grads_ok) {
  const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  const pcr_path_node* nd = nodes + k * stride;
  const uint32_t d = n_nodes[k];
  const V3 t = load3(tx + 3 * k), r = load3(rx + 3 * k);
  V3 prev = t;
  double len = 0.0;
  for (uint32_t q = 0; q < d; ++q) {
    const V3 p = pnode_point(nd[q]);
    len += norm(p - prev);
    prev = p;
  }
  length[k] = len + norm(r - prev);
  if (!grads) return;
  uint32_t gi = 0;
  grads_ok[k] = 1;
  for (uint32_t q = 0; q < d; ++q) {
    const V3 p = pnode_point(nd[q]);
    const V3 pv = q == 0 ? t : pnode_point(nd[q - 1]);
    const V3 nx = q + 1 == d ? r : pnode_point(nd[q + 1]);
    const V3 dp = p - pv, dn = p - nx;
    const double lp = norm(dp), ln = norm(dn);
    if (lp < kTiny || ln < kTiny) {
      grads_ok[k] = 0;
      return;
    }
    const V3 e_sum = dp / lp + dn / ln;
    double* gk = grads + k * 2ull * stride;
    gk[gi++] = dot(load3(nd[q].u), e_sum);
    if (nd[q].kind == 0) gk[gi++] = dot(load3(nd[q].v), e_sum);
  }
}

}  // namespace

void ensure_fan(Ctx& ctx, int n);  // trace.cu

}  // namespace pcr

using namespace pcr;

namespace {
template <typename F>
int guarded_h(pcr_ctx* ctx, F&& f) {
  if (!ctx) return PCR_ERR_INVALID;
  std::lock_guard<std::mutex> lock(ctx->c.mu);
  try {
    PCR_CUDA(cudaSetDevice(ctx->c.device));
    f();
    ctx->c.last_error.clear();
    return PCR_OK;
  } catch (const Error& e) {
    ctx->c.last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    ctx->c.last_error = e.what();
    return PCR_ERR_RUNTIME;
  }
}
void need(bool ok) {
  if (!ok) throw Error(PCR_ERR_INVALID, "null argument");
}
void check_ies(const GridDev& g, const uint32_t* ie, uint64_t n) {
  for (uint64_t k = 0; k < n; ++k)
    if (ie[k] >= g.n_ies) throw Error(PCR_ERR_INVALID, "ie index out of range");
}
}  // namespace

extern "C" {

int pcr_estimate_surface_batch(pcr_ctx* ctx, const pcr_grid* grid, const pcr_scene* scene, const double* x,
                               const uint32_t* ie, uint64_t n, double* p_bar, double* n_bar, double* sdf,
                               double* weight_sum) {
  return guarded_h(ctx, [&] {
    need(grid && scene && (!n || (x && ie && p_bar && n_bar && sdf && weight_sum)));
    check_ies(grid->g, ie, n);
    cudaStream_t s = ctx->c.stream;
    auto dx = up(x, 3 * n, s);
    auto di = up(ie, n, s);
    DBuf<double> pb(3 * n + 3, s), nb(3 * n + 3, s), sd(n + 1, s), ws(n + 1, s);
    if (n) {
      count_launch();
      estimate_surface_kernel<<<hb(n), kHT, 0, s>>>(grid->g.view_for(ctx->c, scene->s), scene->s.view(), dx.get(), di.get(), n, pb.get(),
                                                    nb.get(), sd.get(), ws.get());
      PCR_LAUNCH_CHECK();
      d2h(p_bar, pb.get(), 3 * n, s);
      d2h(n_bar, nb.get(), 3 * n, s);
      d2h(sdf, sd.get(), n, s);
      d2h(weight_sum, ws.get(), n, s);
    }
    stream_wait(s);
  });
}

int pcr_march_segment_batch(pcr_ctx* ctx, const pcr_grid* grid, const pcr_scene* scene, const double* origin,
                            const double* direction, const uint32_t* ie, const double* t_max, uint64_t n,
                            uint8_t* hit, double* position, double* normal, uint32_t* label, double* distance) {
  return guarded_h(ctx, [&] {
    need(grid && scene && (!n || (origin && direction && ie && t_max && hit && position && normal && label && distance)));
    check_ies(grid->g, ie, n);
    cudaStream_t s = ctx->c.stream;
    auto o = up(origin, 3 * n, s);
    auto d = up(direction, 3 * n, s);
    auto di = up(ie, n, s);
    auto tm = up(t_max, n, s);
    DBuf<uint8_t> h(n + 1, s);
    DBuf<double> p(3 * n + 3, s), nr(3 * n + 3, s), ds(n + 1, s);
    DBuf<uint32_t> lb(n + 1, s);
    if (n) {
      count_launch();
      march_segment_kernel<<<hb(n), kHT, 0, s>>>(grid->g.view_for(ctx->c, scene->s), scene->s.view(), o.get(), d.get(), di.get(), tm.get(),
                                                 n, h.get(), p.get(), nr.get(), lb.get(), ds.get());
      PCR_LAUNCH_CHECK();
      d2h(hit, h.get(), n, s);
      d2h(position, p.get(), 3 * n, s);
      d2h(normal, nr.get(), 3 * n, s);
      d2h(label, lb.get(), n, s);
      d2h(distance, ds.get(), n, s);
    }
    stream_wait(s);
  });
}

int pcr_project_to_surface_batch(pcr_ctx* ctx, const pcr_grid* grid, const pcr_scene* scene, const double* x,
                                 const uint32_t* ie, uint64_t n, uint8_t* hit, double* position, double* normal,
                                 uint32_t* label) {
  return guarded_h(ctx, [&] {
    need(grid && scene && (!n || (x && ie && hit && position && normal && label)));
    check_ies(grid->g, ie, n);
    cudaStream_t s = ctx->c.stream;
    auto dx = up(x, 3 * n, s);
    auto di = up(ie, n, s);
    DBuf<uint8_t> h(n + 1, s);
    DBuf<double> p(3 * n + 3, s), nr(3 * n + 3, s);
    DBuf<uint32_t> lb(n + 1, s);
    if (n) {
      count_launch();
      project_kernel<<<hb(n), kHT, 0, s>>>(grid->g.view_for(ctx->c, scene->s), scene->s.view(), dx.get(), di.get(), n, h.get(), p.get(),
                                           nr.get(), lb.get());
      PCR_LAUNCH_CHECK();
      d2h(hit, h.get(), n, s);
      d2h(position, p.get(), 3 * n, s);
      d2h(normal, nr.get(), 3 * n, s);
      d2h(label, lb.get(), n, s);
    }
    stream_wait(s);
  });
}

int pcr_reception_point_batch(pcr_ctx* ctx, const pcr_grid* grid, const pcr_scene* scene, const uint32_t* ie,
                              uint64_t n, double* point) {
  return guarded_h(ctx, [&] {
    need(grid && scene && (!n || (ie && point)));
    check_ies(grid->g, ie, n);
    cudaStream_t s = ctx->c.stream;
    auto di = up(ie, n, s);
    DBuf<double> out(3 * n + 3, s);
    if (n) {
      const SceneDev& sd = scene->s;
      count_launch();
      reception_point_kernel<<<hb(n), kHT, 0, s>>>(grid->g.view(), sd.view(), grid->g.seg_s.get(), grid->g.seg_e.get(),
                                                   sd.rx_pos.get(), sd.rx_id.get(),
                                                   static_cast<uint32_t>(sd.h_rx_id.size()), di.get(), n, out.get());
      PCR_LAUNCH_CHECK();
      d2h(point, out.get(), 3 * n, s);
    }
    stream_wait(s);
  });
}

int pcr_local_frame_batch(pcr_ctx* ctx, const double* normal, uint64_t n, double* u, double* v) {
  return guarded_h(ctx, [&] {
    need(!n || (normal && u && v));
    cudaStream_t s = ctx->c.stream;
    auto dn = up(normal, 3 * n, s);
    DBuf<double> du(3 * n + 3, s), dv(3 * n + 3, s);
    if (n) {
      count_launch();
      local_frame_kernel<<<hb(n), kHT, 0, s>>>(dn.get(), n, du.get(), dv.get());
      PCR_LAUNCH_CHECK();
      d2h(u, du.get(), 3 * n, s);
      d2h(v, dv.get(), 3 * n, s);
    }
    stream_wait(s);
  });
}

int pcr_cone_intersects_sphere_batch(pcr_ctx* ctx, const double* o, const double* d, const double* alpha,
                                     const double* c, const double* r, uint64_t n, uint8_t* out) {
  return guarded_h(ctx, [&] {
    need(!n || (o && d && alpha && c && r && out));
    cudaStream_t s = ctx->c.stream;
    auto a = up(o, 3 * n, s), b = up(d, 3 * n, s), al = up(alpha, n, s), cc = up(c, 3 * n, s), rr = up(r, n, s);
    DBuf<uint8_t> res(n + 1, s);
    if (n) {
      count_launch();
      cone_sphere_kernel<<<hb(n), kHT, 0, s>>>(a.get(), b.get(), al.get(), cc.get(), rr.get(), n, res.get());
      PCR_LAUNCH_CHECK();
      d2h(out, res.get(), n, s);
    }
    stream_wait(s);
  });
}

int pcr_reflect_ray_batch(pcr_ctx* ctx, const pcr_grid* grid, const double* hit_position, const double* hit_normal,
                          const double* incoming, uint64_t n, const pcr_trace_params* params, uint8_t* ok,
                          pcr_ray_desc* rays) {
  return guarded_h(ctx, [&] {
    need(grid && params && (!n || (hit_position && hit_normal && incoming && ok && rays)));
    cudaStream_t s = ctx->c.stream;
    auto p = up(hit_position, 3 * n, s), nr = up(hit_normal, 3 * n, s), in = up(incoming, 3 * n, s);
    DBuf<uint8_t> dok(n + 1, s);
    DBuf<pcr_ray_desc> dr(n + 1, s);
    if (n) {
      count_launch();
      reflect_kernel<<<hb(n), kHT, 0, s>>>(grid->g.view(), p.get(), nr.get(), in.get(), n, params->cone_apex_angle,
                                           dok.get(), dr.get());
      PCR_LAUNCH_CHECK();
      d2h(ok, dok.get(), n, s);
      d2h(rays, dr.get(), n, s);
    }
    stream_wait(s);
  });
}

int pcr_diffract_rays(pcr_ctx* ctx, const pcr_scene* scene, uint32_t edge_index, const double* point,
                      const double* incoming, const pcr_trace_params* params, pcr_ray_desc** rays, uint64_t* n_rays) {
  return guarded_h(ctx, [&] {
    need(scene && point && incoming && params && rays && n_rays);
    if (edge_index >= scene->s.n_edges) throw Error(PCR_ERR_INVALID, "edge index out of range");
    if (params->diffraction_ray_count < 1) throw Error(PCR_ERR_INVALID, "diffraction_ray_count must be >= 1");
    cudaStream_t s = ctx->c.stream;
    const int fan_n = params->diffraction_ray_count;
    ensure_fan(ctx->c, fan_n);
    DBuf<uint8_t> dok(fan_n, s);
    DBuf<pcr_ray_desc> dr(fan_n, s);
    count_launch();
    diffract_kernel<<<hb(fan_n), kHT, 0, s>>>(scene->s.view(), edge_index, load3(point), load3(incoming),
                                              params->cone_apex_angle, FanTable{ctx->c.fan_table.get(), fan_n},
                                              dok.get(), dr.get());
    PCR_LAUNCH_CHECK();
    std::vector<uint8_t> h_ok(fan_n);
    std::vector<pcr_ray_desc> h_r(fan_n);
    d2h(h_ok.data(), dok.get(), fan_n, s);
    d2h(h_r.data(), dr.get(), fan_n, s);
    stream_wait(s);
    uint64_t m = 0;
    for (int j = 0; j < fan_n; ++j) m += h_ok[j];
    pcr_ray_desc* out = halloc<pcr_ray_desc>(m ? m : 1);
    m = 0;
    for (int j = 0; j < fan_n; ++j)
      if (h_ok[j]) out[m++] = h_r[j];
    *rays = out;
    *n_rays = m;
  });
}

int pcr_make_path_state(pcr_ctx* ctx, const pcr_scene* scene, const pcr_paths* candidates, pcr_path_node* nodes) {
  return guarded_h(ctx, [&] {
    need(scene && candidates && (!candidates->n || nodes));
    const uint64_t n = candidates->n;
    const uint32_t st = candidates->stride ? candidates->stride : 1;
    for (uint64_t k = 0; k < n; ++k) {
      if (candidates->n_inter[k] > st) throw Error(PCR_ERR_INVALID, "path longer than its stride");
      for (uint32_t q = 0; q < candidates->n_inter[k]; ++q)
        if (candidates->kind[k * st + q] != 0 && candidates->edge_index[k * st + q] >= scene->s.n_edges)
          throw Error(PCR_ERR_INVALID, "edge index out of range");
    }
    if (!n) return;
    cudaStream_t s = ctx->c.stream;
    auto ni = up(candidates->n_inter, n, s);
    auto kd = up(candidates->kind, n * st, s);
    auto ps = up(candidates->position, 3 * n * st, s);
    auto nr = up(candidates->normal, 3 * n * st, s);
    auto lb = up(candidates->label, n * st, s);
    auto ed = up(candidates->edge_index, n * st, s);
    DBuf<pcr_path_node> out(n * st, s);
    PCR_CUDA(cudaMemsetAsync(out.get(), 0, n * st * sizeof(pcr_path_node), s));
    count_launch();
    make_state_kernel<<<hb(n), kHT, 0, s>>>(scene->s.view(), n, st, ni.get(), kd.get(), ps.get(), nr.get(), lb.get(),
                                            ed.get(), out.get());
    PCR_LAUNCH_CHECK();
    d2h(nodes, out.get(), n * st, s);
    stream_wait(s);
  });
}

int pcr_path_eval_batch(pcr_ctx* ctx, const double* tx, const double* rx, const uint32_t* n_nodes,
                        const pcr_path_node* nodes, uint32_t stride, uint64_t n, double* length, double* gradients,
                        uint8_t* gradients_ok) {
  return guarded_h(ctx, [&] {
    need(!n || (tx && rx && n_nodes && nodes && length && (!gradients || gradients_ok)));
    const uint32_t st = stride ? stride : 1;
    for (uint64_t k = 0; k < n; ++k)
      if (n_nodes[k] > st) throw Error(PCR_ERR_INVALID, "path longer than its stride");
    if (!n) return;
    cudaStream_t s = ctx->c.stream;
    auto t = up(tx, 3 * n, s), r = up(rx, 3 * n, s);
    auto nn = up(n_nodes, n, s);
    auto nd = up(nodes, n * st, s);
    DBuf<double> len(n, s), gr(gradients ? 2 * n * st : 1, s);
    DBuf<uint8_t> gok(n, s);
    count_launch();
    path_eval_kernel<<<hb(n), kHT, 0, s>>>(n, st, t.get(), r.get(), nn.get(), nd.get(), len.get(),
                                           gradients ? gr.get() : nullptr, gok.get());
    PCR_LAUNCH_CHECK();
    d2h(length, len.get(), n, s);
    if (gradients) {
      d2h(gradients, gr.get(), 2 * n * st, s);
      d2h(gradients_ok, gok.get(), n, s);
    }
    stream_wait(s);
  });
}

}  // extern "C"

extern "C" void pcr_free_rays(pcr_ray_desc* rays) { std::free(rays); }
