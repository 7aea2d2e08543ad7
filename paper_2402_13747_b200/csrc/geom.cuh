// geom.cuh — device views of the scene and the voxel grid, and the per-ray
// primitives every stage shares: point-set intersection (surface.cpp), the
// Amanatides–Woo walker, cone/sphere tests and straight-line visibility
// (tracer.cpp). Each function follows the cited reference lines operation by
// operation (see exact.cuh for the arithmetic-order contract).
#pragma once

#include <cstdint>

#include "exact.cuh"
#include "exp_table.cuh"

namespace pcr {

enum : uint32_t { kSurface = 0, kEdge = 1, kReceiver = 2 };
constexpr uint32_t kNoIe = 0xffffffffu;
constexpr int32_t kMarchNoIes = 2147483647;

// Device-resident VoxelGrid (voxel_grid.hpp:58-94). IE fields are SoA; the four
// vectors used by the hot loops are padded to double4 so one record is two
// 16-byte loads. sc.w carries sphere_radius.
struct GridView {
  V3 origin;
  int dims[3];
  double voxel_size;
  int dv;
  double sub_edge, sub_radius, voxel_radius, hit_eps;  // grid helpers, host-computed (voxel_grid.hpp:68-71)
  uint32_t n_cells, n_ies;
  const int4* cells;          // {ie_begin, ie_end, march, 0}
  const uint32_t* ie_meta;    // bits 0-1: kind, bit 2: planar
  const uint32_t* ie_label;
  const double4* ie_sc;       // sphere center, w = sphere radius
  const double4* ie_rp;       // reception point
  const double4* ie_pp;       // plane point
  const double4* ie_pn;       // plane normal
  const uint2* ie_range;      // point_begin, point_end
  const uint32_t* ie_edge;
  const uint32_t* ie_rx;
  const uint32_t* point_indices;
  int march_ok = 0;  // cells[].z are exact march distances (visibility may skip empty space)
  // refinement scan records (built per refine call): {sphere centre, label | meta << 32};
  // rr_radius is every IE's sphere radius when rr_uniform (as build_grid makes them)
  const double4* ie_rr = nullptr;
  double rr_radius = 0.0;
  int rr_uniform = 0;
  // per cell: the surface IEs of its clamped 3x3x3 neighbourhood, scan order (cells
  // z->y->x, IEs in cell order) stably sorted by label, as
  // {sphere centre, label | planar << 32 | ie << 33}
  const uint32_t* nb_off = nullptr;  // n_cells + 1
  const double4* nb_rec = nullptr;
  const uint32_t* nb_lab = nullptr;  // label of each list entry (lists are stably sorted by label)
  const double4* nb_pa = nullptr;    // per entry: plane point, sphere radius
  const double4* nb_pb = nullptr;    // per entry: plane normal
  // exact fast rejection in the planar reprojection scan (refine.cu planar_candidate_at):
  // set when the scene's coordinates are small enough for its error bound
  int fast_reject = 0;
  int seed_scan = 0;  // refine: seed the same-label scans with the last winner (grids with non-planar IEs)
  // non-planar payloads in point_indices order (positions / normals gathered once per
  // stage call, GridDev::view_for): estimate_surface streams them instead of a dependent
  // point_indices -> scene gather per point; null when the grid has no non-planar IE
  const double* pay_pos = nullptr;
  const double* pay_nrm = nullptr;
};

// Device-resident Scene (scene.hpp:38-46).
struct SceneView {
  const double* pos;  // n*3
  const double* nrm;  // n*3
  const uint32_t* label;
  uint64_t n_points;
  const double* edges;  // n_edges*12
  const uint32_t* edge_label;
  uint32_t n_edges;
};

__device__ __forceinline__ V3 ld3(const double4& v) { return V3{v.x, v.y, v.z}; }
__device__ __forceinline__ V3 ie_center(const GridView& g, uint32_t i) { return ld3(g.ie_sc[i]); }
__device__ __forceinline__ double ie_radius(const GridView& g, uint32_t i) { return g.ie_sc[i].w; }
__device__ __forceinline__ uint32_t ie_kind(const GridView& g, uint32_t i) { return g.ie_meta[i] & 3u; }
__device__ __forceinline__ bool ie_planar(const GridView& g, uint32_t i) { return (g.ie_meta[i] >> 2) & 1u; }

__device__ __forceinline__ bool in_bounds(const GridView& g, int x, int y, int z) {
  return x >= 0 && y >= 0 && z >= 0 && x < g.dims[0] && y < g.dims[1] && z < g.dims[2];
}
__device__ __forceinline__ uint32_t linear_index(const GridView& g, int x, int y, int z) {
  return static_cast<uint32_t>(x + g.dims[0] * (y + g.dims[1] * z));
}
// voxel_grid.hpp:90-92: origin + (v + 0.5) * voxel_size
__device__ __forceinline__ V3 voxel_center(const GridView& g, int x, int y, int z) {
  return V3{g.origin.x + (static_cast<double>(x) + 0.5) * g.voxel_size,
            g.origin.y + (static_cast<double>(y) + 0.5) * g.voxel_size,
            g.origin.z + (static_cast<double>(z) + 0.5) * g.voxel_size};
}

// ---------------------------------------------------------------------------------
// Point-set intersection (surface.cpp)
struct SurfaceHit {
  V3 position, normal;
  uint32_t label;
  double distance;
};

struct SurfaceEstimate {
  V3 p_bar, n_bar;
  double sdf, weight_sum;
};

// exp() as the host libm computes it (glibc >= 2.28's table-driven exp, in the FMA
// build the x86-64 loader selects): k = round(x * 128/ln2), r = x - k ln2/128 in two
// parts, exp(r) - 1 by a degree-5 polynomial, times 2^(k/128) from kExpTab, with the
// scaled paths near overflow / underflow. The fused operations are explicit fma()
// (the rest of the library is built without contraction). Equal to the host's exp()
// bit for bit on 20M random arguments over its whole range (tools/gen_exp_table.py,
// tests/test_nonplanar_gpu.py), which makes the non-planar SDF bit-exact.
__device__ __forceinline__ double glibc_exp(double x) {
  const double inv_ln2_n = 0x1.71547652b82fep0 * 128, neg_ln2_hi_n = -0x1.62e42fefa0000p-8,
               neg_ln2_lo_n = -0x1.cf79abc9e3b3ap-47, shift = 0x1.8p52;
  const double c2 = 0x1.ffffffffffdbdp-2, c3 = 0x1.555555555543cp-3, c4 = 0x1.55555cf172b91p-5,
               c5 = 0x1.1111167a4d017p-7;
  auto top12 = [](double v) { return static_cast<uint32_t>(static_cast<uint64_t>(__double_as_longlong(v)) >> 52); };
  uint32_t abstop = top12(x) & 0x7ff;
  if (abstop - top12(0x1p-54) >= top12(512.0) - top12(0x1p-54)) {
    if (static_cast<int32_t>(abstop - top12(0x1p-54)) < 0) return 1.0 + x;  // |x| < 2^-54
    if (abstop >= top12(1024.0)) {
      if (__double_as_longlong(x) == __double_as_longlong(-__longlong_as_double(0x7ff0000000000000ll))) return 0.0;
      if (abstop >= 0x7ff) return 1.0 + x;  // inf or nan
      return (static_cast<uint64_t>(__double_as_longlong(x)) >> 63) ? 0.0
                                                                     : __longlong_as_double(0x7ff0000000000000ll);
    }
    abstop = 0;  // large |x|: scaled below
  }
  double kd = fma(inv_ln2_n, x, shift);
  const uint64_t ki = static_cast<uint64_t>(__double_as_longlong(kd));
  kd -= shift;
  const double r = fma(kd, neg_ln2_lo_n, fma(kd, neg_ln2_hi_n, x));
  const uint64_t idx = 2 * (ki % 128);
  const uint64_t top = ki << 45;
  const double tail = __longlong_as_double(static_cast<long long>(kExpTab[idx]));
  uint64_t sbits = kExpTab[idx + 1] + top;
  const double r2 = r * r;
  const double tmp = fma(r2 * r2, fma(r, c5, c4), fma(r2, fma(r, c3, c2), tail + r));
  if (abstop != 0) {
    const double scale = __longlong_as_double(static_cast<long long>(sbits));
    return fma(scale, tmp, scale);
  }
  if ((ki & 0x80000000u) == 0) {  // k > 0: the scale's exponent may have overflowed
    sbits -= 1009ull << 52;
    const double scale = __longlong_as_double(static_cast<long long>(sbits));
    return 0x1p1009 * fma(scale, tmp, scale);
  }
  sbits += 1022ull << 52;  // k < 0: round once before scaling into the subnormal range
  const double scale = __longlong_as_double(static_cast<long long>(sbits));
  double y = __dadd_rn(scale, __dmul_rn(scale, tmp));
  if (y < 1.0) {
    double lo = __dadd_rn(scale - y, __dmul_rn(scale, tmp));
    const double hi = 1.0 + y;
    lo = 1.0 - hi + y + lo;
    y = (hi + lo) - 1.0;
    if (y == 0.0) y = 0.0;
  }
  return 0x1p-1022 * y;
}

// estimate_surface (surface.cpp:24-62). Non-planar payloads only; exp() is the host
// libm's (glibc_exp above).
static __device__ __noinline__ SurfaceEstimate estimate_surface(const V3& x, uint32_t ie, const GridView& g,
                                                                const SceneView& s) {
  const double h = g.sub_edge;
  const double inv_h2 = 1.0 / (h * h);
  V3 p_sum{0, 0, 0}, n_sum{0, 0, 0};
  double w_sum = 0.0;
  double best_d2 = 1.7976931348623157e308;
  const uint2 r = g.ie_range[ie];
  uint32_t best = r.x;
  const bool staged = g.pay_pos != nullptr;
  // unrolled: consecutive points' exp() chains are independent and overlap; the sums
  // still run in point order
#pragma unroll 4
  for (uint32_t i = r.x; i < r.y; ++i) {
    V3 p, n;
    if (staged) {
      p = load3(g.pay_pos + 3ull * i);
      n = load3(g.pay_nrm + 3ull * i);
    } else {
      const uint32_t pi = g.point_indices[i];
      p = load3(s.pos + 3ull * pi);
      n = load3(s.nrm + 3ull * pi);
    }
    const double d2 = sqnorm(x - p);
    if (d2 < best_d2) {
      best_d2 = d2;
      best = i;
    }
    const double w = glibc_exp(-d2 * inv_h2);
    w_sum += w;
    p_sum = p_sum + w * p;
    n_sum = n_sum + w * n;
  }
  SurfaceEstimate est;
  if (w_sum > 0.0 && norm(n_sum) > 0.0) {
    est.p_bar = p_sum / w_sum;
    est.n_bar = normalized(n_sum);
    est.weight_sum = w_sum;
  } else {
    const uint32_t pi = g.point_indices[best];
    est.p_bar = load3(s.pos + 3ull * pi);
    est.n_bar = load3(s.nrm + 3ull * pi);
    est.weight_sum = 0.0;
  }
  est.sdf = dot(x - est.p_bar, est.n_bar);
  return est;
}

// sdf_value_at (surface.cpp:16-20)
__device__ __forceinline__ double sdf_value_at(const V3& x, uint32_t ie, bool planar, const V3& pp,
                                               const V3& pn, const GridView& g, const SceneView& s) {
  if (planar) return dot(x - pp, pn);
  return estimate_surface(x, ie, g, s).sdf;
}

static __device__ __noinline__ bool march_window(const V3& origin, const V3& dir, uint32_t ie, const GridView& g,
                                                 const SceneView& s, double t_lo, double t_hi, SurfaceHit* out);

// march_segment's planar branch (surface.cpp:74-106) on the window [t_lo, t_hi]:
// endpoint / sign test, then the exact snap t* = (pp-o)·n / (d·n) when it falls in
// the window. Returns the hit distance only (the record is o + t·d, the plane normal
// and the IE label), false for std::nullopt.
__device__ __forceinline__ bool planar_march_t(const V3& origin, const V3& dir, uint32_t ie, const GridView& g,
                                               double t_lo, double t_hi, double& t) {
  if (t_hi <= t_lo) return false;
  const double eps = g.hit_eps;
  const double4 pp4 = g.ie_pp[ie], pn4 = g.ie_pn[ie];
  const V3 pp = ld3(pp4), pn = ld3(pn4);
  double tc;
  const double f = dot((origin + t_lo * dir) - pp, pn);
  if (fabs(f) <= eps) {
    tc = t_lo;
  } else {
    const double f_hi = dot((origin + t_hi * dir) - pp, pn);
    if (f * f_hi < 0.0)
      tc = 0.5 * (t_lo + t_hi);
    else if (fabs(f_hi) <= eps)
      tc = t_hi;
    else
      return false;
  }
  const double dn = dot(dir, pn);
  if (fabs(dn) > 1e-12) {
    const double t_star = dot(pp - origin, pn) / dn;
    if (t_star >= t_lo && t_star <= t_hi) tc = t_star;
  }
  t = tc;
  return true;
}

// march_segment (surface.cpp:64-134); returns false for std::nullopt. The planar
// route (the only one the rectangle scenes take) is inlined; sphere tracing over the
// Gaussian SDF lives out of line in march_window.
__device__ __forceinline__ bool march_segment(const V3& origin, const V3& dir, uint32_t ie, const GridView& g,
                                              const SceneView& s, double t_max, SurfaceHit* out) {
  const double eps = g.hit_eps;
  const double4 sc4 = g.ie_sc[ie];
  const V3 sc = ld3(sc4);
  const double r = sc4.w;
  const double t_center = dot(sc - origin, dir);
  const double t_lo = smax(0.0, t_center - r);
  const double t_hi = smin(t_center + r, t_max);
  if (t_hi <= t_lo) return false;
  if (!ie_planar(g, ie)) return march_window(origin, dir, ie, g, s, t_lo, t_hi, out);
  double t;
  if (!planar_march_t(origin, dir, ie, g, t_lo, t_hi, t)) return false;
  if (out) {  // make_hit (surface.cpp:98-106)
    out->position = origin + t * dir;
    out->normal = ld3(g.ie_pn[ie]);
    out->label = g.ie_label[ie];
    out->distance = t;
  }
  return true;
}

static __device__ __noinline__ bool march_window(const V3& origin, const V3& dir, uint32_t ie, const GridView& g,
                                                 const SceneView& s, double t_lo, double t_hi, SurfaceHit* out) {
  const double eps = g.hit_eps;
  const bool planar = ie_planar(g, ie);
  V3 pp{0, 0, 0}, pn{0, 0, 1};
  if (planar) {
    pp = ld3(g.ie_pp[ie]);
    pn = ld3(g.ie_pn[ie]);
  }
  auto make_hit = [&](double t) {
    if (planar) {
      const double dn = dot(dir, pn);
      if (fabs(dn) > 1e-12) {
        const double t_star = dot(pp - origin, pn) / dn;
        if (t_star >= t_lo && t_star <= t_hi) t = t_star;
      }
    }
    const V3 pos = origin + t * dir;
    if (out) {
      out->position = pos;
      out->normal = planar ? pn : estimate_surface(pos, ie, g, s).n_bar;
      out->label = g.ie_label[ie];
      out->distance = t;
    }
    return true;
  };

  double t = t_lo;
  double f = sdf_value_at(origin + t * dir, ie, planar, pp, pn, g, s);
  if (fabs(f) <= eps) return make_hit(t);

  if (planar) {
    const double f_hi = sdf_value_at(origin + t_hi * dir, ie, planar, pp, pn, g, s);
    if (f * f_hi < 0.0) return make_hit(0.5 * (t_lo + t_hi));
    if (fabs(f_hi) <= eps) return make_hit(t_hi);
    return false;
  }

  for (int step = 0; step < 32; ++step) {
    const bool at_end = t + fabs(f) >= t_hi;
    const double t_next = at_end ? t_hi : t + fabs(f);
    const double f_next = sdf_value_at(origin + t_next * dir, ie, planar, pp, pn, g, s);
    if (fabs(f_next) <= eps) return make_hit(t_next);
    if (f * f_next < 0.0) {
      double a = t, b = t_next, fa = f;
      for (int i = 0; i < 64; ++i) {
        const double m = 0.5 * (a + b);
        const double fm = sdf_value_at(origin + m * dir, ie, planar, pp, pn, g, s);
        if (fabs(fm) <= eps) return make_hit(m);
        if (fa * fm < 0.0) {
          b = m;
        } else {
          a = m;
          fa = fm;
        }
      }
      return make_hit(0.5 * (a + b));
    }
    if (at_end) return false;
    t = t_next;
    f = f_next;
  }
  return false;
}

// project_to_surface (surface.cpp:136-162)
__device__ inline bool project_to_surface(const V3& x, uint32_t ie, const GridView& g, const SceneView& s,
                                          SurfaceHit* out) {
  const double eps = g.hit_eps;
  V3 p = x;
  if (ie_planar(g, ie)) {
    const V3 pp = ld3(g.ie_pp[ie]);
    const V3 pn = ld3(g.ie_pn[ie]);
    p = p - dot(p - pp, pn) * pn;
    out->position = p;
    out->normal = pn;
    out->label = g.ie_label[ie];
    out->distance = 0.0;
    return true;
  }
  for (int i = 0; i < 16; ++i) {
    const SurfaceEstimate est = estimate_surface(p, ie, g, s);
    if (fabs(est.sdf) <= eps) {
      out->position = p;
      out->normal = est.n_bar;
      out->label = g.ie_label[ie];
      out->distance = 0.0;
      return true;
    }
    p = p - est.sdf * est.n_bar;
  }
  return false;
}

// ---------------------------------------------------------------------------------
// GridWalker (tracer.cpp:18-92)
// (inline: out of line the C2 cone walk measured 983 -> 1046 ms, C3 6.86 -> 7.69 s)
#ifndef PCR_INIT_AT_INLINE
#define PCR_INIT_AT_INLINE __forceinline__
#endif
struct Walker {
  V3 o, d;
  double t_end;
  int v[3], step[3];
  double t_next[3], delta[3];
  double t_entry;
  bool active;
  // per-ray part of init (the box clip per axis, the steps and increments): cached so
  // that the cone walk's re-inits after an empty-space skip (march >= 2) only redo the
  // entry point — the same operations on the same inputs, so the same walk. Same box:
  // C2 cone walk 1009 -> 983 ms, C3 8.25 -> 6.87 s (profiles/ab_walker_reinit_r02.log)
  double ta[3], tb[3];
  bool par[3], miss;

  __device__ __forceinline__ void init(const GridView& g, const V3& origin, const V3& dir, double t0, double t1) {
    prepare(g, origin, dir);
    init_at(g, t0, t1);
  }

  __device__ __forceinline__ void prepare(const GridView& g, const V3& origin, const V3& dir) {
    o = origin;
    d = dir;
    miss = false;
    const double od[3] = {o.x, o.y, o.z};
    const double dd[3] = {d.x, d.y, d.z};
    const double gd[3] = {g.origin.x, g.origin.y, g.origin.z};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double bmin = gd[a];
      const double bmax = gd[a] + static_cast<double>(g.dims[a]) * g.voxel_size;
      par[a] = fabs(dd[a]) < kTiny;
      if (par[a]) {
        if (od[a] < bmin || od[a] > bmax) miss = true;
        ta[a] = tb[a] = 0.0;
      } else {
        double lo_a = (bmin - od[a]) / dd[a];
        double hi_a = (bmax - od[a]) / dd[a];
        if (lo_a > hi_a) {
          const double tmp = lo_a;
          lo_a = hi_a;
          hi_a = tmp;
        }
        ta[a] = lo_a;
        tb[a] = hi_a;
      }
      if (dd[a] > kTiny) {
        step[a] = 1;
        delta[a] = g.voxel_size / dd[a];
      } else if (dd[a] < -kTiny) {
        step[a] = -1;
        delta[a] = -g.voxel_size / dd[a];
      } else {
        step[a] = 0;
        delta[a] = 0.0;
      }
    }
  }

  __device__ PCR_INIT_AT_INLINE void init_at(const GridView& g, double t0, double t1) {
    t_end = t1;
    active = false;
    if (miss) return;
    double lo = t0, hi = t1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (par[a]) continue;
      lo = smax(lo, ta[a]);
      hi = smin(hi, tb[a]);
    }
    if (lo > hi) return;
    t_entry = lo;
    const double od[3] = {o.x, o.y, o.z};
    const double dd[3] = {d.x, d.y, d.z};
    const double gd[3] = {g.origin.x, g.origin.y, g.origin.z};
    const double p[3] = {od[0] + lo * dd[0], od[1] + lo * dd[1], od[2] + lo * dd[2]};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      v[a] = sclamp(static_cast<int>(floor((p[a] - gd[a]) / g.voxel_size)), 0, g.dims[a] - 1);
      if (step[a] > 0)
        t_next[a] = ((gd[a] + static_cast<double>(v[a] + 1) * g.voxel_size) - od[a]) / dd[a];
      else if (step[a] < 0)
        t_next[a] = ((gd[a] + static_cast<double>(v[a]) * g.voxel_size) - od[a]) / dd[a];
      else
        t_next[a] = __longlong_as_double(0x7ff0000000000000ll);
    }
    active = true;
  }

  // init() for a walker in shared memory, computed by the warp: lanes 0..2 take one axis
  // each (box clip, step, increment, entry voxel, first crossing), the entry point is
  // reduced over the axes in the serial order on every lane, and each lane writes its
  // axis (lane 0 the rest). Called by all 32 lanes; same fields, same bits as init().
  __device__ __forceinline__ void init_warp(const GridView& g, const V3& origin, const V3& dir, double t0,
                                            double t1, int lane) {
    const int a = lane < 3 ? lane : 0;
    const double od = a == 0 ? origin.x : a == 1 ? origin.y : origin.z;
    const double dd = a == 0 ? dir.x : a == 1 ? dir.y : dir.z;
    const double gd = a == 0 ? g.origin.x : a == 1 ? g.origin.y : g.origin.z;
    const double bmin = gd;
    const double bmax = gd + static_cast<double>(g.dims[a]) * g.voxel_size;
    const bool pa = fabs(dd) < kTiny;
    const bool out = pa && (od < bmin || od > bmax);
    double lo_a = 0.0, hi_a = 0.0;
    if (!pa) {
      lo_a = (bmin - od) / dd;
      hi_a = (bmax - od) / dd;
      if (lo_a > hi_a) {
        const double tmp = lo_a;
        lo_a = hi_a;
        hi_a = tmp;
      }
    }
    double lo = t0, hi = t1;
    bool any_out = false;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const bool pb = __shfl_sync(0xffffffffu, pa, b);
      const bool ob = __shfl_sync(0xffffffffu, out, b);
      const double tab = __shfl_sync(0xffffffffu, lo_a, b), tbb = __shfl_sync(0xffffffffu, hi_a, b);
      any_out = any_out || ob;
      if (!pb) {
        lo = smax(lo, tab);
        hi = smin(hi, tbb);
      }
    }
    const bool ok = !any_out && !(lo > hi);
    if (lane < 3) {
      ta[a] = lo_a;
      tb[a] = hi_a;
      par[a] = pa;
      int st = 0;
      double de = 0.0;
      if (dd > kTiny) {
        st = 1;
        de = g.voxel_size / dd;
      } else if (dd < -kTiny) {
        st = -1;
        de = -g.voxel_size / dd;
      }
      step[a] = st;
      delta[a] = de;
      if (ok) {
        const double pnt = od + lo * dd;
        const int va = sclamp(static_cast<int>(floor((pnt - gd) / g.voxel_size)), 0, g.dims[a] - 1);
        v[a] = va;
        if (st > 0)
          t_next[a] = ((gd + static_cast<double>(va + 1) * g.voxel_size) - od) / dd;
        else if (st < 0)
          t_next[a] = ((gd + static_cast<double>(va) * g.voxel_size) - od) / dd;
        else
          t_next[a] = __longlong_as_double(0x7ff0000000000000ll);
      }
    }
    if (lane == 0) {
      o = origin;
      d = dir;
      t_end = t1;
      miss = any_out;
      if (ok) t_entry = lo;
      active = ok;
    }
  }

  // Returns the stepped axis, or -1 when the walk ended.
  __device__ __forceinline__ int advance(const GridView& g) {
    if (!active) return -1;
    int axis = 0;
    if (t_next[1] < t_next[axis]) axis = 1;
    if (t_next[2] < t_next[axis]) axis = 2;
    if (t_next[axis] > t_end) {
      active = false;
      return -1;
    }
    t_entry = t_next[axis];
    v[axis] += step[axis];
    if (v[axis] < 0 || v[axis] >= g.dims[axis]) {
      active = false;
      return -1;
    }
    t_next[axis] += delta[axis];
    return axis;
  }
};

// cone_intersects_sphere (tracer.cpp:129-136)
__device__ __forceinline__ bool cone_intersects_sphere(const V3& o, const V3& d, double alpha, const V3& c,
                                                       double r) {
  const V3 vc = c - o;
  const double dist = norm(vc);
  if (dist <= r) return true;
  const double beta = angle_between(vc, d);
  return beta <= alpha + asin(smin(1.0, r / dist));
}

// segment_visible (tracer.cpp:138-205). The result is "no SurfacePoints IE other than
// target_ie blocks the windowed span", an existential over the union of the walked
// voxels' 27-neighbourhoods, so the visiting order is free. The reference dedups
// cells with epoch stamps; here a plain DDA step along axis a only exposes the
// 9-cell far slab of the new neighbourhood (voxel coordinates are monotone along
// the walk), so the first voxel scans 27 cells and every later step 9.
__device__ inline bool segment_visible(const V3& origin, const V3& target, uint32_t target_ie, const GridView& g,
                                       const SceneView& s) {
  const V3 diff = target - origin;
  const double dist = norm(diff);
  if (dist < kTiny) return true;
  const V3 d = diff / dist;
  const double er = g.sub_radius;
  const double span = dist - 2.0 * er;
  if (span <= 1e-9) return true;
  const V3 o2 = origin + er * d;
  const double cell_reach = g.voxel_radius + g.sub_radius;

  Walker w;
  w.init(g, origin, d, 0.0, dist);
  int axis = -1;  // -1: full 27-neighbourhood
  int skip = 0;
  while (w.active) {
    // empty-space skipping (exact): march(v) = m >= 2 means every cell within
    // Chebyshev distance m-1 of v is empty, so N(u) is empty for v and for the next
    // m-2 voxels of the walk (each step moves to an adjacent voxel); the walk itself
    // is unchanged, only the screening of empty neighbourhoods is left out. The next
    // screened voxel's far slab still covers its neighbourhood: the rest of it lies
    // in N(previous voxel), screened or empty.
    if (skip > 0) {
      --skip;
      axis = w.advance(g);
      continue;
    }
    const int m = g.march_ok ? g.cells[linear_index(g, w.v[0], w.v[1], w.v[2])].z : 0;
    if (m >= 2) {
      skip = m - 2;
      axis = w.advance(g);
      continue;
    }
    const int sa = axis;
    const int lo0 = (sa == 0) ? w.step[0] : -1, hi0 = (sa == 0) ? w.step[0] : 1;
    const int lo1 = (sa == 1) ? w.step[1] : -1, hi1 = (sa == 1) ? w.step[1] : 1;
    const int lo2 = (sa == 2) ? w.step[2] : -1, hi2 = (sa == 2) ? w.step[2] : 1;
    for (int oz = lo2; oz <= hi2; ++oz) {
      for (int oy = lo1; oy <= hi1; ++oy) {
        for (int ox = lo0; ox <= hi0; ++ox) {
          const int nx = w.v[0] + ox, ny = w.v[1] + oy, nz = w.v[2] + oz;
          if (!in_bounds(g, nx, ny, nz)) continue;
          const int4 cell = g.cells[linear_index(g, nx, ny, nz)];
          if (cell.x == cell.y) continue;
          const V3 cc = voxel_center(g, nx, ny, nz);
          const double tcc = sclamp(dot(cc - o2, d), 0.0, span);
          if (norm((o2 + tcc * d) - cc) > cell_reach) continue;
          for (uint32_t i = static_cast<uint32_t>(cell.x); i < static_cast<uint32_t>(cell.y); ++i) {
            if ((g.ie_meta[i] & 3u) != kSurface) continue;
            if (i == target_ie) continue;
            const double4 sc4 = g.ie_sc[i];
            const V3 sc = ld3(sc4);
            const double tc = sclamp(dot(sc - o2, d), 0.0, span);
            if (norm((o2 + tc * d) - sc) > sc4.w) continue;
            SurfaceHit hit;
            if (!march_segment(o2, d, i, g, s, span, &hit)) continue;
            if (hit.distance <= 1e-9) continue;
            if (hit.distance >= span - 1e-9) continue;
            return false;
          }
        }
      }
    }
    axis = w.advance(g);
  }
  return true;
}

// Warp-cooperative segment_visible (same arguments in every lane, same result): at
// each walker step the lanes take the new cells (27 at the first voxel, the 9-cell
// far slab afterwards), apply the cell prefilter, and the surviving cells' IEs are
// flattened across lanes in rounds of 32; any blocker ends the walk for the warp.
__device__ inline bool warp_segment_visible(const V3& origin, const V3& target, uint32_t target_ie,
                                            const GridView& g, const SceneView& s) {
  const int lane = threadIdx.x & 31;
  const V3 diff = target - origin;
  const double dist = norm(diff);
  if (dist < kTiny) return true;
  const V3 d = diff / dist;
  const double er = g.sub_radius;
  const double span = dist - 2.0 * er;
  if (span <= 1e-9) return true;
  const V3 o2 = origin + er * d;
  const double cell_reach = g.voxel_radius + g.sub_radius;
  // the walker is warp-uniform: one copy per warp in shared memory, stepped by lane 0
  // between two __syncwarp()s (as in warp_cone_walk); callers run 128-thread blocks.
  // Same box: C3 visibility 11.34 -> 9.74 s, C2 297 -> 264 ms
  // (profiles/ab_segvis_walker_smem_r02.log)
#ifndef PCR_SEGVIS_WALKER_SMEM
#define PCR_SEGVIS_WALKER_SMEM 1
#endif
  __shared__ Walker segvis_walk_s[4];
  Walker w_local;
  if (PCR_SEGVIS_WALKER_SMEM && blockDim.x > 128) __trap();  // one shared walker per warp of a 128-thread block
  Walker& w = PCR_SEGVIS_WALKER_SMEM ? segvis_walk_s[(threadIdx.x >> 5) & 3] : w_local;
  __syncwarp();  // every lane is past the previous call's last read of the shared walker
#ifndef PCR_SEGVIS_WARP_INIT
#define PCR_SEGVIS_WARP_INIT 1
#endif
  if (PCR_SEGVIS_WALKER_SMEM && PCR_SEGVIS_WARP_INIT)
    w.init_warp(g, origin, d, 0.0, dist, lane);
  else if (!PCR_SEGVIS_WALKER_SMEM || lane == 0)
    w.init(g, origin, d, 0.0, dist);
  __syncwarp();
  auto advance = [&]() {
    if (!PCR_SEGVIS_WALKER_SMEM) return w.advance(g);
    int a = 0;
    if (lane == 0) a = w.advance(g);
    a = __shfl_sync(0xffffffffu, a, 0);
    __syncwarp();
    return a;
  };
  int axis = -1;
  int skip = 0;
  while (w.active) {
    // empty-space skipping, as in segment_visible (warp-uniform)
    if (skip > 0) {
      --skip;
      __syncwarp();
      axis = advance();
      continue;
    }
    const int m = g.march_ok ? g.cells[linear_index(g, w.v[0], w.v[1], w.v[2])].z : 0;
    if (m >= 2) {
      skip = m - 2;
      __syncwarp();
      axis = advance();
      continue;
    }
    // this lane's cell offset: the 27-neighbourhood, or the far slab across the stepped
    // axis (selects instead of an array indexed by the axis, which lived in local memory)
    int ox_, oy_, oz_;
    bool mine;
    if (axis < 0) {
      mine = lane < 27;
      ox_ = lane % 3 - 1;
      oy_ = (lane / 3) % 3 - 1;
      oz_ = lane / 9 - 1;
    } else {
      mine = lane < 9;
      const int u = lane % 3 - 1, v = (lane / 3) % 3 - 1;
      const int st = w.step[axis];
      ox_ = axis == 0 ? st : axis == 1 ? v : u;
      oy_ = axis == 1 ? st : axis == 2 ? v : u;
      oz_ = axis == 2 ? st : axis == 0 ? v : u;
    }
    const int nx = w.v[0] + ox_, ny = w.v[1] + oy_, nz = w.v[2] + oz_;
    int b = 0, cnt = 0;
    if (mine && in_bounds(g, nx, ny, nz)) {
      const int4 cell = g.cells[linear_index(g, nx, ny, nz)];
      if (cell.x != cell.y) {
        const V3 cc = voxel_center(g, nx, ny, nz);
        const double tcc = sclamp(dot(cc - o2, d), 0.0, span);
        if (!(norm((o2 + tcc * d) - cc) > cell_reach)) {
          b = cell.x;
          cnt = cell.y - cell.x;
        }
      }
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    for (int base = 0; base < total; base += 32) {
      const int f = base + lane;
      int jlo = 0, jhi = 31;
#pragma unroll
      for (int st = 0; st < 5; ++st) {
        const int mid = (jlo + jhi) >> 1;
        const int vv = __shfl_sync(0xffffffffu, incl, mid);
        if (vv > f) jhi = mid;
        else jlo = mid + 1;
      }
      const int cb = __shfl_sync(0xffffffffu, b, jlo);
      const int ce = __shfl_sync(0xffffffffu, incl - cnt, jlo);
      bool blocked = false;
      if (f < total) {
        const uint32_t i = static_cast<uint32_t>(cb + (f - ce));
        if ((g.ie_meta[i] & 3u) == kSurface && i != target_ie) {
          const double4 sc4 = g.ie_sc[i];
          const V3 sc = ld3(sc4);
          const double tc = sclamp(dot(sc - o2, d), 0.0, span);
          if (!(norm((o2 + tc * d) - sc) > sc4.w)) {
            SurfaceHit hit;
            if (march_segment(o2, d, i, g, s, span, &hit) && !(hit.distance <= 1e-9) &&
                !(hit.distance >= span - 1e-9))
              blocked = true;
          }
        }
      }
      if (__any_sync(0xffffffffu, blocked)) return false;
    }
    __syncwarp();
      axis = advance();
  }
  return true;
}

}  // namespace pcr
