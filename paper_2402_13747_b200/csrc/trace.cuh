// trace.cuh — stage-2 device records and the cone walk shared by the kernels.
#pragma once

#include "geom.cuh"

namespace pcr {

constexpr uint32_t kNoNode = 0xffffffffu;
constexpr int kMaxDepth = 8;  // max_interactions supported by the DFS keys

// One interaction of a DFS path (tracer.hpp:31-38 Interaction) plus the links
// the wavefront needs: the parent interaction, the Keller-fan index of the
// parent ray that produced this reception, and the number of child rays.
struct Node {
  double pos[3];
  double nrm[3];  // reflection: surface normal at the hit; diffraction: edge normal_a
  double inc[3];  // incoming direction at this interaction
  uint32_t parent;
  uint32_t parent_j;
  uint32_t ie, label, edge;
  uint32_t task;  // index of the initial hit this path descends from
  uint32_t n_children;
  uint8_t kind, depth, dc, pad;
};

// A materialised conical ray (tracer.hpp:40-47). Separation planes all pass
// through the ray origin (tracer.cpp:265, 306-307), so only normals are kept.
struct Ray {
  V3 o, d;
  double apex;
  V3 pn[2];
  uint32_t node, j;
  uint32_t origin_ie, origin_label;
  uint8_t n_planes, depth, dc, alive;
};

struct Cand {
  uint32_t node, j, rx_ie, pad;
};

// Visibility work item: ray r may receive IE i.
struct Task {
  uint32_t ray, ie;
};

// passes_separation_planes (tracer.cpp:99-104)
__device__ __forceinline__ bool passes_planes(const Ray& r, const V3& q) {
  for (int k = 0; k < r.n_planes; ++k)
    if (dot(q - r.o, r.pn[k]) < 0.0) return false;
  return true;
}

// voxel_cone_trace walk (tracer.cpp:313-398). on_eval(cell) sees every newly
// evaluated in-bounds cell (TraceDebug::evaluated); on_ie(i) every IE that passes
// the self-exclusion, cone, plane and coincidence tests and so reaches
// segment_visible. The `evaluated` byte array (tracer.cpp:329) is replaced by an
// exact ring of the last evaluating voxels: voxel coordinates are monotone along
// the walk (DDA steps and forward re-inits), so a cell of N(v) was evaluated iff
// it lies in N(u) for an earlier evaluating voxel u within Chebyshev distance 2
// of v, and those u are a suffix of at most 6 voxels.
template <typename OnEval, typename OnIE>
__device__ __forceinline__ void cone_walk(const GridView& g, const Ray& r, OnEval on_eval, OnIE on_ie,
                                          uint32_t* n_cells = nullptr, uint32_t* n_ies = nullptr) {
  if (g.n_ies == 0) return;
  uint32_t cells_seen = 0, ies_seen = 0;
  const double half_angle = 0.5 * r.apex;
  const double exempt_radius = 2.0 * g.sub_radius;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  int ring[8][3];
  int ring_n = 0;
  Walker w;
  w.init(g, r.o, r.d, 0.0, inf);
  while (w.active) {
    const int4 here = g.cells[linear_index(g, w.v[0], w.v[1], w.v[2])];
    const int march = here.z;
    if (here.x != here.y || march <= 1) {
      for (int oz = -1; oz <= 1; ++oz) {
        for (int oy = -1; oy <= 1; ++oy) {
          for (int ox = -1; ox <= 1; ++ox) {
            const int nx = w.v[0] + ox, ny = w.v[1] + oy, nz = w.v[2] + oz;
            if (!in_bounds(g, nx, ny, nz)) continue;
            bool seen = false;
            for (int k = 0; k < ring_n; ++k) {
              if (abs(nx - ring[k][0]) <= 1 && abs(ny - ring[k][1]) <= 1 && abs(nz - ring[k][2]) <= 1) {
                seen = true;
                break;
              }
            }
            if (seen) continue;
            const uint32_t ni = linear_index(g, nx, ny, nz);
            on_eval(ni);
            ++cells_seen;
            const int4 cell = g.cells[ni];
            if (cell.x == cell.y) continue;
            if (!cone_intersects_sphere(r.o, r.d, half_angle, voxel_center(g, nx, ny, nz), g.voxel_radius)) continue;
            ies_seen += static_cast<uint32_t>(cell.y - cell.x);
            for (uint32_t i = static_cast<uint32_t>(cell.x); i < static_cast<uint32_t>(cell.y); ++i) {
              if (i == r.origin_ie) continue;
              const double4 sc4 = g.ie_sc[i];
              const V3 sc = ld3(sc4);
              if (r.origin_ie != kNoIe && g.ie_label[i] == r.origin_label && norm(sc - r.o) <= exempt_radius)
                continue;
              if (!cone_intersects_sphere(r.o, r.d, half_angle, sc, sc4.w)) continue;
              const V3 rp = ld3(g.ie_rp[i]);
              if (!passes_planes(r, rp)) continue;
              if (norm(rp - r.o) < kTiny) continue;
              on_ie(i);
            }
          }
        }
      }
      // keep only earlier evaluating voxels still within Chebyshev distance 2
      int m = 0;
      for (int k = 0; k < ring_n; ++k) {
        if (abs(w.v[0] - ring[k][0]) <= 2 && abs(w.v[1] - ring[k][1]) <= 2 && abs(w.v[2] - ring[k][2]) <= 2) {
          ring[m][0] = ring[k][0];
          ring[m][1] = ring[k][1];
          ring[m][2] = ring[k][2];
          ++m;
        }
      }
      if (m == 8) {  // cannot happen (<= 6 by monotonicity); keep the newest 7
        for (int k = 0; k < 7; ++k) {
          ring[k][0] = ring[k + 1][0];
          ring[k][1] = ring[k + 1][1];
          ring[k][2] = ring[k + 1][2];
        }
        m = 7;
      }
      ring[m][0] = w.v[0];
      ring[m][1] = w.v[1];
      ring[m][2] = w.v[2];
      ring_n = m + 1;
    }
    if (march >= 2) {
      w.init_at(g, w.t_entry + static_cast<double>(march - 1) * g.voxel_size, inf);
    } else {
      w.advance(g);
    }
  }
  if (n_cells) *n_cells += cells_seen;
  if (n_ies) *n_ies += ies_seen;
}

// Knife-edge libm decisions. The reference decides `atan2(..) <= alpha +
// asin(..)` (tracer.cpp:129-136, geometry.hpp:33-37) and `angle_between(na, nb) <=
// 1e-9` (tracer.cpp:275-284) with glibc; the device evaluates the same expressions
// with CUDA's libm. Both libms are within a few ulp of the exact values (glibc < 1 ulp,
// CUDA atan2/asin <= 2 ulp), so whenever the two sides differ by more than `ulps`
// units in the last place of the larger one the decision is the reference's; a
// comparison inside that margin is counted here (read per propagate call into
// TraceStats::libm_unresolved, reported in the RunSummary counters, asserted zero by
// the contract tests) — a run with a zero count is bit-exact in every such decision.
static __device__ unsigned long long g_libm_unresolved = 0;
__device__ __forceinline__ double ulp_of(double x) {
  const long long e = __double_as_longlong(fabs(x)) & 0x7ff0000000000000ll;
  return e ? __longlong_as_double(e) * 2.220446049250313e-16 : 4.9406564584124654e-324;
}
__device__ __forceinline__ bool libm_le(double a, double b, double ulps) {
  const double m = fabs(a - b);
  const double sc = fabs(a) < fabs(b) ? fabs(b) : fabs(a);
  if (!(m > ulps * ulp_of(sc))) atomicAdd(&g_libm_unresolved, 1ull);
  return a <= b;
}

// cone_intersects_sphere (tracer.cpp:129-136) with an exact-equivalent fast path.
// beta = atan2(|vc x d|, vc.d) <= rhs = alpha + asin(min(1, r/dist)) is, on [0, pi],
// cos(beta) >= cos(rhs) with cos(beta) = vc.d / (|vc||d|) and
// cos(rhs) = cos(alpha) sqrt((1-s)(1+s)) - sin(alpha) s. Both sides are evaluated to
// ~1e-15; libm's atan2/asin are within a few ulp; so whenever the cosines differ by
// more than 1e-9 the reference's comparison has the same outcome, and only the rare
// knife edge inside that band pays for the transcendental evaluation. alpha < 1 rad
// keeps rhs < pi (the reference's default half-angle is 0.5 deg).
struct ConeConsts {
  double alpha, ca, sa, dnorm;
  bool fast;
};
__device__ __forceinline__ ConeConsts cone_consts(double alpha, const V3& d) {
  ConeConsts k;
  k.alpha = alpha;
  k.ca = cos(alpha);
  k.sa = sin(alpha);
  k.dnorm = norm(d);
  k.fast = alpha >= 0.0 && alpha < 1.0 && k.dnorm > 0.0;
  return k;
}
#ifndef PCR_CONE_NODIV
#define PCR_CONE_NODIV 1
#endif
__device__ __forceinline__ bool cone_test(const V3& o, const V3& d, const ConeConsts& k, const V3& c, double r) {
  const V3 vc = c - o;
  if (PCR_CONE_NODIV) {
    // The same decision with one square root and no division in the common case.
    // dist <= r is norm_le (the squared norm outside its rounding band, sqrt inside).
    // Multiplying cb >= cr by dist |d| > 0: P = vc.d against
    // Q = |d| (cos(alpha) sqrt(dist^2 - r^2) - sin(alpha) r). P and Q carry ~1e-15
    // dist |d| of rounding, so |P - Q| > T = 1e-9 |d| |vc|_1 (>= 1e-9 |d| dist) means
    // |cb - cr| > 1e-9 in exact arithmetic, the fast path's certified margin above.
    // dist^2 - r^2 is used only when it is >= 1e-6 dist^2 (its rounding then stays
    // below 1e-10 relative, so the square root is well conditioned); grazing spheres
    // and everything inside the margin take the reference's expression below.
    if (norm_le(vc, r)) return true;
    const double d2 = sqnorm(vc), q2 = d2 - r * r;
    if (k.fast && q2 >= 1e-6 * d2) {
      const double P = dot(vc, d);
      const double Q = k.dnorm * (k.ca * sqrt(q2) - k.sa * r);
      const double T = 1e-9 * k.dnorm * ((fabs(vc.x) + fabs(vc.y)) + fabs(vc.z));
      if (P - Q > T) return true;
      if (P - Q < -T) return false;
    }
    const double beta = angle_between(vc, d);
    return libm_le(beta, k.alpha + asin(smin(1.0, r / norm(vc))), 8.0);
  }
  const double dist = norm(vc);
  if (dist <= r) return true;
  if (k.fast) {
    const double s = smin(1.0, r / dist);
    const double cb = dot(vc, d) / (dist * k.dnorm);
    const double cr = k.ca * sqrt((1.0 - s) * (1.0 + s)) - k.sa * s;
    const double diff = cb - cr;
    if (diff > 1e-9) return true;
    if (diff < -1e-9) return false;
  }
  // the band: the reference's expression; atan2 and asin each within 3 ulp of glibc's
  // and one rounding of the sum -> 8 ulp of [0, pi] values certify the outcome
  const double beta = angle_between(vc, d);
  return libm_le(beta, k.alpha + asin(smin(1.0, r / dist)), 8.0);
}

// Warp-cooperative voxel_cone_trace walk: the 32 lanes hold the same ray, walker
// and dedup ring (warp-uniform control flow); at an evaluating voxel lane l < 27
// takes neighbour l (z -> y -> x order as in tracer.cpp:339-341), and the IEs of
// the cells that pass the voxel cone test are flattened across lanes in rounds of
// 32. on_ie(i, pass) is called by every lane each round (pass = the IE survived the
// self-exclusion / cone / plane / coincidence tests), so it may use warp
// collectives. Same evaluated set and same surviving IEs as cone_walk.
template <typename OnEval, typename OnIE>
__device__ __forceinline__ void warp_cone_walk(const GridView& g, const Ray& r, OnEval on_eval, OnIE on_ie,
                                               uint32_t* n_cells = nullptr, uint32_t* n_ies = nullptr) {
  if (g.n_ies == 0) return;
  const int lane = threadIdx.x & 31;
  const double half_angle = 0.5 * r.apex;
  const double exempt_radius = 2.0 * g.sub_radius;
  const ConeConsts kc = cone_consts(half_angle, r.d);
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const int ox = lane % 3 - 1, oy = (lane / 3) % 3 - 1, oz = lane / 9 - 1;
  // the dedup ring is warp-uniform: one copy per warp in shared memory (broadcast reads)
  // instead of an identical local-memory array in every lane (ncu, C2: the per-lane
  // ring's loops were 24 % of the walk kernel's stall samples). Same box: C2 cone walk
  // 981 -> 838 ms, C3 6.86 -> 6.13 s (profiles/ab_ring_smem_r02.log)
#ifndef PCR_RING_SMEM
#define PCR_RING_SMEM 1
#endif
  __shared__ int4 ring_s[4][8];  // walk_kernel: 128 threads = 4 warps per block
  int4* rs = ring_s[(threadIdx.x >> 5) & 3];
  int ring[8][3];
  int ring_n = 0;
  uint32_t cells_seen = 0, ies_seen = 0;
  // the walker is warp-uniform too: one copy per warp in shared memory, stepped by
  // lane 0 between two __syncwarp()s, read by every lane (C2 cone walk 845 -> 747 ms,
  // C3 6.17 -> 5.81 s same box, profiles/ab_walker_smem_r02.log)
#ifndef PCR_WALKER_SMEM
#define PCR_WALKER_SMEM 1
#endif
  __shared__ Walker walk_s[4];
  Walker w_local;
  if ((PCR_WALKER_SMEM || PCR_RING_SMEM) && blockDim.x > 128) __trap();  // per-warp shared state of a 128-thread block
  Walker& w = PCR_WALKER_SMEM ? walk_s[(threadIdx.x >> 5) & 3] : w_local;
  __syncwarp();  // every lane is past the previous walk's last read of the shared walker
  if (!PCR_WALKER_SMEM || lane == 0) w.init(g, r.o, r.d, 0.0, inf);
  __syncwarp();
  while (w.active) {
    const int4 here = g.cells[linear_index(g, w.v[0], w.v[1], w.v[2])];
    const int march = here.z;
    if (here.x != here.y || march <= 1) {
      const int nx = w.v[0] + ox, ny = w.v[1] + oy, nz = w.v[2] + oz;
      bool valid = lane < 27 && in_bounds(g, nx, ny, nz);
      if (PCR_RING_SMEM) {
        for (int k = 0; k < ring_n && valid; ++k) {
          const int4 e = rs[k];
          if (abs(nx - e.x) <= 1 && abs(ny - e.y) <= 1 && abs(nz - e.z) <= 1) valid = false;
        }
      } else {
        for (int k = 0; k < ring_n && valid; ++k)
          if (abs(nx - ring[k][0]) <= 1 && abs(ny - ring[k][1]) <= 1 && abs(nz - ring[k][2]) <= 1) valid = false;
      }
      int b = 0, cnt = 0;
      if (valid) {
        const uint32_t ni = linear_index(g, nx, ny, nz);
        on_eval(ni);
        const int4 cell = g.cells[ni];
        if (cell.x != cell.y && cone_test(r.o, r.d, kc, voxel_center(g, nx, ny, nz), g.voxel_radius)) {
          b = cell.x;
          cnt = cell.y - cell.x;
        }
      }
      cells_seen += __popc(__ballot_sync(0xffffffffu, valid));
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      ies_seen += static_cast<uint32_t>(total);
      for (int base = 0; base < total; base += 32) {
        const int f = base + lane;
        int jlo = 0, jhi = 31;  // owning lane: first j with incl_j > f
#pragma unroll
        for (int s = 0; s < 5; ++s) {
          const int mid = (jlo + jhi) >> 1;
          const int v = __shfl_sync(0xffffffffu, incl, mid);
          if (v > f) jhi = mid;
          else jlo = mid + 1;
        }
        const int cb = __shfl_sync(0xffffffffu, b, jlo);
        const int ce = __shfl_sync(0xffffffffu, incl - cnt, jlo);
        bool pass = false;
        uint32_t i = 0;
        if (f < total) {
          i = static_cast<uint32_t>(cb + (f - ce));
          pass = i != r.origin_ie;
          if (pass) {
            const double4 sc4 = g.ie_sc[i];
            const V3 sc = ld3(sc4);
            if (r.origin_ie != kNoIe && g.ie_label[i] == r.origin_label && norm(sc - r.o) <= exempt_radius)
              pass = false;
            else if (!cone_test(r.o, r.d, kc, sc, sc4.w))
              pass = false;
            else {
              const V3 rp = ld3(g.ie_rp[i]);
              if (!passes_planes(r, rp) || norm(rp - r.o) < kTiny) pass = false;
            }
          }
        }
        on_ie(i, pass);
      }
      // dedup ring: keep earlier evaluating voxels within Chebyshev distance 2
      if (PCR_RING_SMEM) {
        // lane k < ring_n tests entry k; kept entries move to their rank among the kept
        // ones (dropping the oldest when all 8 stay), then the current voxel is appended
        const int4 e = lane < ring_n ? rs[lane] : make_int4(0, 0, 0, 0);
        const bool keep = lane < ring_n && abs(w.v[0] - e.x) <= 2 && abs(w.v[1] - e.y) <= 2 &&
                          abs(w.v[2] - e.z) <= 2;
        const uint32_t km = __ballot_sync(0xffffffffu, keep);
        const int m = __popc(km);
        const int drop = m == 8 ? 1 : 0;
        const int at = __popc(km & ((1u << lane) - 1u)) - drop;
        __syncwarp();
        if (keep && at >= 0) rs[at] = e;
        if (lane == 0) rs[m - drop] = make_int4(w.v[0], w.v[1], w.v[2], 0);
        ring_n = m - drop + 1;
        __syncwarp();
      } else {
      int m = 0;
      for (int k = 0; k < ring_n; ++k) {
        if (abs(w.v[0] - ring[k][0]) <= 2 && abs(w.v[1] - ring[k][1]) <= 2 && abs(w.v[2] - ring[k][2]) <= 2) {
          ring[m][0] = ring[k][0];
          ring[m][1] = ring[k][1];
          ring[m][2] = ring[k][2];
          ++m;
        }
      }
      if (m == 8) {
        for (int k = 0; k < 7; ++k) {
          ring[k][0] = ring[k + 1][0];
          ring[k][1] = ring[k + 1][1];
          ring[k][2] = ring[k + 1][2];
        }
        m = 7;
      }
      ring[m][0] = w.v[0];
      ring[m][1] = w.v[1];
      ring[m][2] = w.v[2];
      ring_n = m + 1;
      }
    }
    __syncwarp();
    if (!PCR_WALKER_SMEM || lane == 0) {
      if (march >= 2) {
        w.init_at(g, w.t_entry + static_cast<double>(march - 1) * g.voxel_size, inf);
      } else {
        w.advance(g);
      }
    }
    __syncwarp();
  }
  if (n_cells) *n_cells += cells_seen;
  if (n_ies) *n_ies += ies_seen;
}

// Warp-aggregated 64-bit counter add.
__device__ __forceinline__ void warp_add_u64(unsigned long long* dst, unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

// Keller-fan sin/cos table (host libm, trace.cu ensure_fan): per j cos phi, sin phi,
// sin/cos(phi + dphi/2), sin/cos(phi - dphi/2)
struct FanTable {
  const double* t;  // n*6
  int n;
};

// diffract_rays degeneracy tests (tracer.cpp:275-284); returns false for "no rays".
__device__ __forceinline__ bool fan_frame(const double* edge, const V3& incoming, V3& w, V3& e1, V3& e2,
                                          double& cos_b, double& sin_b, V3& na, V3& nb) {
  const V3 s = load3(edge), e = load3(edge + 3);
  na = load3(edge + 6);
  nb = load3(edge + 9);
  w = normalized(e - s);
  cos_b = dot(incoming, w);
  if (fabs(cos_b) > 0.999) return false;
  if (libm_le(angle_between(na, nb), 1e-9, 4.0)) return false;  // atan2: see libm_le
  if (dot(incoming, na) >= 0.0 && dot(incoming, nb) >= 0.0) return false;
  e1 = safe_normalized(incoming - cos_b * w);
  if (is_zero(e1)) return false;
  e2 = cross(w, e1);
  sin_b = sqrt(smax(0.0, 1.0 - cos_b * cos_b));
  return true;
}


}  // namespace pcr
