// refine.cu — stage 3: refine_path (proj/src/refine.cpp:189-286) on the device,
// one thread per coarse path, FP64 in the reference's operation order.
//
// Per iteration: local_gradients (:167-187), backtracking with up to 9 trial steps
// (:209-232), front-to-back reprojection of reflection nodes (:234-250) through
// surface_ies_near (:34-52) + march_segment / project_to_surface + polish (:62-130).
// Shortcut (bit-exact): when no trial step is accepted the state is unchanged, so
// every remaining iteration repeats the same computation and the outcome is
// not_converged; the kernel stops there instead of spinning to rho.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "host_alloc.hpp"
#include "pipeline.hpp"
#include "sort.cuh"
#include "stages.cuh"
#include "trace.cuh"

namespace pcr {

constexpr double kSpeedOfLight = 299792458.0;

namespace {

struct RNode {
  V3 c, a, b, n;  // reflection: c, u, v, normal; diffraction: c, w, -, -
  double p0, p1;  // reflection: r, s; diffraction: t, -
  double lo, hi;  // diffraction t range
  uint32_t label, edge;
  uint8_t kind;
};

__device__ __forceinline__ V3 node_point(const RNode& nd, double p0, double p1) {
  return nd.kind == 0 ? (nd.c + p0 * nd.a) + p1 * nd.b : nd.c + p0 * nd.a;
}

__device__ __forceinline__ double chain_len(const V3& tx, const V3* pts, int n, const V3& rx) {
  V3 prev = tx;
  double len = 0.0;
  for (int k = 0; k < n; ++k) {
    len += norm(pts[k] - prev);
    prev = pts[k];
  }
  return len + norm(rx - prev);
}

struct Reproj {
  V3 pos, nrm;
  uint32_t label;
};

// polish (refine.cpp:62-75)
__device__ void polish(Reproj& re, uint32_t ie, const GridView& g, const SceneView& s) {
  if (ie_planar(g, ie)) {
    const V3 pp = ld3(g.ie_pp[ie]), pn = ld3(g.ie_pn[ie]);
    re.pos = re.pos - dot(re.pos - pp, pn) * pn;
    re.nrm = pn;
    return;
  }
  for (int i = 0; i < 4; ++i) {
    const SurfaceEstimate est = estimate_surface(re.pos, ie, g, s);
    re.pos = re.pos - est.sdf * est.n_bar;
    re.nrm = est.n_bar;
    if (fabs(est.sdf) <= 1e-12) break;
  }
}

__device__ __forceinline__ int voxel_floor(double p, double o, double vs) {
  return static_cast<int>(floor((p - o) / vs));
}

// Planar march_segment (surface.cpp:74-106) of one reprojection candidate, reordered:
// a hit's distance is the snap t* when t* falls in the window, so such a window
// cannot win once t* >= best_t and the two endpoint tests are skipped. Coplanar IEs
// (same normal and plane-offset bits, e.g. the IEs of one wall) share t*: the
// division is done once per plane (cache c_num, c_dn -> c_t). Returns true and
// lowers best_t when this IE's hit is strictly nearer.
//
// Fast rejection (exact; off by default, PCR_FAST_REJECT=1 enables it: same-box A/B on
// C2 depth 3, refine 554-565 ms without vs 566-574 ms with — the kernel is latency-bound
// and the extra branch costs more than the skipped endpoint tests): the sdf along the ray is f(t) = dot((o + t d) - pp, n), and
// in exact arithmetic f(t) = dn (t - t_e) with t_e the plane crossing. The computed
// f(t) and the computed dn (t - t*) differ by at most ~30 u (|o| + |pp| + |t|)
// (u = 2^-53: the dot products' rounding, num and dn's rounding, the division), which
// kMarginFast bounds whenever the scene's coordinates are below ~10^5 m (refine_device
// sets fast_reject from the grid's extent). So when t* lies outside the window by more
// than (eps + kMarginFast) / |dn|, both endpoint values have |f| > eps and the same
// sign: the reference's march returns no hit, decided without evaluating them.
constexpr double kMarginFast = 1e-9;
__device__ __forceinline__ bool planar_candidate_at(const V3& prev, const V3& dir, const V3& pp, const V3& pn,
                                                    double eps, double t_lo, double t_hi, double& best_t,
                                                    long long& c_num, long long& c_dn, double& c_t,
                                                    bool fast = false) {
  if (t_hi <= t_lo) return false;
  const double dn = dot(dir, pn);
  const bool snap = fabs(dn) > 1e-12;
  double t_star = 0.0;
  if (snap) {
    const double num = dot(pp - prev, pn);
    const long long nbits = __double_as_longlong(num), dbits = __double_as_longlong(dn);
    if (nbits != c_num || dbits != c_dn) {
      c_num = nbits;
      c_dn = dbits;
      c_t = num / dn;
    }
    t_star = c_t;
  }
  const bool in_win = snap && t_star >= t_lo && t_star <= t_hi;
  if (in_win && t_star >= best_t) return false;
  if (fast && snap && !in_win) {
    const double gap = t_star < t_lo ? t_lo - t_star : t_star - t_hi;
    if (fabs(dn) * gap > eps + kMarginFast) return false;
  }
  double tc;
  const double f = dot((prev + t_lo * dir) - pp, pn);
  if (fabs(f) <= eps) {
    tc = t_lo;
  } else {
    const double f_hi = dot((prev + t_hi * dir) - pp, pn);
    if (f * f_hi < 0.0)
      tc = 0.5 * (t_lo + t_hi);
    else if (fabs(f_hi) <= eps)
      tc = t_hi;
    else
      return false;
  }
  const double t = in_win ? t_star : tc;
  if (t >= best_t) return false;
  best_t = t;
  return true;
}
__device__ __forceinline__ bool planar_candidate(const V3& prev, const V3& dir, uint32_t ie, const GridView& g,
                                                 double t_lo, double t_hi, double& best_t, long long& c_num,
                                                 long long& c_dn, double& c_t) {
  if (t_hi <= t_lo) return false;
  return planar_candidate_at(prev, dir, ld3(g.ie_pp[ie]), ld3(g.ie_pn[ie]), g.hit_eps, t_lo, t_hi, best_t, c_num,
                             c_dn, c_t);
}

// reproject (refine.cpp:80-130) with surface_ies_near (:34-52) scanned in place.
// first_pass = 1 skips the same-label pass (done cooperatively by refine_warp_kernel).
__device__ __noinline__ bool reproject(const V3& prev, const V3& predicted, uint32_t label, const GridView& g, const SceneView& s,
                          Reproj& out, uint32_t& n_march, int first_pass = 0) {
  const V3 diff = predicted - prev;
  const double dist = norm(diff);
  if (dist < kTiny) return false;
  const V3 dir = diff / dist;
  const double radius = 2.0 * g.sub_edge;
  const double pc[3] = {predicted.x, predicted.y, predicted.z};
  const double oc[3] = {g.origin.x, g.origin.y, g.origin.z};
  int lo[3], hi[3];
  bool nb = g.nb_off != nullptr;
  int cc[3];
  for (int a = 0; a < 3; ++a) {
    const int l = voxel_floor(pc[a] - radius, oc[a], g.voxel_size);
    const int h = voxel_floor(pc[a] + radius, oc[a], g.voxel_size);
    lo[a] = smin(smax(l, 0), g.dims[a] - 1);
    hi[a] = smin(smax(h, 0), g.dims[a] - 1);
    // the clamped box is the neighbourhood list of cell l + 1 when it spans l..l+2
    cc[a] = l + 1;
    nb = nb && h == l + 2 && cc[a] >= 0 && cc[a] < g.dims[a];
  }
  uint32_t nb_begin = 0, nb_end = 0;
  if (nb) {
    const uint32_t c = linear_index(g, cc[0], cc[1], cc[2]);
    nb_begin = g.nb_off[c];
    nb_end = g.nb_off[c + 1];
  }
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  for (int pass = first_pass; pass < 2; ++pass) {
    const bool same = pass == 0;
    uint32_t best_ie = kNoIe;
    double best_t = 1.7976931348623157e308;
    Reproj best;  // only for a non-planar winner; planar winners are rebuilt below
    long long c_num = 0x7ff8dead7ff8deadll, c_dn = 0x7ff8dead7ff8deadll;  // (num, dn) bits of the cached t*
    double c_t = 0.0;
    // one flat loop over (cell z→y→x, IE in cell order): lanes of a warp stay in the
    // same loop body whatever their cells' occupancy
    if (nb && same) {
      // the box is the 3x3x3 neighbourhood of the predicted point's cell: one list of
      // its surface-IE records, stably sorted by label, so the same-label candidates
      // are one contiguous run still in scan order (ties keep the reference's winner)
      uint32_t j = nb_begin;
      while (j < nb_end && g.nb_lab[j] < label) ++j;
      for (; j < nb_end && g.nb_lab[j] == label; ++j) {
        const double4 r4 = g.nb_rec[j];
        const uint64_t w = static_cast<uint64_t>(__double_as_longlong(r4.w));
        const uint32_t ie = static_cast<uint32_t>(w >> 33);
        const V3 sc = ld3(r4);
        const double rad = g.rr_uniform ? g.rr_radius : g.ie_sc[ie].w;
        if (!norm_le(sc - predicted, radius + rad)) continue;
        ++n_march;  // counts the reference's march_segment call
        const double t_center = dot(sc - prev, dir);
        const double t_lo = smax(0.0, t_center - rad);
        if (t_lo >= best_t) continue;
        if ((w >> 32) & 1u) {
          if (!planar_candidate(prev, dir, ie, g, t_lo, t_center + rad, best_t, c_num, c_dn, c_t)) continue;
          best_ie = ie;
        } else {
          SurfaceHit hit;
          if (!march_segment(prev, dir, ie, g, s, inf, &hit)) continue;
          if (hit.distance >= best_t) continue;
          best_t = hit.distance;
          best = Reproj{hit.position, hit.normal, g.ie_label[ie]};
          best_ie = ie;
        }
      }
    } else {
    int x = lo[0], y = lo[1], z = lo[2];
    int4 cell = g.cells[linear_index(g, x, y, z)];
    uint32_t i = static_cast<uint32_t>(cell.x);
    for (;;) {
      if (i >= static_cast<uint32_t>(cell.y)) {
        if (++x > hi[0]) {
          x = lo[0];
          if (++y > hi[1]) {
            y = lo[1];
            if (++z > hi[2]) break;
          }
        }
        cell = g.cells[linear_index(g, x, y, z)];
        i = static_cast<uint32_t>(cell.x);
        continue;
      }
      const uint32_t ie = i++;
      // one 32-byte record answers the three filters (pure predicates, cheapest first)
      const double4 r4 = g.ie_rr[ie];
      const uint64_t lm = static_cast<uint64_t>(__double_as_longlong(r4.w));
      if (same != (static_cast<uint32_t>(lm) == label)) continue;
      if (((lm >> 32) & 3u) != kSurface) continue;
      const V3 sc = ld3(r4);
      const double rad = g.rr_uniform ? g.rr_radius : g.ie_sc[ie].w;
      if (!norm_le(sc - predicted, radius + rad)) continue;
      ++n_march;  // counts the reference's march_segment call
      // march_segment's window (surface.cpp:64-72): every hit it returns lies at
      // t >= t_lo, so a window starting at or past the best t cannot win (strict <)
      const double t_center = dot(sc - prev, dir);
      const double t_lo = smax(0.0, t_center - rad);
      if (t_lo >= best_t) continue;
      if ((lm >> 34) & 1u) {
        if (!planar_candidate(prev, dir, ie, g, t_lo, t_center + rad, best_t, c_num, c_dn, c_t)) continue;
        best_ie = ie;
      } else {
        SurfaceHit hit;
        if (!march_segment(prev, dir, ie, g, s, inf, &hit)) continue;
        if (hit.distance >= best_t) continue;
        best_t = hit.distance;
        best = Reproj{hit.position, hit.normal, g.ie_label[ie]};
        best_ie = ie;
      }
    }
    }
    if (best_ie != kNoIe) {
      if (ie_planar(g, best_ie))  // make_hit's record (surface.cpp:98-106)
        best = Reproj{prev + best_t * dir, ld3(g.ie_pn[best_ie]), g.ie_label[best_ie]};
      polish(best, best_ie, g, s);
      out = best;
      return true;
    }
  }
  for (int pass = 0; pass < 2; ++pass) {
    const bool same = pass == 0;
    bool found = false;
    uint32_t best_ie = 0;
    double best_d = 1.7976931348623157e308;
    Reproj best;
    for (int z = lo[2]; z <= hi[2]; ++z)
      for (int y = lo[1]; y <= hi[1]; ++y)
        for (int x = lo[0]; x <= hi[0]; ++x) {
          const int4 cell = g.cells[linear_index(g, x, y, z)];
          for (uint32_t i = static_cast<uint32_t>(cell.x); i < static_cast<uint32_t>(cell.y); ++i) {
            if ((g.ie_meta[i] & 3u) != kSurface) continue;
            const double4 sc4 = g.ie_sc[i];
            const V3 sc = ld3(sc4);
            if (!(norm(sc - predicted) <= radius + sc4.w)) continue;
            if (same != (g.ie_label[i] == label)) continue;
            const double d = norm(sc - predicted);
            if (d >= best_d) continue;
            SurfaceHit hit;
            ++n_march;
            if (!project_to_surface(predicted, i, g, s, &hit)) continue;
            best_d = d;
            best = Reproj{hit.position, hit.normal, g.ie_label[i]};
            best_ie = i;
            found = true;
          }
        }
    if (found) {
      polish(best, best_ie, g, s);
      out = best;
      return true;
    }
  }
  return false;
}

struct CandIn {
  uint32_t first, step;  // candidate subset first + i * step
  uint32_t stride;
  const double* tx;
  const double* rx;
  const uint32_t* n_inter;
  const uint8_t* kind;
  const double* pos;
  const uint32_t* label;
  const double* nrm;
  const uint32_t* edge;
  const double* coarse_length;
  const uint32_t* order;  // optional: the warp kernel's visiting order of the subset (nullptr: 0..n-1)
};

struct RefOut {
  int32_t* reason;
  uint8_t* has_path;
  double* pos;
  double* nrm;
  uint32_t* label;
  double* length;
  double* delay;
  double* gnorm;
  uint32_t* iters;
  unsigned long long* stats;  // [0] trials, [1] reprojection marches, [2] trial nodes, [3] iteration nodes
};

// Dynamic state of a path between iterations: reflection nodes are (c, normal,
// label) with r = s = 0 and (u, v) = local_frame(normal); diffraction nodes are t.
// The iteration is a pure function of it, so a bitwise repeat means the trajectory
// is periodic and can never reach ||g|| < delta (every state of the cycle already
// failed the test) — the reference would spin to rho and report not_converged.
// Every per-path array is sized by the kernel's depth bound D (the candidates' stride
// rounded up to 3, 5 or 8), so the thread's local-memory frame stays small.
template <int D>
struct Snapshot {
  double v[D][7];
};

template <int D>
__device__ __forceinline__ void take_snapshot(Snapshot<D>& sn, const RNode* nd, int d) {
#pragma unroll
  for (int q = 0; q < D; ++q) {
    if (q >= d) break;
    if (nd[q].kind == 0) {
      sn.v[q][0] = nd[q].c.x;
      sn.v[q][1] = nd[q].c.y;
      sn.v[q][2] = nd[q].c.z;
      sn.v[q][3] = nd[q].n.x;
      sn.v[q][4] = nd[q].n.y;
      sn.v[q][5] = nd[q].n.z;
      sn.v[q][6] = __longlong_as_double(static_cast<long long>(nd[q].label));
    } else {
      sn.v[q][0] = nd[q].p0;
    }
  }
}

template <int D>
__device__ __forceinline__ bool same_snapshot(const Snapshot<D>& sn, const RNode* nd, int d) {
#pragma unroll
  for (int q = 0; q < D; ++q) {
    if (q >= d) break;
    if (nd[q].kind == 0) {
      if (__double_as_longlong(sn.v[q][0]) != __double_as_longlong(nd[q].c.x) ||
          __double_as_longlong(sn.v[q][1]) != __double_as_longlong(nd[q].c.y) ||
          __double_as_longlong(sn.v[q][2]) != __double_as_longlong(nd[q].c.z) ||
          __double_as_longlong(sn.v[q][3]) != __double_as_longlong(nd[q].n.x) ||
          __double_as_longlong(sn.v[q][4]) != __double_as_longlong(nd[q].n.y) ||
          __double_as_longlong(sn.v[q][5]) != __double_as_longlong(nd[q].n.z) ||
          static_cast<uint32_t>(__double_as_longlong(sn.v[q][6])) != nd[q].label)
        return false;
    } else if (__double_as_longlong(sn.v[q][0]) != __double_as_longlong(nd[q].p0)) {
      return false;
    }
  }
  return true;
}

// Cycle detection without keeping the last states: a 64-bit hash of every post-iteration
// state is compared with the hashes of the states 1 and 2 iterations back and of
// Brent's saved state (taken at power-of-two steps). A hash match only SCHEDULES an
// exact check: the matching state S_i is copied and compared bitwise with S_{i+p},
// p being the suspected period. S_{i+p} == S_i means the trajectory repeats with
// period p from i, every state of the cycle has already failed ||g|| < delta, and the
// reference iterates to rho and reports not_converged — so the exit is exact whatever
// the hash did. One snapshot instead of three, and no snapshot store per iteration.
__device__ __forceinline__ uint64_t mix64(uint64_t h, uint64_t w) {
  h ^= w;
  h *= 0x9e3779b97f4a7c15ull;
  return h ^ (h >> 29);
}
template <int D>
__device__ __forceinline__ uint64_t state_hash(const RNode* nd, int d) {
  uint64_t h = 0x243f6a8885a308d3ull;
#pragma unroll
  for (int q = 0; q < D; ++q) {
    if (q >= d) break;
    if (nd[q].kind == 0) {
      h = mix64(h, static_cast<uint64_t>(__double_as_longlong(nd[q].c.x)));
      h = mix64(h, static_cast<uint64_t>(__double_as_longlong(nd[q].c.y)));
      h = mix64(h, static_cast<uint64_t>(__double_as_longlong(nd[q].c.z)));
      h = mix64(h, static_cast<uint64_t>(__double_as_longlong(nd[q].n.x)));
      h = mix64(h, static_cast<uint64_t>(__double_as_longlong(nd[q].n.y)));
      h = mix64(h, static_cast<uint64_t>(__double_as_longlong(nd[q].n.z)));
      h = mix64(h, nd[q].label);
    } else {
      h = mix64(h, static_cast<uint64_t>(__double_as_longlong(nd[q].p0)));
    }
  }
  return h;
}
// A second saved hash refreshed every PCR_CYC_FIXED iterations catches short cycles that
// start late (after Brent's last power-of-two save). Measured on C2: 2.006 G -> 1.985 G
// iterations (same outcomes and hash), refine 6.48 -> 6.44 s; so the ~685 k paths that
// run to rho are not short-periodic — they drift (profiles/ab_cycle_fixed_r02.log)
#ifndef PCR_CYC_FIXED
#define PCR_CYC_FIXED 64
#endif
template <int D>
struct CycleCheck {
  uint64_t h1, h2, hs;   // hashes of S_{i-1}, S_{i-2} and of Brent's saved state
  int saved_iter, power, lam, pend_at;
  uint64_t hf;           // PCR_CYC_FIXED > 0: a second saved hash, refreshed every PCR_CYC_FIXED iterations
  int fixed_iter;
  Snapshot<D> pending;   // a state suspected to recur at iteration pend_at
  __device__ __forceinline__ void init(const RNode* nd, int d) {
    h1 = h2 = hs = hf = state_hash<D>(nd, d);
    fixed_iter = -1;
    saved_iter = -1;
    power = 1;
    lam = 0;
    pend_at = -1;
  }
  // after iteration i produced the state nd: true when the trajectory is periodic
  __device__ __forceinline__ bool periodic(const RNode* nd, int d, int i) {
    const uint64_t h = state_hash<D>(nd, d);
    bool cyc = false;
    if (pend_at == i) {
      cyc = same_snapshot(pending, nd, d);  // the exact test
      pend_at = -1;
    }
    if (!cyc && pend_at < 0) {
      int p = h == h1 ? 1 : h == h2 ? 2 : h == hs ? i - saved_iter : 0;
      if (PCR_CYC_FIXED > 0 && p == 0 && h == hf) p = i - fixed_iter;
      if (p > 0) {
        take_snapshot(pending, nd, d);
        pend_at = i + p;
      }
    }
    h2 = h1;
    h1 = h;
    if (++lam == power) {
      hs = h;
      saved_iter = i;
      power <<= 1;
      lam = 0;
    }
    if (PCR_CYC_FIXED > 0 && (i + 1) % (PCR_CYC_FIXED > 0 ? PCR_CYC_FIXED : 1) == 0) {
      hf = h;
      fixed_iter = i;
    }
    return cyc;
  }
};

template <int D>
__device__ __forceinline__ void refine_one(uint32_t k, const CandIn& in, const GridView& g, const SceneView& s,
                                           double delta, int rho, double step_size, const RefOut& o);

// Persistent threads with per-thread work stealing: iteration counts range from 1 to
// rho, so a thread that finishes a path takes the next one instead of idling until
// the slowest lane of its warp is done.
constexpr int kRefineThreads = 128;
__device__ unsigned long long* g_refine_dbg = nullptr;
template <int D, int kMinBlocks>
__global__ void __launch_bounds__(kRefineThreads, kMinBlocks) refine_kernel(CandIn in, uint32_t n, GridView g, SceneView s,
                                                                   double delta, int rho, double step_size, RefOut o,
                                                                   uint32_t* next_cand, int rev) {
  uint32_t done = 0;
  unsigned long long t_start = 0;
  if (g_refine_dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  for (;;) {
    const uint32_t idx = atomicAdd(next_cand, 1u);
    if (idx >= n) break;
    // this shard's candidates are first, first + step, ... (SURVEY 8e round-robin)
    // list order by default (measured faster than back to front, PCR_REFINE_REV=1:
    // neighbours in DFS order are similar paths, so a warp's lanes diverge less)
    refine_one<D>(in.first + (rev ? n - 1 - idx : idx) * in.step, in, g, s, delta, rho, step_size, o);
    ++done;
  }
  if (g_refine_dbg) {  // development trace (PCR_REFINE_TRACE): per-thread finish time, paths
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    g_refine_dbg[3 * tid] = t_start;
    g_refine_dbg[3 * tid + 1] = t;
    g_refine_dbg[3 * tid + 2] = done;
  }
}

template <int D>
__device__ __forceinline__ void refine_one(uint32_t k, const CandIn& in, const GridView& g, const SceneView& s,
                                           double delta, int rho, double step_size, const RefOut& o) {
  const int d = static_cast<int>(in.n_inter[k]);
  const V3 tx = load3(in.tx + 3ull * k), rx = load3(in.rx + 3ull * k);
  o.has_path[k] = 0;
  o.iters[k] = 0;
  if (d == 0) {
    // LOS passes through (pipeline.cpp:160-170)
    o.has_path[k] = 1;
    o.reason[k] = PCR_NOT_CONVERGED;
    o.length[k] = in.coarse_length[k];
    o.delay[k] = in.coarse_length[k] / kSpeedOfLight;
    o.gnorm[k] = 0.0;
    return;
  }
  RNode nd[D];
  // make_path_state (refine.cpp:134-161)
  for (int q = 0; q < d; ++q) {
    const size_t j = static_cast<size_t>(k) * in.stride + q;
    RNode& x = nd[q];
    x.kind = in.kind[j];
    x.c = load3(in.pos + 3 * j);
    x.label = in.label[j];
    x.edge = in.edge[j];
    x.p0 = 0.0;
    x.p1 = 0.0;
    if (x.kind == 0) {
      x.n = load3(in.nrm + 3 * j);
      local_frame(x.n, x.a, x.b);
      x.lo = x.hi = 0.0;
    } else {
      const double* e = s.edges + 12ull * x.edge;
      const V3 es = load3(e), ee = load3(e + 3);
      x.a = normalized(ee - es);
      x.lo = dot(es - x.c, x.a);
      x.hi = dot(ee - x.c, x.a);
      x.b = V3{0, 1, 0};
      x.n = V3{0, 0, 1};
    }
  }
  V3 pts[D];
  for (int q = 0; q < d; ++q) pts[q] = node_point(nd[q], nd[q].p0, nd[q].p1);
  double f = chain_len(tx, pts, d, rx);
  double gnorm = 0.0;
  bool converged = false;
  int iter = 0;
  uint32_t n_trials = 0, n_march = 0;
  uint64_t n_iter_nodes = 0;
  auto flush = [&]() {
    atomicAdd(o.stats, static_cast<unsigned long long>(n_trials));
    atomicAdd(o.stats + 1, static_cast<unsigned long long>(n_march));
    atomicAdd(o.stats + 2, static_cast<unsigned long long>(n_trials) * d);
    atomicAdd(o.stats + 3, static_cast<unsigned long long>(n_iter_nodes));
  };
  // cycle detection on the post-iteration state (CycleCheck)
  CycleCheck<D> cyc;
  cyc.init(nd, d);
  bool stalled = false;
  for (; iter < rho; ++iter) {
    n_iter_nodes += d;
    // local_gradients
    double gr[2 * D];
    int ng = 0;
    for (int q = 0; q < d; ++q) {
      const V3 prev = q == 0 ? tx : pts[q - 1];
      const V3 next = q + 1 == d ? rx : pts[q + 1];
      const V3 dp = pts[q] - prev;
      const V3 dn = pts[q] - next;
      const double lp = norm(dp), ln = norm(dn);
      if (lp < kTiny || ln < kTiny) {
        o.reason[k] = PCR_DEGENERATE;
        o.iters[k] = iter + 1;
        flush();
        return;
      }
      const V3 e_sum = dp / lp + dn / ln;
      if (nd[q].kind == 0) {
        gr[ng++] = dot(nd[q].a, e_sum);
        gr[ng++] = dot(nd[q].b, e_sum);
      } else {
        gr[ng++] = dot(nd[q].a, e_sum);
      }
    }
    gnorm = 0.0;
    for (int q = 0; q < ng; ++q) gnorm += gr[q] * gr[q];
    gnorm = sqrt(gnorm);
    if (gnorm < delta) {
      converged = true;
      break;
    }
    // backtracking (refine.cpp:209-232)
    double step = step_size;
    bool accepted = false;
    double tp0[D], tp1[D];
    for (int h = 0; h <= 8; ++h) {
      int gi = 0;
      V3 tpts[D];
      for (int q = 0; q < d; ++q) {
        if (nd[q].kind == 0) {
          tp0[q] = nd[q].p0 - step * gr[gi++];
          tp1[q] = nd[q].p1 - step * gr[gi++];
        } else {
          tp0[q] = sclamp(nd[q].p0 - step * gr[gi++], nd[q].lo, nd[q].hi);
          tp1[q] = nd[q].p1;
        }
        tpts[q] = node_point(nd[q], tp0[q], tp1[q]);
      }
      ++n_trials;
      if (chain_len(tx, tpts, d, rx) <= f + 1e-15) {
        accepted = true;
        break;
      }
      step *= 0.5;
    }
    if (!accepted) {
      stalled = true;  // fixed point: every remaining iteration repeats this one
      break;
    }
    for (int q = 0; q < d; ++q) {
      nd[q].p0 = tp0[q];
      nd[q].p1 = tp1[q];
    }
    // reprojection, front to back (refine.cpp:234-250)
    for (int q = 0; q < d; ++q) {
      if (nd[q].kind != 0) continue;
      const V3 prev = q == 0 ? tx : node_point(nd[q - 1], nd[q - 1].p0, nd[q - 1].p1);
      const V3 predicted = node_point(nd[q], nd[q].p0, nd[q].p1);
      Reproj re;
      if (!reproject(prev, predicted, nd[q].label, g, s, re, n_march)) {
        o.reason[k] = PCR_RAY_MISSED;
        o.iters[k] = iter + 1;
        flush();
        return;
      }
      nd[q].c = re.pos;
      nd[q].n = re.nrm;
      local_frame(re.nrm, nd[q].a, nd[q].b);
      nd[q].p0 = 0.0;
      nd[q].p1 = 0.0;
      nd[q].label = re.label;
    }
    for (int q = 0; q < d; ++q) pts[q] = node_point(nd[q], nd[q].p0, nd[q].p1);
    f = chain_len(tx, pts, d, rx);
    // periodic trajectory: never converges (see Snapshot / CycleCheck)
    if (cyc.periodic(nd, d, iter)) {
      stalled = true;
      break;
    }
  }
  o.iters[k] = static_cast<uint32_t>(converged || stalled ? iter + 1 : iter);  // iterations executed
  flush();
  if (!converged) {
    o.reason[k] = PCR_NOT_CONVERGED;
    return;
  }
  // final per-segment visibility (refine.cpp:256-265)
  V3 prev = tx;
  for (int q = 0; q <= d; ++q) {
    const V3 next = q < d ? pts[q] : rx;
    if (!segment_visible(prev, next, kNoIe, g, s)) {
      o.reason[k] = PCR_OCCLUDED;
      return;
    }
    prev = next;
  }
  for (int q = 0; q < d; ++q) {
    const size_t j = static_cast<size_t>(k) * in.stride + q;
    store3(o.pos + 3 * j, pts[q]);
    if (nd[q].kind == 0) {
      store3(o.nrm + 3 * j, nd[q].n);
      o.label[j] = nd[q].label;
    }
  }
  const double total = chain_len(tx, pts, d, rx);
  o.length[k] = total;
  o.delay[k] = total / kSpeedOfLight;
  o.gnorm[k] = gnorm;
  o.reason[k] = PCR_NOT_CONVERGED;
  o.has_path[k] = 1;
}

// ---- warp-cooperative refinement ----------------------------------------------------
// Measured on C2 (PCR_REFINE_TRACE): the thread-per-path kernel empties its queue after
// ~1/4 of its run and spends the rest draining the last paths (up to rho = 2000
// iterations each) with most lanes idle. Here the 32 lanes of a warp iterate their own
// paths in lockstep, and the same-label reprojection scan (the bulk of an iteration)
// runs as one flat loop over the concatenated label runs of every lane reprojecting
// the same node index: lanes without a path (queue empty) scan for the others. Each
// record's hit distance is computed as in the serial scan; the winner per path is the
// least distance, ties to the earliest record in scan order — what the serial strict-<
// scan returns — found by a segmented (t, index) min over the round's lane segments.
// The scan's pruning (t_lo / t* against the best so far) only ever skips records that
// cannot win, so pruning against the best of earlier rounds changes nothing.

// The scan and the per-path steps are separate (not inlined) functions: each gets its
// own register allocation instead of one 168-register budget shared with the whole
// path state, which spilled inside the scan loop (measured: 714 -> 677 ms on C2).
#ifndef PCR_COOP_INLINE
#define PCR_COOP_INLINE __noinline__
#endif
#ifndef PCR_STEP_INLINE
#define PCR_STEP_INLINE __noinline__
#endif

struct ScanSlot {  // one per lane: the reprojection it posted and its best record so far
  double prev[3], dir[3], pred[3];
  double best_t;
  uint32_t pre, j0, best_f, pad;
};

// A node's last label run: (neighbourhood list, label) -> [j0, j0 + len). Successive
// iterations mostly reproject into the same cell, so the two binary searches are skipped.
struct RunCache {
  uint32_t cell, label, j0, len;
  uint32_t win;  // the last scan's winner, as a position in this run (kNoRec: none)
};

template <int D>
struct PathState {
  uint32_t k;
  int d, iter;
  V3 tx, rx;
  double f, gnorm;
  RNode nd[D];  // node points are recomputed from them (node_point: same bits every time)
  CycleCheck<D> cyc;
  RunCache rc[D];
};

constexpr uint32_t kNoRec = 0xffffffffu;
constexpr unsigned kFull = 0xffffffffu;

// make_path_state (refine.cpp:134-161); false when the path is done at once (LOS)
template <int D>
__device__ PCR_STEP_INLINE bool path_init(PathState<D>& st, uint32_t k, const CandIn& in, const SceneView& s, const RefOut& o) {
  const int d = static_cast<int>(in.n_inter[k]);
  st.k = k;
  st.d = d;
  st.tx = load3(in.tx + 3ull * k);
  st.rx = load3(in.rx + 3ull * k);
  o.has_path[k] = 0;
  o.iters[k] = 0;
  if (d == 0) {  // LOS passes through (pipeline.cpp:160-170)
    o.has_path[k] = 1;
    o.reason[k] = PCR_NOT_CONVERGED;
    o.length[k] = in.coarse_length[k];
    o.delay[k] = in.coarse_length[k] / kSpeedOfLight;
    o.gnorm[k] = 0.0;
    return false;
  }
  for (int q = 0; q < d; ++q) {
    const size_t j = static_cast<size_t>(k) * in.stride + q;
    RNode& x = st.nd[q];
    x.kind = in.kind[j];
    x.c = load3(in.pos + 3 * j);
    x.label = in.label[j];
    x.edge = in.edge[j];
    x.p0 = 0.0;
    x.p1 = 0.0;
    if (x.kind == 0) {
      x.n = load3(in.nrm + 3 * j);
      local_frame(x.n, x.a, x.b);
      x.lo = x.hi = 0.0;
    } else {
      const double* e = s.edges + 12ull * x.edge;
      const V3 es = load3(e), ee = load3(e + 3);
      x.a = normalized(ee - es);
      x.lo = dot(es - x.c, x.a);
      x.hi = dot(ee - x.c, x.a);
      x.b = V3{0, 1, 0};
      x.n = V3{0, 0, 1};
    }
  }
  V3 pts[D];
  for (int q = 0; q < d; ++q) {
    pts[q] = node_point(st.nd[q], st.nd[q].p0, st.nd[q].p1);
    st.rc[q].cell = 0xffffffffu;
  }
  st.f = chain_len(st.tx, pts, d, st.rx);
  st.gnorm = 0.0;
  st.iter = 0;
  st.cyc.init(st.nd, d);
  return true;
}

// converged: final per-segment visibility (refine.cpp:256-265) and the refined path.
// The warp kernel defers the visibility part (PCR_DEFER_VIS, default): it writes the
// refined path with the private reason kPendingVis, and converged_vis_kernel runs the
// d + 1 segment tests afterwards with warp_segment_visible, 32 lanes per segment,
// instead of one lane walking alone while its warp-mates wait (the converging lane is
// alone in this branch). An occluded path then gets the outcome the inline test gives:
// reason occluded, no path, the candidate's own points / normals / labels.
#ifndef PCR_DEFER_VIS
#define PCR_DEFER_VIS 1
#endif
constexpr int32_t kPendingVis = 0x7fff0001;
template <int D>
__device__ PCR_STEP_INLINE void path_converged(const PathState<D>& st, const CandIn& in, const GridView& g, const SceneView& s,
                               const RefOut& o) {
  const uint32_t k = st.k;
  const int d = st.d;
  V3 pts[D];
  for (int q = 0; q < d; ++q) pts[q] = node_point(st.nd[q], st.nd[q].p0, st.nd[q].p1);
  if (!PCR_DEFER_VIS) {
    V3 prev = st.tx;
    for (int q = 0; q <= d; ++q) {
      const V3 next = q < d ? pts[q] : st.rx;
      if (!segment_visible(prev, next, kNoIe, g, s)) {
        o.reason[k] = PCR_OCCLUDED;
        return;
      }
      prev = next;
    }
  }
  for (int q = 0; q < d; ++q) {
    const size_t j = static_cast<size_t>(k) * in.stride + q;
    store3(o.pos + 3 * j, pts[q]);
    if (st.nd[q].kind == 0) {
      store3(o.nrm + 3 * j, st.nd[q].n);
      o.label[j] = st.nd[q].label;
    }
  }
  const double total = chain_len(st.tx, pts, d, st.rx);
  o.length[k] = total;
  o.delay[k] = total / kSpeedOfLight;
  o.gnorm[k] = st.gnorm;
  o.reason[k] = PCR_DEFER_VIS ? kPendingVis : PCR_NOT_CONVERGED;
  o.has_path[k] = 1;
}

// One iteration up to the reprojection: rho bound, local_gradients (:167-187), the
// convergence test, backtracking (:209-232). False when the path is finished.
template <int D>
__device__ PCR_STEP_INLINE bool path_step_a(PathState<D>& st, const CandIn& in, const GridView& g, const SceneView& s, double delta,
                            int rho, double step_size, const RefOut& o, uint32_t& n_trials,
                            unsigned long long& n_nodes) {
  const uint32_t k = st.k;
  const int d = st.d;
  if (st.iter >= rho) {
    o.iters[k] = static_cast<uint32_t>(st.iter);
    o.reason[k] = PCR_NOT_CONVERGED;
    return false;
  }
  // loops unrolled to the depth bound with q < d guards: the per-node values stay in
  // registers (a runtime-indexed array would live in local memory)
  n_nodes += static_cast<unsigned long long>(d) << 32;  // iteration executed (high word)
  double ga[D], gb[D];
  bool refl[D];
  V3 pts[D];
#pragma unroll
  for (int q = 0; q < D; ++q) {
    if (q < d) {
      pts[q] = node_point(st.nd[q], st.nd[q].p0, st.nd[q].p1);
      refl[q] = st.nd[q].kind == 0;
    }
  }
#pragma unroll
  for (int q = 0; q < D; ++q) {
    if (q < d) {
      const V3 prev = q == 0 ? st.tx : pts[q > 0 ? q - 1 : 0];
      const V3 next = (q + 1 < D && q + 1 < d) ? pts[q + 1 < D ? q + 1 : q] : st.rx;
      const V3 dp = pts[q] - prev;
      const V3 dn = pts[q] - next;
      const double lp = norm(dp), ln = norm(dn);
      if (lp < kTiny || ln < kTiny) {
        o.reason[k] = PCR_DEGENERATE;
        o.iters[k] = static_cast<uint32_t>(st.iter + 1);
        return false;
      }
      const V3 e_sum = dp / lp + dn / ln;
      ga[q] = dot(st.nd[q].a, e_sum);
      gb[q] = refl[q] ? dot(st.nd[q].b, e_sum) : 0.0;
    }
  }
  double gn = 0.0;  // same order as the reference's gradient vector: (u, v) per reflection, w per edge
#pragma unroll
  for (int q = 0; q < D; ++q) {
    if (q < d) {
      gn += ga[q] * ga[q];
      if (refl[q]) gn += gb[q] * gb[q];
    }
  }
  st.gnorm = sqrt(gn);
  if (st.gnorm < delta) {
    o.iters[k] = static_cast<uint32_t>(st.iter + 1);
    path_converged(st, in, g, s, o);
    return false;
  }
  double step = step_size;
  for (int h = 0; h <= 8; ++h) {
    double tp0[D], tp1[D];
    V3 prev = st.tx;
    double len = 0.0;  // chain_len over the trial points, same summation order
#pragma unroll
    for (int q = 0; q < D; ++q) {
      if (q < d) {
        const RNode& nd = st.nd[q];
        if (refl[q]) {
          tp0[q] = nd.p0 - step * ga[q];
          tp1[q] = nd.p1 - step * gb[q];
        } else {
          tp0[q] = sclamp(nd.p0 - step * ga[q], nd.lo, nd.hi);
          tp1[q] = nd.p1;
        }
        const V3 tp = node_point(nd, tp0[q], tp1[q]);
        len += norm(tp - prev);
        prev = tp;
      }
    }
    ++n_trials;
    n_nodes += static_cast<unsigned long long>(d);  // trial nodes (low word)
    if (len + norm(st.rx - prev) <= st.f + 1e-15) {
#pragma unroll
      for (int q = 0; q < D; ++q) {
        if (q < d) {
          st.nd[q].p0 = tp0[q];
          st.nd[q].p1 = tp1[q];
        }
      }
      return true;
    }
    step *= 0.5;
  }
  // fixed point: every remaining iteration repeats this one (not_converged)
  o.iters[k] = static_cast<uint32_t>(st.iter + 1);
  o.reason[k] = PCR_NOT_CONVERGED;
  return false;
}

// After the reprojection: new chain length, cycle checks (see Snapshot), next iteration.
template <int D>
__device__ PCR_STEP_INLINE bool path_step_c(PathState<D>& st, const RefOut& o) {
  const int d = st.d;
  V3 prev = st.tx;
  double len = 0.0;  // chain_len, same summation order
#pragma unroll
  for (int q = 0; q < D; ++q) {
    if (q < d) {
      const V3 p = node_point(st.nd[q], st.nd[q].p0, st.nd[q].p1);
      len += norm(p - prev);
      prev = p;
    }
  }
  st.f = len + norm(st.rx - prev);
  if (st.cyc.periodic(st.nd, d, st.iter)) {
    o.iters[st.k] = static_cast<uint32_t>(st.iter + 1);
    o.reason[st.k] = PCR_NOT_CONVERGED;
    return false;
  }
  ++st.iter;
  return true;
}

// reproject's set-up (refine.cpp:80-90): 0 = missed (degenerate direction), 1 = the
// same-label pass is the label run [j0, j0 + len) of the 3x3x3 neighbourhood list,
// 2 = no neighbourhood list for this box (serial reproject)
__device__ __forceinline__ int reproject_setup(const V3& prev, const V3& predicted, uint32_t label, const GridView& g,
                                               V3& dir, uint32_t& j0, uint32_t& len, RunCache& rc) {
  const V3 diff = predicted - prev;
  const double dist = norm(diff);
  if (dist < kTiny) return 0;
  dir = diff / dist;
  if (g.nb_off == nullptr) return 2;
  const double radius = 2.0 * g.sub_edge;
  const double pc[3] = {predicted.x, predicted.y, predicted.z};
  const double oc[3] = {g.origin.x, g.origin.y, g.origin.z};
  int cc[3];
  for (int a = 0; a < 3; ++a) {
    const int l = voxel_floor(pc[a] - radius, oc[a], g.voxel_size);
    const int h = voxel_floor(pc[a] + radius, oc[a], g.voxel_size);
    cc[a] = l + 1;
    if (!(h == l + 2 && cc[a] >= 0 && cc[a] < g.dims[a])) return 2;
  }
  const uint32_t c = linear_index(g, cc[0], cc[1], cc[2]);
  if (c == rc.cell && label == rc.label) {  // same list and label as this node's last scan
    j0 = rc.j0;
    len = rc.len;
    return 1;
  }
  uint32_t lo = g.nb_off[c], hi = g.nb_off[c + 1];
  const uint32_t end = hi;
  while (lo < hi) {
    const uint32_t m = (lo + hi) >> 1;
    if (g.nb_lab[m] < label) lo = m + 1; else hi = m;
  }
  j0 = lo;
  hi = end;
  while (lo < hi) {
    const uint32_t m = (lo + hi) >> 1;
    if (g.nb_lab[m] <= label) lo = m + 1; else hi = m;
  }
  len = lo - j0;
  rc = RunCache{c, label, j0, len, 0xffffffffu};
  return 1;
}

// Per-lane scan scratch kept across calls: the plane division cache and the march count.
struct ScanCache {
  long long c_num, c_dn;
  double c_t;
  uint32_t n_march;
};

// read-only global loads of a 32-byte record (the scan's arrays never change in a launch)
__device__ __forceinline__ double4 ldg4(const double4* p) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p)), b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

// the warps' scan slots and round owner maps (file scope, so the out-of-line scan
// addresses them as shared memory rather than through generic pointers)
__shared__ ScanSlot g_slots[kRefineThreads];
__shared__ uint8_t g_owner_at[kRefineThreads];

// A non-planar record of the cooperative scan: its march_segment distance when it is a
// hit nearer than bt, else +inf. Out of line with the vectors passed by value: taking
// their address for march_segment put the scan's vectors in local memory every round.
__device__ __noinline__ double march_np(double px, double py, double pz, double dx, double dy, double dz, uint32_t ie,
                                        const GridView& g, const SceneView& s, double bt) {
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const V3 pv{px, py, pz}, dv{dx, dy, dz};
  SurfaceHit hit;
  if (march_segment(pv, dv, ie, g, s, inf, &hit) && hit.distance < bt) return hit.distance;
  return inf;
}

// The warp's same-label scans as one flat loop (every lane calls it). A posting lane
// (len > 0) has written prev, dir, pred and j0 into its slot. Not inlined: the caller's
// path state stays out of the loop's registers (it spilled inside the loop otherwise).
__device__ PCR_COOP_INLINE void coop_scan(int lane, uint32_t len, const GridView& g, const SceneView& s,
                                          ScanCache* cache) {
  const uint32_t wb = threadIdx.x & ~31u;
  ScanSlot* ws = g_slots + wb;
  uint8_t* owner_at = g_owner_at + wb;
  // the grid fields the loop reads, in registers (g is a reference into the caller's frame)
  const double4* __restrict__ nb_rec = g.nb_rec;
  const double4* __restrict__ nb_pa = g.nb_pa;
  const double4* __restrict__ nb_pb = g.nb_pb;
  const double eps = g.hit_eps;
#ifndef PCR_FAST_REJECT
#define PCR_FAST_REJECT 0
#endif
  const bool fast = PCR_FAST_REJECT && g.fast_reject != 0;
  const bool uniform = g.rr_uniform != 0;
  const double uradius = g.rr_radius;
  long long c_num = cache->c_num, c_dn = cache->c_dn;
  double c_t = cache->c_t;
  uint32_t n_march = cache->n_march;
  uint32_t incl = len;
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t v = __shfl_up_sync(kFull, incl, off);
    if (lane >= off) incl += v;
  }
  const uint32_t total = __shfl_sync(kFull, incl, 31);
  const uint32_t pre = incl - len;
  ScanSlot& me = ws[lane];
  // the caller may seed the best with its last winner (best_f = position in the run):
  // the scan then only evaluates records that can still beat it, (t, index)-wise
  const uint32_t seed = len ? me.best_f : kNoRec;
  me.best_f = seed == kNoRec ? kNoRec : pre + seed;
  if (total == 0) return;
  if (seed == kNoRec) me.best_t = 1.7976931348623157e308;
  me.pre = pre;
  __syncwarp();
  const double radius = 2.0 * g.sub_edge;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  int carry = 0;
  for (uint32_t base = 0; base < total; base += 32) {
    const bool starts = len && pre >= base && pre - base < 32u;
    if (starts) owner_at[pre - base] = static_cast<uint8_t>(lane);
    const uint32_t smask = __reduce_or_sync(kFull, starts ? 1u << (pre - base) : 0u);
    __syncwarp();
    const uint32_t F = base + lane;
    const bool valid = F < total;
    const uint32_t below = smask & (kFull >> (31 - lane));
    int o = below ? owner_at[31 - __clz(below)] : carry;
    double t = inf;
    if (valid) {
      const ScanSlot& sl = ws[o];
      const uint32_t j = sl.j0 + (F - sl.pre);
      // the record first; its plane (side arrays, no dependent load through the IE
      // index) only for records that survive the radius and window tests
      const double4 r4 = ldg4(nb_rec + j);
#ifndef PCR_SCAN_EAGER
#define PCR_SCAN_EAGER 1
#endif
      // PCR_SCAN_EAGER (default): the plane loads issued with the record's — one memory
      // round trip per round instead of two dependent ones, extra bytes for rejected
      // records. Same box: C2 refine 6.82-7.11 s -> 6.52-6.53 s, C2d3 576-592 -> 568-572
      // ms (profiles/ab_eager_r02.log)
      double4 pa_e, pb_e;
      if (PCR_SCAN_EAGER) {
        pa_e = ldg4(nb_pa + j);
        pb_e = ldg4(nb_pb + j);
      }
      const uint64_t w = static_cast<uint64_t>(__double_as_longlong(r4.w));
      const uint32_t ie = static_cast<uint32_t>(w >> 33);
      const V3 sc = ld3(r4);
      const double rad = uniform ? uradius : PCR_SCAN_EAGER ? pa_e.w : __ldg(&nb_pa[j].w);
      const V3 pq{sl.pred[0], sl.pred[1], sl.pred[2]};
      if (norm_le(sc - pq, radius + rad)) {
        ++n_march;  // counts the reference's march_segment call
        const V3 pv{sl.prev[0], sl.prev[1], sl.prev[2]}, dv{sl.dir[0], sl.dir[1], sl.dir[2]};
        const double t_center = dot(sc - pv, dv);
        const double t_lo = smax(0.0, t_center - rad);
        const double best = sl.best_t;
        // every hit of this window lies at t >= t_lo: it can only win if t_lo < best,
        // or t_lo == best with a lower record index than the best's (seeds may sit
        // anywhere in the run); a lower index wins ties, so its bound admits t == best
        const bool lower = F < sl.best_f;
        if (t_lo < best || (t_lo == best && lower)) {
          double bt = lower ? nextafter(best, inf) : best;
          if (__builtin_expect(((w >> 32) & 1u) != 0, 1)) {  // planar records are the common case
            const double4 pa = PCR_SCAN_EAGER ? pa_e : ldg4(nb_pa + j);
            const double4 pb = PCR_SCAN_EAGER ? pb_e : ldg4(nb_pb + j);
            if (planar_candidate_at(pv, dv, ld3(pa), ld3(pb), eps, t_lo, t_center + rad, bt, c_num, c_dn, c_t, fast))
              t = bt;
          } else {
            t = march_np(pv.x, pv.y, pv.z, dv.x, dv.y, dv.z, ie, g, s, bt);
          }
        }
      }
    } else {
      o = 32;  // no record: a segment of its own
    }
    carry = __shfl_sync(kFull, o, 31);
    // rounds without a hit (every record pruned or missed) leave the owners' bests as they are
#ifndef PCR_SKIP_EMPTY
#define PCR_SKIP_EMPTY 1
#endif
    if (PCR_SKIP_EMPTY && !__any_sync(kFull, t < inf)) {
      __syncwarp();
      continue;
    }
    // segmented (t, F) min towards each segment's first lane; ties keep the lower F.
    // Segments are the owners' runs within the round: they start at lane 0 and at the
    // run starts (smask); lanes past the last record (t = +inf) never win.
    const uint32_t heads = smask | 1u;
    const uint32_t above = heads & ~(kFull >> (31 - lane));
    const int seg_end = above ? __ffs(above) - 1 : 32;
    double bt = t;
    uint32_t bf = F;
    for (int off = 1; off < 32; off <<= 1) {
      const double ot = __shfl_down_sync(kFull, bt, off);
      const uint32_t of = __shfl_down_sync(kFull, bf, off);
      if (lane + off < seg_end && ot < bt) {
        bt = ot;
        bf = of;
      }
    }
    __syncwarp();
    if (valid && ((heads >> lane) & 1u) && (bt < ws[o].best_t || (bt == ws[o].best_t && bf < ws[o].best_f))) {
      ws[o].best_t = bt;
      ws[o].best_f = bf;
    }
    __syncwarp();
  }
  cache->c_num = c_num;
  cache->c_dn = c_dn;
  cache->c_t = c_t;
  cache->n_march = n_march;
}

// Two-records-per-lane variant of the packed scan (PCR_SCAN_ILP2=1): rounds of 64
// records, lane l evaluating positions base + l and base + 32 + l with straight-line
// code (both records' loads, radius tests, windows, plane snaps and endpoint tests
// computed unconditionally and combined by selects), so each lane carries two
// independent FP64 chains through the round instead of one. Same decisions per record
// as planar_candidate_at (the division cache is not used: t* is recomputed, same
// bits); non-planar records march afterwards. The second half prunes against the
// bests from before the first half's update, which only evaluates more records. The
// two halves are then reduced and merged into the owners' bests one after the other.
#ifndef PCR_SCAN_ILP2
#define PCR_SCAN_ILP2 0
#endif
__shared__ uint8_t g_owner_at2[2 * kRefineThreads];

__device__ PCR_COOP_INLINE void coop_scan_ilp2(int lane, uint32_t len, const GridView& g, const SceneView& s,
                                               ScanCache* cache) {
  const uint32_t wb = threadIdx.x & ~31u;
  ScanSlot* ws = g_slots + wb;
  uint8_t* owner_at = g_owner_at2 + 2 * wb;
  const double4* __restrict__ nb_rec = g.nb_rec;
  const double4* __restrict__ nb_pa = g.nb_pa;
  const double4* __restrict__ nb_pb = g.nb_pb;
  const double eps = g.hit_eps;
  const bool uniform = g.rr_uniform != 0;
  const double uradius = g.rr_radius;
  uint32_t n_march = cache->n_march;
  uint32_t incl = len;
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t v = __shfl_up_sync(kFull, incl, off);
    if (lane >= off) incl += v;
  }
  const uint32_t total = __shfl_sync(kFull, incl, 31);
  const uint32_t pre = incl - len;
  ScanSlot& me = ws[lane];
  const uint32_t seed = len ? me.best_f : kNoRec;
  me.best_f = seed == kNoRec ? kNoRec : pre + seed;
  if (total == 0) return;
  if (seed == kNoRec) me.best_t = 1.7976931348623157e308;
  me.pre = pre;
  __syncwarp();
  const double radius = 2.0 * g.sub_edge;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const uint32_t lmask = kFull >> (31 - lane);  // lanes 0..lane
  int carry = 0;
  for (uint32_t base = 0; base < total; base += 64) {
    const uint32_t rel = pre - base;
    const bool in_round = len && pre >= base && rel < 64u;
    if (in_round) owner_at[rel] = static_cast<uint8_t>(lane);
    const uint32_t sm0 = __reduce_or_sync(kFull, in_round && rel < 32u ? 1u << rel : 0u);
    const uint32_t sm1 = __reduce_or_sync(kFull, in_round && rel >= 32u ? 1u << (rel - 32u) : 0u);
    __syncwarp();
    const uint32_t b0 = sm0 & lmask, b1 = sm1 & lmask;
    const int last0 = sm0 ? owner_at[31 - __clz(sm0)] : carry;  // owner of position base + 31
    int o[2];
    o[0] = b0 ? owner_at[31 - __clz(b0)] : carry;
    o[1] = b1 ? owner_at[63 - __clz(b1)] : last0;
    uint32_t F[2] = {base + lane, base + 32 + lane};
    bool valid[2] = {F[0] < total, F[1] < total};
    double t[2];
    bool np[2];
    double4 r4[2], pa[2], pb[2];
    uint32_t j[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const ScanSlot& sl = ws[valid[k] ? o[k] : 0];
      j[k] = valid[k] ? sl.j0 + (F[k] - sl.pre) : 0u;
      r4[k] = ldg4(nb_rec + j[k]);
      pa[k] = ldg4(nb_pa + j[k]);
      pb[k] = ldg4(nb_pb + j[k]);
    }
    bool band[2], near[2], cand[2];
    double bt[2], yv[2], sq[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const ScanSlot& sl = ws[valid[k] ? o[k] : 0];
      const V3 sc = ld3(r4[k]);
      const uint64_t w = static_cast<uint64_t>(__double_as_longlong(r4[k].w));
      const bool planar = ((w >> 32) & 1u) != 0;
      const double rad = uniform ? uradius : pa[k].w;
      const V3 pq{sl.pred[0], sl.pred[1], sl.pred[2]};
      const V3 pv{sl.prev[0], sl.prev[1], sl.prev[2]}, dv{sl.dir[0], sl.dir[1], sl.dir[2]};
      // norm_le(sc - pq, radius + rad), its band resolved below
      yv[k] = radius + rad;
      sq[k] = sqnorm(sc - pq);
      const double yy = yv[k] * yv[k];
      const bool in_ = sq[k] <= yy * (1.0 - 1e-12), out_ = sq[k] >= yy * (1.0 + 1e-12);
      band[k] = valid[k] && !in_ && !out_;
      near[k] = in_;
      const double t_center = dot(sc - pv, dv);
      const double t_lo = smax(0.0, t_center - rad);
      const double t_hi = t_center + rad;
      const double best = sl.best_t;
      const bool lower = F[k] < sl.best_f;
      cand[k] = valid[k] && (t_lo < best || (t_lo == best && lower));
      // nextafter(best, +inf) for best >= +0 (bests are hit distances >= 0 or DBL_MAX)
      bt[k] = lower ? __longlong_as_double(__double_as_longlong(best) + 1) : best;
      // planar_candidate_at without early exits (same operations, same bits)
      const V3 pp = ld3(pa[k]), pn = ld3(pb[k]);
      const double dn = dot(dv, pn);
      const bool snap = fabs(dn) > 1e-12;
      const double num = dot(pp - pv, pn);
      const double t_star = num / dn;
      const bool in_win = snap && t_star >= t_lo && t_star <= t_hi;
      const double f = dot((pv + t_lo * dv) - pp, pn);
      const double f_hi = dot((pv + t_hi * dv) - pp, pn);
      const bool hit_lo = fabs(f) <= eps, sign = f * f_hi < 0.0, hit_hi = fabs(f_hi) <= eps;
      const double tc = hit_lo ? t_lo : sign ? 0.5 * (t_lo + t_hi) : t_hi;
      const double tt = in_win ? t_star : tc;
      const bool hit = t_hi > t_lo && (hit_lo || sign || hit_hi) && tt < bt[k];
      t[k] = planar && hit ? tt : inf;
      np[k] = !planar;
    }
    if (__any_sync(kFull, band[0] || band[1])) {
#pragma unroll
      for (int k = 0; k < 2; ++k)
        if (band[k]) near[k] = sqrt(sq[k]) <= yv[k];
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      n_march += valid[k] && near[k];  // counts the reference's march_segment call
      if (!(valid[k] && near[k] && cand[k])) t[k] = inf;
      np[k] = np[k] && valid[k] && near[k] && cand[k];
    }
    if (__any_sync(kFull, np[0] || np[1])) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (np[k]) {
          const ScanSlot& sl = ws[o[k]];
          const uint64_t w = static_cast<uint64_t>(__double_as_longlong(r4[k].w));
          t[k] = march_np(sl.prev[0], sl.prev[1], sl.prev[2], sl.dir[0], sl.dir[1], sl.dir[2],
                          static_cast<uint32_t>(w >> 33), g, s, bt[k]);
        }
      }
    }
    carry = __shfl_sync(kFull, valid[1] ? o[1] : 32, 31);
    // the two halves' segmented (t, F) mins, merged into the owners' bests in order
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (!__any_sync(kFull, t[k] < inf)) continue;
      const uint32_t heads = (k == 0 ? sm0 : sm1) | 1u;
      const uint32_t above = heads & ~lmask;
      const int seg_end = above ? __ffs(above) - 1 : 32;
      double bv = t[k];
      uint32_t bf = F[k];
      for (int off = 1; off < 32; off <<= 1) {
        const double ot = __shfl_down_sync(kFull, bv, off);
        const uint32_t of = __shfl_down_sync(kFull, bf, off);
        if (lane + off < seg_end && ot < bv) {
          bv = ot;
          bf = of;
        }
      }
      __syncwarp();
      const int ok = o[k];
      if (valid[k] && ((heads >> lane) & 1u) &&
          (bv < ws[ok].best_t || (bv == ws[ok].best_t && bf < ws[ok].best_f))) {
        ws[ok].best_t = bv;
        ws[ok].best_f = bf;
      }
      __syncwarp();
    }
  }
  cache->n_march = n_march;
}

// The seed of a same-label scan: the record at position `win` of the run (the node's
// previous winner), evaluated exactly as the scan evaluates a record against an empty
// best — radius test, window, planar snap or march. A hit becomes the scan's initial
// best (t, position); a miss leaves the scan unseeded. Not counted in n_march (the scan
// visits and counts the record itself).
// Off by default since the eager plane loads: on the planar contract configs the seed
// evaluation costs more than it prunes (same box: C2 refine 6.44-6.47 -> 6.27-6.28 s,
// C2d3 543-582 -> 527-577 ms, C3 4.12 -> 3.49 s without; profiles/ab_noseed_r02.log).
// A runtime switch on the grid's planarity kept the seeding call in the kernel and lost
// the gain (6.45 s), so it is compile-time; non-planar grids (C2-np) gave up ~2.6 %
// (depth 1: 34.0 s with seeds, 34.9 s without, measured before the eager loads).
#ifndef PCR_SCAN_SEED
#define PCR_SCAN_SEED 0
#endif
__device__ __noinline__ void seed_winner(const V3& prev, const V3& dir, const V3& pred, uint32_t j0, uint32_t win,
                                         const GridView& g, const SceneView& s, ScanSlot& me) {
  const uint32_t j = j0 + win;
  const double4 r4 = ldg4(g.nb_rec + j);
  const double4 pa = ldg4(g.nb_pa + j);
  const double4 pb = ldg4(g.nb_pb + j);
  const V3 sc = ld3(r4);
  const double rad = pa.w;
  if (!norm_le(sc - pred, 2.0 * g.sub_edge + rad)) return;
  const double t_center = dot(sc - prev, dir);
  const double t_lo = smax(0.0, t_center - rad);
  const uint64_t w = static_cast<uint64_t>(__double_as_longlong(r4.w));
  double bt = 1.7976931348623157e308;
  if ((w >> 32) & 1u) {
    long long c_num = 0x7ff8dead7ff8deadll, c_dn = 0x7ff8dead7ff8deadll;
    double c_t = 0.0;
    if (!planar_candidate_at(prev, dir, ld3(pa), ld3(pb), g.hit_eps, t_lo, t_center + rad, bt, c_num, c_dn, c_t))
      return;
  } else {
    bt = march_np(prev.x, prev.y, prev.z, dir.x, dir.y, dir.z, static_cast<uint32_t>(w >> 33), g, s, bt);
    if (!(bt < __longlong_as_double(0x7ff0000000000000ll))) return;
  }
  me.best_t = bt;
  me.best_f = win;
}

// Prefetching variant of the packed scan (PCR_SCAN_PREFETCH=1; measured slower and off:
// C2 depth 4 refine 7.20-7.21 s without vs 7.70-7.72 s with, depth 3 574 vs 622 ms,
// same box — the record loads are not what the rounds wait on): the same rounds of 32
// records over the concatenated runs, but each lane copies its NEXT round's record
// (96 bytes: the list record and its plane) into a per-lane shared-memory slot with
// cp.async while the current round computes, so the round reads its record from shared
// memory instead of waiting on L2. The owner of a record index is found by a binary
// search over the lanes' inclusive run ends (warp shuffles), which needs no per-round
// owner map. Winners, pruning and the segmented (t, index) min are the packed scan's.
__shared__ double4 g_pf[2][kRefineThreads][3];

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

// owning lane of concatenated record F: the first lane whose inclusive run end exceeds F
__device__ __forceinline__ int owner_of(uint32_t F, uint32_t incl) {
  int lo = 0, hi = 31;
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int mid = (lo + hi) >> 1;
    const uint32_t v = __shfl_sync(kFull, incl, mid);
    if (v > F) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

__device__ PCR_COOP_INLINE void coop_scan_pf(int lane, uint32_t len, const GridView& g, const SceneView& s,
                                             ScanCache* cache) {
  const uint32_t wb = threadIdx.x & ~31u;
  ScanSlot* ws = g_slots + wb;
  const double4* __restrict__ nb_rec = g.nb_rec;
  const double4* __restrict__ nb_pa = g.nb_pa;
  const double4* __restrict__ nb_pb = g.nb_pb;
  const double eps = g.hit_eps;
  const bool fast = PCR_FAST_REJECT && g.fast_reject != 0;
  long long c_num = cache->c_num, c_dn = cache->c_dn;
  double c_t = cache->c_t;
  uint32_t n_march = cache->n_march;
  uint32_t incl = len;
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t v = __shfl_up_sync(kFull, incl, off);
    if (lane >= off) incl += v;
  }
  const uint32_t total = __shfl_sync(kFull, incl, 31);
  const uint32_t pre = incl - len;
  ScanSlot& me = ws[lane];
  me.best_f = kNoRec;
  if (total == 0) return;
  me.best_t = 1.7976931348623157e308;
  me.pre = pre;
  __syncwarp();
  const double radius = 2.0 * g.sub_edge;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  // issue the copy of record F into buffer b (lanes past the end copy nothing)
  auto prefetch = [&](uint32_t F, int b) {
    const int po = owner_of(F < total ? F : total - 1, incl);  // warp-uniform shuffles
    if (F < total) {
      const ScanSlot& sl = ws[po];
      const uint32_t j = sl.j0 + (F - sl.pre);
      double4* dst = g_pf[b][threadIdx.x];
      cp_async16(&dst[0], nb_rec + j);
      cp_async16(reinterpret_cast<char*>(&dst[0]) + 16, reinterpret_cast<const char*>(nb_rec + j) + 16);
      cp_async16(&dst[1], nb_pa + j);
      cp_async16(reinterpret_cast<char*>(&dst[1]) + 16, reinterpret_cast<const char*>(nb_pa + j) + 16);
      cp_async16(&dst[2], nb_pb + j);
      cp_async16(reinterpret_cast<char*>(&dst[2]) + 16, reinterpret_cast<const char*>(nb_pb + j) + 16);
    }
    cp_async_commit();
  };
  prefetch(lane, 0);
  int buf = 0;
  for (uint32_t base = 0; base < total; base += 32) {
    prefetch(base + 32 + lane, buf ^ 1);
    cp_async_wait1();  // this round's record has landed
    const uint32_t F = base + lane;
    const bool valid = F < total;
    const int o = owner_of(valid ? F : total - 1, incl);
    double t = inf;
    if (valid) {
      const ScanSlot& sl = ws[o];
      const double4* rec = g_pf[buf][threadIdx.x];
      const double4 r4 = rec[0];
      const double4 pa = rec[1];
      const uint64_t w = static_cast<uint64_t>(__double_as_longlong(r4.w));
      const uint32_t ie = static_cast<uint32_t>(w >> 33);
      const V3 sc = ld3(r4);
      const double rad = pa.w;
      const V3 pq{sl.pred[0], sl.pred[1], sl.pred[2]};
      if (norm_le(sc - pq, radius + rad)) {
        ++n_march;  // counts the reference's march_segment call
        const V3 pv{sl.prev[0], sl.prev[1], sl.prev[2]}, dv{sl.dir[0], sl.dir[1], sl.dir[2]};
        const double t_center = dot(sc - pv, dv);
        const double t_lo = smax(0.0, t_center - rad);
        double bt = sl.best_t;
        if (t_lo < bt) {
          if (__builtin_expect(((w >> 32) & 1u) != 0, 1)) {
            const double4 pb = rec[2];
            if (planar_candidate_at(pv, dv, ld3(pa), ld3(pb), eps, t_lo, t_center + rad, bt, c_num, c_dn, c_t, fast))
              t = bt;
          } else {
            t = march_np(pv.x, pv.y, pv.z, dv.x, dv.y, dv.z, ie, g, s, bt);
          }
        }
      }
    }
    buf ^= 1;
    if (PCR_SKIP_EMPTY && !__any_sync(kFull, t < inf)) continue;
    // segmented (t, F) min towards each owner segment's first lane in this round
    const int ow = valid ? o : 32;
    const int prev_o = __shfl_up_sync(kFull, ow, 1);
    const bool head = lane == 0 || prev_o != ow;
    const uint32_t heads = __ballot_sync(kFull, head);
    const uint32_t above = heads & ~(kFull >> (31 - lane));
    const int seg_end = above ? __ffs(above) - 1 : 32;
    double bt = t;
    uint32_t bf = F;
    for (int off = 1; off < 32; off <<= 1) {
      const double ot = __shfl_down_sync(kFull, bt, off);
      const uint32_t of = __shfl_down_sync(kFull, bf, off);
      if (lane + off < seg_end && ot < bt) {
        bt = ot;
        bf = of;
      }
    }
    __syncwarp();
    if (valid && head && bt < ws[o].best_t) {
      ws[o].best_t = bt;
      ws[o].best_f = bf;
    }
    __syncwarp();
  }
  asm volatile("cp.async.wait_all;\n" ::);
  cache->c_num = c_num;
  cache->c_dn = c_dn;
  cache->c_t = c_t;
  cache->n_march = n_march;
}

#ifndef PCR_SCAN_PREFETCH
#define PCR_SCAN_PREFETCH 0
#endif

// Owner-major variant of the same scan (A/B alternative, PCR_SCAN_OWNER=1; measured
// slower: C2 depth 3 refine 557-563 ms packed vs 715-751 ms owner-major, depth 4
// 7.54 s vs 9.93 s, same box — runs of ~25 records leave a quarter of the lanes idle
// and the kernel is latency-bound, so the lighter per-record code does not pay): the
// posting lanes' runs are walked one owner at a time, all 32 lanes on records
// j0 + base + lane of that owner's run. The owner's ray
// is warp-uniform (broadcast shared-memory loads, no per-record owner lookup), and the
// round's winner is a plain warp (t, index) min — usually a single hit, found by a
// ballot — instead of the packed variant's segmented reduction. Pruning uses the best
// of the owner's earlier rounds (lower record indices), so the winner is again the
// least distance, ties to the earliest record: the serial scan's strict-< result.
__device__ PCR_COOP_INLINE void coop_scan_owner(int lane, uint32_t len, const GridView& g, const SceneView& s,
                                                ScanCache* cache) {
  ScanSlot* ws = g_slots + (threadIdx.x & ~31u);
  const double4* __restrict__ nb_rec = g.nb_rec;
  const double4* __restrict__ nb_pa = g.nb_pa;
  const double4* __restrict__ nb_pb = g.nb_pb;
  const double eps = g.hit_eps;
  const bool fast = PCR_FAST_REJECT && g.fast_reject != 0;
  long long c_num = cache->c_num, c_dn = cache->c_dn;
  double c_t = cache->c_t;
  uint32_t n_march = cache->n_march;
  ScanSlot& me = ws[lane];
  me.best_f = kNoRec;
  me.pre = 0;
  unsigned owners = __ballot_sync(kFull, len > 0);
  const double radius = 2.0 * g.sub_edge;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  __syncwarp();
  while (owners) {
    const int o = __ffs(owners) - 1;
    owners &= owners - 1;
    const uint32_t olen = __shfl_sync(kFull, len, o);
    const ScanSlot& sl = ws[o];
    const V3 pv{sl.prev[0], sl.prev[1], sl.prev[2]}, dv{sl.dir[0], sl.dir[1], sl.dir[2]};
    const V3 pq{sl.pred[0], sl.pred[1], sl.pred[2]};
    const uint32_t j0 = sl.j0;
    double best = 1.7976931348623157e308;
    uint32_t best_f = kNoRec;
    for (uint32_t base = 0; base < olen; base += 32) {
      const uint32_t F = base + lane;
      double t = inf;
      if (F < olen) {
        const uint32_t j = j0 + F;
        const double4 r4 = ldg4(nb_rec + j);
        const double4 pa = ldg4(nb_pa + j);
        const V3 sc = ld3(r4);
        const double rad = pa.w;
        if (norm_le(sc - pq, radius + rad)) {
          ++n_march;  // counts the reference's march_segment call
          const double t_center = dot(sc - pv, dv);
          const double t_lo = smax(0.0, t_center - rad);
          double bt = best;
          if (t_lo < bt) {
            const uint64_t w = static_cast<uint64_t>(__double_as_longlong(r4.w));
            if (__builtin_expect(((w >> 32) & 1u) != 0, 1)) {  // planar records are the common case
              const double4 pb = ldg4(nb_pb + j);
              if (planar_candidate_at(pv, dv, ld3(pa), ld3(pb), eps, t_lo, t_center + rad, bt, c_num, c_dn, c_t,
                                      fast))
                t = bt;
            } else {
              t = march_np(pv.x, pv.y, pv.z, dv.x, dv.y, dv.z, static_cast<uint32_t>(w >> 33), g, s, bt);
            }
          }
        }
      }
      unsigned hit = __ballot_sync(kFull, t < inf);
      if (!hit) continue;
      int win = __ffs(hit) - 1;
      if (hit & (hit - 1)) {  // several hits: (t, lane) min, ties to the lower lane = lower index
        double bt = t;
        int bl = lane;
        for (int off = 16; off > 0; off >>= 1) {
          const double ot = __shfl_xor_sync(kFull, bt, off);
          const int ol = __shfl_xor_sync(kFull, bl, off);
          if (ot < bt || (ot == bt && ol < bl)) {
            bt = ot;
            bl = ol;
          }
        }
        win = bl;
      }
      best = __shfl_sync(kFull, t, win);  // < best of the earlier rounds (pruned against it)
      best_f = base + win;
    }
    if (lane == o) {
      me.best_t = best;
      me.best_f = best_f;
    }
  }
  __syncwarp();
  cache->c_num = c_num;
  cache->c_dn = c_dn;
  cache->c_t = c_t;
  cache->n_march = n_march;
}

#ifndef PCR_SCAN_OWNER
#define PCR_SCAN_OWNER 0
#endif

template <int D, int kMinBlocks>
__global__ void __launch_bounds__(kRefineThreads, kMinBlocks)
    refine_warp_kernel(const __grid_constant__ CandIn in, uint32_t n, const __grid_constant__ GridView g,
                       const __grid_constant__ SceneView s, double delta, int rho, double step_size,
                       const __grid_constant__ RefOut o, uint32_t* next_cand) {
  const int lane = threadIdx.x & 31;
  ScanSlot* ws = g_slots + (threadIdx.x & ~31u);
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  PathState<D> st;
  bool active = false, open = true;
  uint32_t n_trials = 0, n_march = 0;
  unsigned long long n_nodes = 0;  // per lane: iteration nodes << 32 | trial nodes
  ScanCache cache{0x7ff8dead7ff8deadll, 0x7ff8dead7ff8deadll, 0.0, 0u};
  uint32_t done = 0;
  unsigned long long t_start = 0, t_last = 0;
  if (g_refine_dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  for (;;) {
    while (!active && open) {
      const uint32_t idx = atomicAdd(next_cand, 1u);
      if (idx >= n) {
        open = false;
        break;
      }
      active = path_init(st, in.first + (in.order ? in.order[idx] : idx) * in.step, in, s, o);
    }
    if (!__any_sync(kFull, active)) break;
    bool alive = active && path_step_a(st, in, g, s, delta, rho, step_size, o, n_trials, n_nodes);
    // reprojection, front to back (refine.cpp:234-250), node index by node index
    for (int q = 0; q < D; ++q) {
      bool need = alive && q < st.d && st.nd[q].kind == 0;
      if (!__any_sync(kFull, need)) continue;
      uint32_t len = 0;
      bool coop = false;
      Reproj re;
      bool got = false;
      if (need) {
        const V3 prev = q == 0 ? st.tx : node_point(st.nd[q - 1], st.nd[q - 1].p0, st.nd[q - 1].p1);
        const V3 pred = node_point(st.nd[q], st.nd[q].p0, st.nd[q].p1);
        V3 dir{};
        uint32_t j0 = 0;
        const int r = reproject_setup(prev, pred, st.nd[q].label, g, dir, j0, len, st.rc[q]);
        if (r == 1) {
          coop = true;
          ScanSlot& me = ws[lane];
          me.prev[0] = prev.x, me.prev[1] = prev.y, me.prev[2] = prev.z;
          me.dir[0] = dir.x, me.dir[1] = dir.y, me.dir[2] = dir.z;
          me.pred[0] = pred.x, me.pred[1] = pred.y, me.pred[2] = pred.z;
          me.j0 = j0;
          // seed the scan with this node's last winner when it still hits: the scan
          // then evaluates only the records that could beat it (coop_scan)
          me.best_f = kNoRec;
          me.best_t = 1.7976931348623157e308;
          if (PCR_SCAN_SEED && g.seed_scan && st.rc[q].win < len)
            seed_winner(prev, dir, pred, j0, st.rc[q].win, g, s, me);
        } else if (r == 2) {
          got = reproject(prev, pred, st.nd[q].label, g, s, re, n_march);
        }
      }
      if (PCR_SCAN_ILP2)
        coop_scan_ilp2(lane, coop ? len : 0u, g, s, &cache);
      else if (PCR_SCAN_OWNER)
        coop_scan_owner(lane, coop ? len : 0u, g, s, &cache);
      else if (PCR_SCAN_PREFETCH)
        coop_scan_pf(lane, coop ? len : 0u, g, s, &cache);
      else
        coop_scan(lane, coop ? len : 0u, g, s, &cache);
      if (coop) {
        const ScanSlot& me = ws[lane];
        const V3 prev{me.prev[0], me.prev[1], me.prev[2]}, dir{me.dir[0], me.dir[1], me.dir[2]};
        const V3 pred{me.pred[0], me.pred[1], me.pred[2]};
        const uint32_t bf = len ? me.best_f : kNoRec;
        st.rc[q].win = bf != kNoRec ? bf - me.pre : kNoRec;
        if (bf != kNoRec) {
          const double bt = me.best_t;
          const uint32_t ie =
              static_cast<uint32_t>(static_cast<uint64_t>(__double_as_longlong(g.nb_rec[me.j0 + (bf - me.pre)].w)) >> 33);
          if (ie_planar(g, ie)) {  // make_hit's record (surface.cpp:98-106)
            re = Reproj{prev + bt * dir, ld3(g.ie_pn[ie]), g.ie_label[ie]};
          } else {
            SurfaceHit hit;
            march_segment(prev, dir, ie, g, s, inf, &hit);
            re = Reproj{hit.position, hit.normal, g.ie_label[ie]};
          }
          polish(re, ie, g, s);
          got = true;
        } else {
          got = reproject(prev, pred, st.nd[q].label, g, s, re, n_march, 1);
        }
      }
      if (need) {
        if (!got) {
          o.reason[st.k] = PCR_RAY_MISSED;
          o.iters[st.k] = static_cast<uint32_t>(st.iter + 1);
          alive = false;
        } else {
          RNode& x = st.nd[q];
          x.c = re.pos;
          x.n = re.nrm;
          local_frame(re.nrm, x.a, x.b);
          x.p0 = 0.0;
          x.p1 = 0.0;
          x.label = re.label;
        }
      }
    }
    if (alive) alive = path_step_c(st, o);
    if (active && !alive && g_refine_dbg) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_last));
      ++done;
    }
    active = alive;
  }
  if (g_refine_dbg) {  // development trace (PCR_REFINE_TRACE): start, last path's end, paths
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    g_refine_dbg[3 * tid] = t_start;
    g_refine_dbg[3 * tid + 1] = t_last ? t_last : t_start;
    g_refine_dbg[3 * tid + 2] = done;
  }
  atomicAdd(o.stats, static_cast<unsigned long long>(n_trials));
  atomicAdd(o.stats + 1, static_cast<unsigned long long>(n_march + cache.n_march));
  atomicAdd(o.stats + 2, n_nodes & 0xffffffffull);
  atomicAdd(o.stats + 3, n_nodes >> 32);
}

// 3 blocks of 128 threads per SM (168 registers): measured 4 -> 873 ms, 3 -> 686 ms,
// 2 -> 796 ms on C2 (same box)
#ifndef PCR_WARP_MINB
#define PCR_WARP_MINB 3
#endif
constexpr int kWarpMinBlocks = PCR_WARP_MINB;
#ifndef PCR_WARP_MINB_D4
#define PCR_WARP_MINB_D4 4
#endif
constexpr int kWarpMinBlocksD4 = PCR_WARP_MINB_D4;

int refine_mode() {
  static const int m = [] {
    const char* e = std::getenv("PCR_REFINE_MODE");  // 1 = thread per path (A/B aid)
    return e ? std::atoi(e) : 0;
  }();
  return m;
}

// refinement scan records: {sphere centre, label | meta << 32}; flags any IE whose
// sphere radius differs (bitwise) from the first one's
__global__ void refine_records_kernel(GridView g, double4* __restrict__ rr, int* __restrict__ nonuniform) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n_ies) return;
  const double4 sc = g.ie_sc[i];
  const uint64_t lm = static_cast<uint64_t>(g.ie_label[i]) | (static_cast<uint64_t>(g.ie_meta[i]) << 32);
  rr[i] = make_double4(sc.x, sc.y, sc.z, __longlong_as_double(static_cast<long long>(lm)));
  if (__double_as_longlong(sc.w) != __double_as_longlong(g.ie_sc[0].w)) *nonuniform = 1;
}

// neighbourhood lists: count, then fill (cells z->y->x clamped to the grid, surface IEs)
__global__ void nb_count_kernel(GridView g, uint32_t* __restrict__ cnt) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.n_cells) return;
  const int x = static_cast<int>(c % g.dims[0]), y = static_cast<int>((c / g.dims[0]) % g.dims[1]),
            z = static_cast<int>(c / (static_cast<uint32_t>(g.dims[0]) * g.dims[1]));
  uint32_t n = 0;
  for (int zz = max(z - 1, 0); zz <= min(z + 1, g.dims[2] - 1); ++zz)
    for (int yy = max(y - 1, 0); yy <= min(y + 1, g.dims[1] - 1); ++yy)
      for (int xx = max(x - 1, 0); xx <= min(x + 1, g.dims[0] - 1); ++xx) {
        const int4 cell = g.cells[linear_index(g, xx, yy, zz)];
        for (uint32_t i = static_cast<uint32_t>(cell.x); i < static_cast<uint32_t>(cell.y); ++i)
          n += (g.ie_meta[i] & 3u) == kSurface;
      }
  cnt[c] = n;
}
__global__ void nb_fill_kernel(GridView g, const uint32_t* __restrict__ off, double4* __restrict__ rec,
                               uint32_t* __restrict__ lab) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.n_cells) return;
  const int x = static_cast<int>(c % g.dims[0]), y = static_cast<int>((c / g.dims[0]) % g.dims[1]),
            z = static_cast<int>(c / (static_cast<uint32_t>(g.dims[0]) * g.dims[1]));
  uint32_t o = off[c];
  for (int zz = max(z - 1, 0); zz <= min(z + 1, g.dims[2] - 1); ++zz)
    for (int yy = max(y - 1, 0); yy <= min(y + 1, g.dims[1] - 1); ++yy)
      for (int xx = max(x - 1, 0); xx <= min(x + 1, g.dims[0] - 1); ++xx) {
        const int4 cell = g.cells[linear_index(g, xx, yy, zz)];
        for (uint32_t i = static_cast<uint32_t>(cell.x); i < static_cast<uint32_t>(cell.y); ++i) {
          const uint32_t m = g.ie_meta[i];
          if ((m & 3u) != kSurface) continue;
          const double4 sc = g.ie_sc[i];
          const uint64_t w = static_cast<uint64_t>(g.ie_label[i]) | (static_cast<uint64_t>((m >> 2) & 1u) << 32) |
                             (static_cast<uint64_t>(i) << 33);
          rec[o] = make_double4(sc.x, sc.y, sc.z, __longlong_as_double(static_cast<long long>(w)));
          lab[o++] = g.ie_label[i];
        }
      }
  // stable insertion sort of the list by label (lists are a few dozen entries)
  const uint32_t b = off[c];
  for (uint32_t k = b + 1; k < o; ++k) {
    const uint32_t lk = lab[k];
    const double4 rk = rec[k];
    uint32_t m = k;
    while (m > b && lab[m - 1] > lk) {
      lab[m] = lab[m - 1];
      rec[m] = rec[m - 1];
      --m;
    }
    lab[m] = lk;
    rec[m] = rk;
  }
}

// plane of each neighbourhood-list entry, in list order: {plane point, sphere radius},
// {plane normal, 0} (the warp kernel's scan reads them beside the record)
__global__ void nb_geo_kernel(GridView g, uint32_t total, const double4* __restrict__ rec, double4* __restrict__ pa,
                              double4* __restrict__ pb) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= total) return;
  const uint32_t ie = static_cast<uint32_t>(static_cast<uint64_t>(__double_as_longlong(rec[j].w)) >> 33);
  const double4 pp = g.ie_pp[ie], pn = g.ie_pn[ie];
  pa[j] = make_double4(pp.x, pp.y, pp.z, g.rr_uniform ? g.rr_radius : g.ie_sc[ie].w);
  pb[j] = make_double4(pn.x, pn.y, pn.z, 0.0);
}

// The deferred final visibility of converged paths (path_converged): one warp per
// pending candidate, segments tx -> p_0 -> ... -> p_{d-1} -> rx through
// warp_segment_visible (the same predicate as segment_visible, tested bitwise by the
// trace suites); any blocked segment makes the path occluded.
__global__ void __launch_bounds__(128) converged_vis_kernel(const __grid_constant__ CandIn in, uint32_t n_sub,
                                                            const __grid_constant__ GridView g,
                                                            const __grid_constant__ SceneView s,
                                                            const __grid_constant__ RefOut o) {
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n_sub; i += warps) {
    const uint32_t k = in.first + i * in.step;
    if (o.reason[k] != kPendingVis) continue;
    const int d = static_cast<int>(in.n_inter[k]);
    const V3 tx = load3(in.tx + 3ull * k), rx = load3(in.rx + 3ull * k);
    bool visible = true;
    V3 prev = tx;
    for (int q = 0; q <= d && visible; ++q) {
      const V3 next = q < d ? load3(o.pos + 3 * (static_cast<size_t>(k) * in.stride + q)) : rx;
      visible = warp_segment_visible(prev, next, kNoIe, g, s);
      prev = next;
    }
    __syncwarp();
    if (lane == 0) {
      if (visible) {
        o.reason[k] = PCR_NOT_CONVERGED;
      } else {
        o.reason[k] = PCR_OCCLUDED;
        o.has_path[k] = 0;
        for (int q = 0; q < d; ++q) {
          const size_t j = static_cast<size_t>(k) * in.stride + q;
          store3(o.pos + 3 * j, load3(in.pos + 3 * j));
          if (in.kind[j] == 0) {
            store3(o.nrm + 3 * j, load3(in.nrm + 3 * j));
            o.label[j] = in.label[j];
          }
        }
      }
    }
  }
}

// Visiting order of the warp kernel: candidates stably sorted by (depth, diffraction
// mask), so the 32 paths a warp holds at any time mostly share the same node count and
// node kinds — the per-path steps (q < d guards, reflection / diffraction branches, the
// reprojection loop's per-node `need`) then run with full warps. Outcomes are per
// candidate, so the order changes no result; within a class the candidates keep the
// trace's DFS order (spatially coherent neighbourhood lists). Same box, C2 (4/1):
// refine 7.54 s -> 6.93 s (ascending classes) -> 6.90 s (deepest first, the default);
// C2d3 unchanged within noise (profiles/ab_refine_order_r02.log).
__global__ void order_key_kernel(CandIn in, uint32_t n_sub, uint64_t* __restrict__ key) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_sub) return;
  const uint32_t k = in.first + i * in.step;
  const uint32_t d = in.n_inter[k];
  uint32_t mask = 0;
  for (uint32_t q = 0; q < d && q < 8; ++q) mask |= static_cast<uint32_t>(in.kind[static_cast<size_t>(k) * in.stride + q] & 1u) << q;
#ifndef PCR_REFINE_SORT_DEEP_FIRST
#define PCR_REFINE_SORT_DEEP_FIRST 1
#endif
  // deepest classes first: the most expensive paths start early, and the kernel's tail
  // is made of the cheap ones
  const uint32_t dk = PCR_REFINE_SORT_DEEP_FIRST ? 15u - (d < 15 ? d : 15) : (d < 15 ? d : 15);
  key[i] = (static_cast<uint64_t>(dk) << 8) | mask;
}

int rev_order() {
  static const int r = [] {
    const char* e = std::getenv("PCR_REFINE_REV");
    return e ? std::atoi(e) : 0;
  }();
  return r;
}

unsigned nb(uint64_t n, unsigned t) { return static_cast<unsigned>((n + t - 1) / t ? (n + t - 1) / t : 1); }

}  // namespace

void refine_device(Ctx& ctx, const GridDev& grid, const SceneDev& scene, const RefineDevIn& in,
                   const pcr_refine_params& p, RefineDevOut& out) {
  cudaStream_t s = ctx.stream;
  const size_t m = in.n ? in.n : 1;
  const size_t ms = m * in.stride;
  out.reason.alloc(m, s);
  out.has_path.alloc(m, s);
  out.length.alloc(m, s);
  out.delay.alloc(m, s);
  out.gnorm.alloc(m, s);
  out.iters.alloc(m, s);
  out.pos.alloc(3 * ms, s);
  out.nrm.alloc(3 * ms, s);
  out.label.alloc(ms, s);
  // positions/normals/labels start as the candidate's (kinds, ie and edge never change)
  PCR_CUDA(cudaMemcpyAsync(out.pos.get(), in.pos, 3 * ms * sizeof(double), cudaMemcpyDeviceToDevice, s));
  PCR_CUDA(cudaMemcpyAsync(out.nrm.get(), in.nrm, 3 * ms * sizeof(double), cudaMemcpyDeviceToDevice, s));
  PCR_CUDA(cudaMemcpyAsync(out.label.get(), in.label, ms * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  if (!in.n) return;
  const uint32_t step = in.step ? in.step : 1;
  const uint32_t n_sub = in.n > in.first ? (in.n - in.first + step - 1) / step : 0;
  if (!n_sub) return;
  GridView gv = grid.view_for(ctx, scene);
  DBuf<double4> rr(grid.n_ies ? grid.n_ies : 1, s);
  {
    DBuf<int> nonuni(1, s);
    PCR_CUDA(cudaMemsetAsync(nonuni.get(), 0, sizeof(int), s));
    if (grid.n_ies) {
      count_launch();
      refine_records_kernel<<<nb(grid.n_ies, 256), 256, 0, s>>>(gv, rr.get(), nonuni.get());
      PCR_LAUNCH_CHECK();
    }
    int h = 0;
    d2h(&h, nonuni.get(), 1, s);
    double r0 = 0.0;
    if (grid.n_ies) d2h(&r0, &grid.sc.get()->w, 1, s);
    stream_wait(s);
    gv.ie_rr = rr.get();
    gv.rr_uniform = grid.n_ies && !h;
    gv.rr_radius = r0;
  }
  {
    // planar_candidate_at's fast rejection: prev, pp and the window lie in the grid box
    // (nodes are reprojected onto IEs inside it; TX/RX are inside scene_bounds), so
    // |prev| + |pp| + |t| <= 2 R + diam with R the farthest box corner from the origin;
    // its rounding bound 30 u (2 R + diam) must stay 4x below kMarginFast
    double r2 = 0.0, d2 = 0.0;
    for (int a = 0; a < 3; ++a) {
      const double lo = (&grid.origin.x)[a], hi = lo + grid.dims[a] * grid.voxel_size;
      const double m = std::fabs(lo) > std::fabs(hi) ? std::fabs(lo) : std::fabs(hi);
      r2 += m * m;
      d2 += (hi - lo) * (hi - lo);
    }
    const double extent = 2.0 * std::sqrt(r2) + std::sqrt(d2) + 1.0;
    gv.fast_reject = 4.0 * 30.0 * 1.1102230246251565e-16 * extent < kMarginFast ? 1 : 0;
    gv.seed_scan = PCR_SCAN_SEED ? 1 : 0;
  }
  // neighbourhood lists (the reprojection box is a cell's 3x3x3 neighbourhood whenever
  // 2 * subvoxel_edge spans exactly one voxel each way, i.e. division_factor 2)
  DBuf<uint32_t> nb_off, nb_lab;
  DBuf<double4> nb_rec, nb_pa, nb_pb;
  if (grid.n_cells && grid.n_ies && grid.n_ies < (1ull << 31) && grid.n_cells < (1ull << 31)) {
    const uint32_t nc = static_cast<uint32_t>(grid.n_cells);
    DBuf<uint32_t> cnt(nc, s), tot(1, s);
    nb_off.alloc(nc + 1ull, s);
    count_launch();
    nb_count_kernel<<<nb(nc, 256), 256, 0, s>>>(gv, cnt.get());
    PCR_LAUNCH_CHECK();
    exclusive_scan_u32(cnt.get(), nb_off.get(), nc, nb_off.get() + nc, s);
    uint32_t total = 0;
    d2h(&total, nb_off.get() + nc, 1, s);
    stream_wait(s);
    nb_rec.alloc(total ? total : 1, s);
    nb_lab.alloc(total ? total : 1, s);
    count_launch();
    nb_fill_kernel<<<nb(nc, 256), 256, 0, s>>>(gv, nb_off.get(), nb_rec.get(), nb_lab.get());
    PCR_LAUNCH_CHECK();
    nb_pa.alloc(total ? total : 1, s);
    nb_pb.alloc(total ? total : 1, s);
    if (total) {
      count_launch();
      nb_geo_kernel<<<nb(total, 256), 256, 0, s>>>(gv, total, nb_rec.get(), nb_pa.get(), nb_pb.get());
      PCR_LAUNCH_CHECK();
    }
    gv.nb_off = nb_off.get();
    gv.nb_rec = nb_rec.get();
    gv.nb_lab = nb_lab.get();
    gv.nb_pa = nb_pa.get();
    gv.nb_pb = nb_pb.get();
  }
  CandIn ci{in.first, step, in.stride, in.tx, in.rx, in.n_inter, in.kind, in.pos, in.label, in.nrm, in.edge, in.coarse_length,
            nullptr};
#ifndef PCR_REFINE_SORT
#define PCR_REFINE_SORT 1
#endif
  DBuf<uint32_t> order;
  if (PCR_REFINE_SORT && refine_mode() == 0 && n_sub > 1) {
    DBuf<uint64_t> key(n_sub, s);
    order.alloc(n_sub, s);
    count_launch();
    order_key_kernel<<<nb(n_sub, 256), 256, 0, s>>>(ci, n_sub, key.get());
    PCR_LAUNCH_CHECK();
    iota_u32(order.get(), n_sub, s);
    radix_sort_pairs(key.get(), order.get(), n_sub, 0, 12, s);
    ci.order = order.get();
  }
  DBuf<unsigned long long> stats(4, s);
  DBuf<uint32_t> next(1, s);
  PCR_CUDA(cudaMemsetAsync(next.get(), 0, sizeof(uint32_t), s));
  PCR_CUDA(cudaMemsetAsync(stats.get(), 0, 4 * sizeof(unsigned long long), s));
  RefOut ro{out.reason.get(), out.has_path.get(), out.pos.get(), out.nrm.get(), out.label.get(),
            out.length.get(), out.delay.get(), out.gnorm.get(), out.iters.get(), stats.get()};
  count_launch();
  {
    KTimer kt(ctx, "refine");
    const char* trace = std::getenv("PCR_REFINE_TRACE");
    // enough resident threads to fill every SM at the kernel's occupancy
    int per_sm = 0;
    // depth bound of this batch: the smallest instantiation that holds its stride.
    // Default: the warp-cooperative kernel; PCR_REFINE_MODE=1 selects the thread-per-path
    // kernel (4 blocks of 128 threads per SM, 128 registers), kept as the A/B baseline.
    const bool warp = refine_mode() == 0;
#ifndef PCR_REFINE_D4
#define PCR_REFINE_D4 1
#endif
    // depth bounds 3, 4 (the contract C2: max_interactions 4), 5 and 8
    // depth 4 (the contract C2) at 4 blocks/SM (128 registers): C2 refine 6.57-6.62 s ->
    // 6.47-6.49 s, while depth 3 prefers 3 (541-580 vs 592-637 ms), same box
    // (profiles/ab_minblocks_r02.log)
    auto kern = in.stride <= 3                      ? refine_warp_kernel<3, kWarpMinBlocks>
                : (PCR_REFINE_D4 && in.stride <= 4) ? refine_warp_kernel<4, kWarpMinBlocksD4>
                : in.stride <= 5                    ? refine_warp_kernel<5, kWarpMinBlocks>
                                                    : refine_warp_kernel<kMaxDepth, kWarpMinBlocks>;
    auto kern2 = in.stride <= 3 ? refine_kernel<3, 4> : in.stride <= 5 ? refine_kernel<5, 4> : refine_kernel<kMaxDepth, 4>;
    // shared-memory carveout: the kernel needs 3 x 13.4 KB (scan slots), and the driver's
    // own choice for it was the 100 KB configuration (ncu launch__shared_mem_config_size
    // 102.4 KB), leaving L1 short for the per-lane path state. A 25 % hint selects the
    // 64 KB configuration: C2d3 refine 620 -> 608 ms, C2 7.60 -> 7.43 s (same box,
    // profiles/ab_carveout_r02.log); 0 % starves occupancy (1.10 s), 60 % is slower.
#ifndef PCR_REFINE_CARVEOUT
#define PCR_REFINE_CARVEOUT 25
#endif
    if (warp && PCR_REFINE_CARVEOUT >= 0)
      PCR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, PCR_REFINE_CARVEOUT));
    if (warp)
      PCR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRefineThreads, 0));
    else
      PCR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern2, kRefineThreads, 0));
    const uint64_t want = (static_cast<uint64_t>(n_sub) + kRefineThreads - 1) / kRefineThreads;
    const uint64_t cap = static_cast<uint64_t>(ctx.sm_count) * (per_sm > 0 ? per_sm : 1);
    const unsigned grid_n = static_cast<unsigned>(want < cap ? want : cap);
    DBuf<unsigned long long> dbg;
    unsigned long long t0 = 0;
    if (trace) {
      dbg.alloc(3ull * grid_n * kRefineThreads, s);
      PCR_CUDA(cudaMemsetAsync(dbg.get(), 0, 24ull * grid_n * kRefineThreads, s));
      unsigned long long* p = dbg.get();
      PCR_CUDA(cudaMemcpyToSymbolAsync(g_refine_dbg, &p, sizeof(p), 0, cudaMemcpyHostToDevice, s));
      stream_wait(s);
      t0 = static_cast<unsigned long long>(std::chrono::duration_cast<std::chrono::nanoseconds>(
          std::chrono::system_clock::now().time_since_epoch()).count());
    }
    if (warp) {
      kern<<<grid_n, kRefineThreads, 0, s>>>(ci, n_sub, gv, scene.view(), p.delta, p.rho, p.step_size, ro, next.get());
      if (PCR_DEFER_VIS) {
        PCR_LAUNCH_CHECK();
        count_launch();
        converged_vis_kernel<<<static_cast<unsigned>(ctx.sm_count) * 16u, 128, 0, s>>>(ci, n_sub, gv, scene.view(), ro);
      }
    }
    else
      kern2<<<grid_n, kRefineThreads, 0, s>>>(
          ci, n_sub, gv, scene.view(), p.delta, p.rho, p.step_size, ro, next.get(), rev_order());
    if (trace) {
      std::vector<unsigned long long> h(3ull * grid_n * kRefineThreads);
      d2h(h.data(), dbg.get(), h.size(), s);
      stream_wait(s);
      unsigned long long* z = nullptr;
      PCR_CUDA(cudaMemcpyToSymbol(g_refine_dbg, &z, sizeof(z)));
      if (FILE* f = std::fopen(trace, "wb")) {
        std::fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
        std::fclose(f);
      }
      // per-candidate iterations, depth, kinds, reason (for cost predictors)
      std::vector<uint32_t> it(in.n), ni(in.n);
      std::vector<int32_t> rs(in.n);
      std::vector<uint8_t> kd(static_cast<size_t>(in.n) * in.stride);
      d2h(it.data(), out.iters.get(), in.n, s);
      d2h(rs.data(), out.reason.get(), in.n, s);
      d2h(ni.data(), in.n_inter, in.n, s);
      d2h(kd.data(), in.kind, kd.size(), s);
      stream_wait(s);
      if (FILE* f = std::fopen((std::string(trace) + ".cand").c_str(), "wb")) {
        for (uint32_t i = 0; i < in.n; ++i) {
          uint32_t kinds = 0;
          for (uint32_t q = 0; q < ni[i] && q < in.stride; ++q) kinds |= (kd[static_cast<size_t>(i) * in.stride + q] & 1u) << q;
          const uint32_t row[4] = {it[i], ni[i], kinds, static_cast<uint32_t>(rs[i])};
          std::fwrite(row, sizeof(uint32_t), 4, f);
        }
        std::fclose(f);
      }
      (void)t0;
    }
  }
  PCR_LAUNCH_CHECK();
  unsigned long long hs[4];
  d2h(hs, stats.get(), 4, s);
  stream_wait(s);
  out.trials = hs[0];
  out.marches = hs[1];
  out.trial_nodes = hs[2];
  out.iter_nodes = hs[3];
}

void api_refine_batch(Ctx& ctx, const GridDev& grid, const SceneDev& scene, const pcr_paths& c,
                      const pcr_refine_params& p, pcr_outcomes** out) {
  cudaStream_t s = ctx.stream;
  const size_t n = c.n, st = c.stride ? c.stride : 1;
  const size_t m = n ? n : 1, ms = m * st;
  DBuf<double> tx(3 * m, s), rx(3 * m, s), pos(3 * ms, s), nrm(3 * ms, s), cl(m, s);
  DBuf<uint32_t> ni(m, s), lab(ms, s), edge(ms, s);
  DBuf<uint8_t> kind(ms, s);
  h2d(tx.get(), c.tx_position, 3 * n, s);
  h2d(rx.get(), c.rx_position, 3 * n, s);
  h2d(pos.get(), c.position, 3 * n * st, s);
  h2d(nrm.get(), c.normal, 3 * n * st, s);
  h2d(cl.get(), c.length, n, s);
  h2d(ni.get(), c.n_inter, n, s);
  h2d(lab.get(), c.label, n * st, s);
  h2d(edge.get(), c.edge_index, n * st, s);
  h2d(kind.get(), c.kind, n * st, s);
  for (size_t i = 0; i < n; ++i)
    if (c.n_inter[i] > st || c.n_inter[i] > static_cast<uint32_t>(kMaxDepth))
      throw Error(1, "refine: path longer than its stride");
  RefineDevIn in{static_cast<uint32_t>(n), static_cast<uint32_t>(st), tx.get(), rx.get(), pos.get(), nrm.get(),
                 cl.get(), ni.get(), lab.get(), edge.get(), kind.get()};
  RefineDevOut ro;
  refine_device(ctx, grid, scene, in, p, ro);
  pcr_outcomes* o = halloc<pcr_outcomes>(1);
  pcr_paths* pp = alloc_paths(n, static_cast<uint32_t>(st));
  o->paths = *pp;
  std::free(pp);
  o->has_path = halloc<uint8_t>(n);
  o->reason = halloc<int32_t>(n);
  std::vector<double> rpos(3 * n * st), rnrm(3 * n * st), len(n), del(n), gn(n);
  std::vector<uint32_t> rlab(n * st);
  d2h(o->has_path, ro.has_path.get(), n, s);
  d2h(o->reason, ro.reason.get(), n, s);
  d2h(rpos.data(), ro.pos.get(), rpos.size(), s);
  d2h(rnrm.data(), ro.nrm.get(), rnrm.size(), s);
  d2h(rlab.data(), ro.label.get(), rlab.size(), s);
  d2h(len.data(), ro.length.get(), n, s);
  d2h(del.data(), ro.delay.get(), n, s);
  d2h(gn.data(), ro.gnorm.get(), n, s);
  stream_wait(s);
  pcr_paths& P = o->paths;
  for (size_t i = 0; i < n; ++i) {
    if (!o->has_path[i]) continue;
    P.tx_id[i] = c.tx_id[i];
    P.rx_id[i] = c.rx_id[i];
    std::memcpy(P.tx_position + 3 * i, c.tx_position + 3 * i, 3 * sizeof(double));
    std::memcpy(P.rx_position + 3 * i, c.rx_position + 3 * i, 3 * sizeof(double));
    P.length[i] = len[i];
    P.delay[i] = del[i];
    P.converged[i] = 1;
    P.gradient_norm[i] = gn[i];
    P.n_inter[i] = c.n_inter[i];
    for (uint32_t q = 0; q < c.n_inter[i]; ++q) {
      const size_t j = i * st + q;
      P.kind[j] = c.kind[j];
      std::memcpy(P.position + 3 * j, &rpos[3 * j], 3 * sizeof(double));
      P.label[j] = rlab[j];
      std::memcpy(P.normal + 3 * j, &rnrm[3 * j], 3 * sizeof(double));
      P.ie_index[j] = c.ie_index[j];
      P.edge_index[j] = c.edge_index[j];
    }
  }
  *out = o;
}

}  // namespace pcr
