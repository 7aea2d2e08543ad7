// voxelize.cu — stage 1: build_grid (proj/src/voxel_grid.cpp:82-227) and
// compute_march_distances (voxel_grid.cpp:229-268) on the device.
//
// Pipeline (all device-resident; host only sizes allocations):
//   K1 bounds_kernel        min/max of point positions + max label (order-free, exact)
//   K2 bin_kernel           per point: global subvoxel lattice -> (voxel, subvoxel) key
//   K3 radix_sort_pairs     stable LSD sort of (voxel, subvoxel, label) with point index values
//   K4 head_kernel + scan   run heads -> SurfacePoints IE ids
//   K5 surface_ie_kernel    warp per IE: planar flag + centroid summed sequentially in
//                           point_indices order (the sum order is the parity contract)
//   K6 edge_*_kernel        edge clipping against the subvoxel lattice (3-way merge of
//                           the per-axis monotone cut sequences = std::sort of the cuts)
//   K7 extra_rank_kernel    canonical order of edge pieces + receivers (few); merged
//                           with the already-sorted surface IEs by binary search
//   K8 scatter + cells      final SoA IE records, per-voxel [ie_begin, ie_end)
//   K9 dt_*_kernel          exact Chebyshev transform as three separable min-max passes
#include <algorithm>
#include <cmath>
#include <limits>
#include <stdexcept>
#include <vector>

#include "device_state.cuh"
#include "sort.cuh"

namespace pcr {
namespace {

constexpr int kThreads = 256;

// ---------------------------------------------------------------------------------
// K1: bounds over points + max label. Per-block partials, host finishes (tiny).
struct BoundsPartial {
  double mn[3], mx[3];
  uint32_t max_label;
};

__global__ void bounds_kernel(const double* __restrict__ pos, const uint32_t* __restrict__ label, uint64_t n,
                              BoundsPartial* __restrict__ out) {
  double mn[3] = {1.7976931348623157e308, 1.7976931348623157e308, 1.7976931348623157e308};
  double mx[3] = {-1.7976931348623157e308, -1.7976931348623157e308, -1.7976931348623157e308};
  uint32_t ml = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double p = pos[3 * i + a];
      mn[a] = smin(mn[a], p);
      mx[a] = smax(mx[a], p);
    }
    ml = max(ml, label[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      mn[a] = smin(mn[a], __shfl_down_sync(0xffffffffu, mn[a], o));
      mx[a] = smax(mx[a], __shfl_down_sync(0xffffffffu, mx[a], o));
    }
    ml = max(ml, __shfl_down_sync(0xffffffffu, ml, o));
  }
  __shared__ BoundsPartial sh[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    for (int a = 0; a < 3; ++a) {
      sh[wid].mn[a] = mn[a];
      sh[wid].mx[a] = mx[a];
    }
    sh[wid].max_label = ml;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    BoundsPartial r = sh[0];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
      for (int a = 0; a < 3; ++a) {
        r.mn[a] = smin(r.mn[a], sh[w].mn[a]);
        r.mx[a] = smax(r.mx[a], sh[w].mx[a]);
      }
      r.max_label = max(r.max_label, sh[w].max_label);
    }
    out[blockIdx.x] = r;
  }
}

// locate_subvoxel + local_linear (voxel_grid.cpp:19-34)
struct Lattice {
  double ox, oy, oz, se;
  int dims[3];
  int dv;
};

__device__ __forceinline__ void locate(const Lattice& L, const V3& p, uint32_t& voxel, uint32_t& sub) {
  const double pc[3] = {p.x, p.y, p.z};
  const double oc[3] = {L.ox, L.oy, L.oz};
  int vox[3], loc[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    int g = static_cast<int>(floor((pc[a] - oc[a]) / L.se));
    const int g_max = L.dims[a] * L.dv - 1;
    g = sclamp(g, 0, g_max);
    vox[a] = g / L.dv;
    loc[a] = g - vox[a] * L.dv;
  }
  voxel = static_cast<uint32_t>(vox[0] + L.dims[0] * (vox[1] + L.dims[1] * vox[2]));
  sub = static_cast<uint32_t>(loc[0] + L.dv * (loc[1] + L.dv * loc[2]));
}

// K2: keys. packed = (voxel << sub_bits | sub) << label_bits | label  when it fits,
// else the (voxel, sub) part alone (label sorted by a preceding stable pass).
__global__ void bin_kernel(Lattice L, const double* __restrict__ pos, const uint32_t* __restrict__ label,
                           const uint32_t* __restrict__ perm, uint64_t n, int sub_bits, int label_bits,
                           bool with_label, uint64_t* __restrict__ key) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t pi = perm ? perm[i] : i;
    uint32_t voxel, sub;
    locate(L, V3{pos[3 * pi], pos[3 * pi + 1], pos[3 * pi + 2]}, voxel, sub);
    uint64_t k = (static_cast<uint64_t>(voxel) << sub_bits) | sub;
    if (with_label) k = (k << label_bits) | label[pi];
    key[i] = k;
  }
}

// Sharded voxelization: voxel of every point, for the per-voxel point
// histogram (splitters) and the shard's point filter
__global__ void voxel_of_kernel(Lattice L, const double* __restrict__ pos, uint64_t n, uint32_t* __restrict__ vox) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint32_t v, s;
    locate(L, V3{pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]}, v, s);
    vox[i] = v;
  }
}
__global__ void voxel_hist_kernel(const uint32_t* __restrict__ vox, uint64_t n, uint32_t* __restrict__ hist) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    atomicAdd(hist + vox[i], 1u);
}
__global__ void in_range_kernel(const uint32_t* __restrict__ vox, uint64_t n, uint32_t lo, uint32_t hi,
                                uint32_t* __restrict__ flag) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    flag[i] = vox[i] >= lo && vox[i] < hi;
}
// the shard's point ids, ascending (a stable compaction keeps the reference's tie order)
__global__ void compact_ids_kernel(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos, uint64_t n,
                                   uint32_t* __restrict__ ids) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    if (flag[i]) ids[pos[i]] = static_cast<uint32_t>(i);
}

__global__ void gather_label_key_kernel(const uint32_t* __restrict__ label, const uint32_t* __restrict__ perm,
                                        uint64_t n, uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = label[perm[i]];
}

// after the sorts: split the sorted key into (voxel/sub key, label)
__global__ void unpack_kernel(const uint64_t* __restrict__ skey, const uint32_t* __restrict__ sidx,
                              const uint32_t* __restrict__ label, uint64_t n, int label_bits, bool with_label,
                              uint64_t* __restrict__ vs_key, uint32_t* __restrict__ slabel) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = skey[i];
    if (with_label) {
      vs_key[i] = k >> label_bits;
      slabel[i] = static_cast<uint32_t>(k & ((label_bits >= 64) ? ~0ull : ((1ull << label_bits) - 1ull)));
    } else {
      vs_key[i] = k;
      slabel[i] = label[sidx[i]];
    }
  }
}

// K4: run heads of (voxel, sub, label)
__global__ void head_kernel(const uint64_t* __restrict__ vs_key, const uint32_t* __restrict__ slabel, uint64_t n,
                            uint32_t* __restrict__ head) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    head[i] = (i == 0 || vs_key[i] != vs_key[i - 1] || slabel[i] != slabel[i - 1]) ? 1u : 0u;
}

__global__ void starts_kernel(const uint32_t* __restrict__ head, const uint32_t* __restrict__ ie_id, uint64_t n,
                              uint32_t* __restrict__ starts) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    if (head[i]) starts[ie_id[i]] = static_cast<uint32_t>(i);
}

// K5: one warp per SurfacePoints IE (voxel_grid.cpp:128-157 + reception_point_of :64-69).
struct SurfaceTmp {
  uint64_t* vs_key;  // per IE (voxel << sub_bits | sub)
  uint32_t* label;
  uint2* range;
  double4* centroid;
  double4* pp;
  double4* pn;
  uint32_t* planar;
};

__global__ void surface_ie_kernel(const uint64_t* __restrict__ vs_key, const uint32_t* __restrict__ slabel,
                                  const uint32_t* __restrict__ sidx, const uint32_t* __restrict__ starts,
                                  uint32_t n_ie, uint64_t n_pts, const double* __restrict__ pos,
                                  const double* __restrict__ nrm, SurfaceTmp t) {
  const int lane = threadIdx.x & 31;
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  // the round's positions staged per warp; lanes 0, 1, 2 then run the x, y and z sums,
  // each sequential in point_indices order
  __shared__ double stage[kThreads / 32][32][3];
  double (*buf)[3] = stage[threadIdx.x >> 5];
  for (uint32_t ie = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; ie < n_ie; ie += warps) {
    const uint32_t b = starts[ie];
    const uint32_t e = (ie + 1 < n_ie) ? starts[ie + 1] : static_cast<uint32_t>(n_pts);
    const uint32_t first = sidx[b];
    const V3 p0 = load3(pos + 3ull * first);
    const V3 n0 = load3(nrm + 3ull * first);
    bool planar = true;
    V3 sum{0.0, 0.0, 0.0};
    for (uint32_t base = b; base < e; base += 32) {
      const uint32_t k = base + lane;
      V3 p{0, 0, 0};
      bool bad = false;
      if (k < e) {
        const uint32_t pi = sidx[k];
        p = load3(pos + 3ull * pi);
        const V3 n = load3(nrm + 3ull * pi);
        bad = dot(n, n0) < 1.0 - 1e-12 || fabs(dot(p - p0, n0)) > 1e-9;
      }
      if (__any_sync(0xffffffffu, bad)) planar = false;
      const uint32_t cnt = min(32u, e - base);
      buf[lane][0] = p.x;
      buf[lane][1] = p.y;
      buf[lane][2] = p.z;
      __syncwarp();
      if (lane < 3) {
        double acc = lane == 0 ? sum.x : lane == 1 ? sum.y : sum.z;
        for (uint32_t j = 0; j < cnt; ++j) acc += buf[j][lane];
        if (lane == 0) sum.x = acc;
        else if (lane == 1) sum.y = acc;
        else sum.z = acc;
      }
      __syncwarp();
    }
    sum.y = __shfl_sync(0xffffffffu, sum.y, 1);
    sum.z = __shfl_sync(0xffffffffu, sum.z, 2);
    if (lane == 0) {
      const V3 c = sum / static_cast<double>(e - b);
      t.vs_key[ie] = vs_key[b];
      t.label[ie] = slabel[b];
      t.range[ie] = make_uint2(b, e);
      t.centroid[ie] = make_double4(c.x, c.y, c.z, 0.0);
      t.pp[ie] = make_double4(p0.x, p0.y, p0.z, 0.0);
      t.pn[ie] = make_double4(n0.x, n0.y, n0.z, 0.0);
      t.planar[ie] = planar ? 1u : 0u;
    }
  }
}

// K6: edge clipping (voxel_grid.cpp:160-195).
struct ExtraIE {
  uint64_t vs_key;  // voxel << sub_bits | sub
  uint32_t voxel, sub, kind, label, edge, rx;
  double ss[3], se[3];  // seg_start, seg_end
};

struct AxisCuts {
  bool on;
  int k, k_end, kstep;
};

__device__ __forceinline__ double cut_t(const Lattice& L, const double* start, const double* dir, int a, int k) {
  const double o = a == 0 ? L.ox : (a == 1 ? L.oy : L.oz);
  return ((o + static_cast<double>(k) * L.se) - start[a]) / dir[a];
}

// Streams the sorted cut list {0, len, filtered lattice crossings} of one edge and
// calls emit(t0, t1) for every kept piece; returns the piece count.
template <typename Emit>
__device__ uint32_t clip_edge(const Lattice& L, const double* g, Emit emit) {
  const V3 s = load3(g), en = load3(g + 3);
  const double len = norm(en - s);
  if (!(len > 0.0)) return 0;
  const V3 dv3 = (en - s) / len;
  const double start[3] = {s.x, s.y, s.z};
  const double dir[3] = {dv3.x, dv3.y, dv3.z};
  const double endp[3] = {en.x, en.y, en.z};
  const double oc[3] = {L.ox, L.oy, L.oz};
  AxisCuts ax[3];
  for (int a = 0; a < 3; ++a) {
    ax[a].on = !(fabs(dir[a]) < 1e-15);
    if (!ax[a].on) continue;
    const double lo = smin(start[a], endp[a]);
    const double hi = smax(start[a], endp[a]);
    const int k_lo = static_cast<int>(ceil((lo - oc[a]) / L.se));
    const int k_hi = static_cast<int>(floor((hi - oc[a]) / L.se));
    if (k_lo > k_hi) {
      ax[a].on = false;
      continue;
    }
    // t is monotone in k: ascending for dir > 0, descending for dir < 0
    if (dir[a] > 0) {
      ax[a].k = k_lo;
      ax[a].k_end = k_hi + 1;
      ax[a].kstep = 1;
    } else {
      ax[a].k = k_hi;
      ax[a].k_end = k_lo - 1;
      ax[a].kstep = -1;
    }
  }
  auto head = [&](int a, double& t) -> bool {
    while (ax[a].on && ax[a].k != ax[a].k_end) {
      t = cut_t(L, start, dir, a, ax[a].k);
      if (t > 1e-12 && t < len - 1e-12) return true;
      ax[a].k += ax[a].kstep;
    }
    return false;
  };
  uint32_t pieces = 0;
  double prev = 0.0;
  for (;;) {
    double best = 0.0;
    int ba = -1;
    for (int a = 0; a < 3; ++a) {
      double t;
      if (head(a, t) && (ba < 0 || t < best)) {
        best = t;
        ba = a;
      }
    }
    const double cur = ba < 0 ? len : best;
    if (ba >= 0) ax[ba].k += ax[ba].kstep;
    if (!(cur - prev < 1e-12)) {
      emit(prev, cur, s, dv3, pieces);
      ++pieces;
    }
    prev = cur;
    if (ba < 0) break;
  }
  return pieces;
}

__global__ void edge_count_kernel(Lattice L, const double* __restrict__ edges, uint32_t n_edges,
                                  uint32_t* __restrict__ count) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_edges) return;
  count[e] = clip_edge(L, edges + 12ull * e, [](double, double, const V3&, const V3&, uint32_t) {});
}

__global__ void edge_emit_kernel(Lattice L, const double* __restrict__ edges, const uint32_t* __restrict__ elabel,
                                 uint32_t n_edges, const uint32_t* __restrict__ offset, int sub_bits,
                                 ExtraIE* __restrict__ out) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_edges) return;
  const uint32_t base = offset[e];
  const uint32_t lab = elabel[e];
  clip_edge(L, edges + 12ull * e, [&](double t0, double t1, const V3& s, const V3& d, uint32_t k) {
    const V3 a = s + t0 * d;
    const V3 b = s + t1 * d;
    uint32_t voxel, sub;
    locate(L, 0.5 * (a + b), voxel, sub);
    ExtraIE x;
    x.voxel = voxel;
    x.sub = sub;
    x.vs_key = (static_cast<uint64_t>(voxel) << sub_bits) | sub;
    x.kind = kEdge;
    x.label = lab;
    x.edge = e;
    x.rx = 0;
    x.ss[0] = a.x;
    x.ss[1] = a.y;
    x.ss[2] = a.z;
    x.se[0] = b.x;
    x.se[1] = b.y;
    x.se[2] = b.z;
    out[base + k] = x;
  });
}

// K7a: receivers (voxel_grid.cpp:197-208)
__global__ void rx_kernel(Lattice L, const double* __restrict__ rx_pos, const uint32_t* __restrict__ rx_id,
                          uint32_t n_rx, int sub_bits, ExtraIE* __restrict__ out) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rx) return;
  uint32_t voxel, sub;
  locate(L, load3(rx_pos + 3ull * r), voxel, sub);
  ExtraIE x;
  x.voxel = voxel;
  x.sub = sub;
  x.vs_key = (static_cast<uint64_t>(voxel) << sub_bits) | sub;
  x.kind = kReceiver;
  x.label = rx_id[r];
  x.edge = 0;
  x.rx = rx_id[r];
  for (int a = 0; a < 3; ++a) x.ss[a] = x.se[a] = 0.0;
  out[r] = x;
}

__global__ void extract_keys_kernel(const ExtraIE* __restrict__ ex, uint32_t n, uint64_t* __restrict__ keys) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) keys[r] = ex[r].vs_key;
}

// canonical_ie_less (voxel_grid.cpp:50-57)
__device__ __forceinline__ bool canon_less(const ExtraIE& a, const ExtraIE& b) {
  if (a.voxel != b.voxel) return a.voxel < b.voxel;
  if (a.sub != b.sub) return a.sub < b.sub;
  if (a.kind != b.kind) return a.kind < b.kind;
  if (a.label != b.label) return a.label < b.label;
  if (a.edge != b.edge) return a.edge < b.edge;
  if (a.rx != b.rx) return a.rx < b.rx;
  if (a.ss[0] != b.ss[0]) return a.ss[0] < b.ss[0];
  if (a.ss[1] != b.ss[1]) return a.ss[1] < b.ss[1];
  return a.ss[2] < b.ss[2];
}

// K7b: rank of each extra IE in canonical order (ties by input index; tied records are identical)
__global__ void extra_rank_kernel(const ExtraIE* __restrict__ in, uint32_t n, ExtraIE* __restrict__ out) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const ExtraIE me = in[e];
  uint32_t r = 0;
  for (uint32_t f = 0; f < n; ++f) {
    const ExtraIE o = in[f];
    if (canon_less(o, me) || (f < e && !canon_less(me, o))) ++r;
  }
  out[r] = me;
}

__device__ __forceinline__ uint32_t lower_bound_u64(const uint64_t* a, uint32_t n, uint64_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t m = (lo + hi) >> 1;
    if (a[m] < x) lo = m + 1;
    else hi = m;
  }
  return lo;
}
__device__ __forceinline__ uint32_t upper_bound_u64(const uint64_t* a, uint32_t n, uint64_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t m = (lo + hi) >> 1;
    if (a[m] <= x) lo = m + 1;
    else hi = m;
  }
  return lo;
}

struct FinalOut {
  uint32_t *meta, *label, *edge, *rx, *voxel, *sub;
  double4 *sc, *rp, *pp, *pn, *seg_s, *seg_e;
  uint2* range;
};

// subvoxel_center (voxel_grid.cpp:36-48)
__device__ __forceinline__ double4 subvoxel_center(const Lattice& L, double vs, uint32_t voxel, uint32_t sub,
                                                   double radius) {
  const int dx = L.dims[0], dy = L.dims[1], dv = L.dv;
  const int v[3] = {static_cast<int>(voxel) % dx, (static_cast<int>(voxel) / dx) % dy,
                    static_cast<int>(voxel) / (dx * dy)};
  const int l[3] = {static_cast<int>(sub) % dv, (static_cast<int>(sub) / dv) % dv, static_cast<int>(sub) / (dv * dv)};
  const double o[3] = {L.ox, L.oy, L.oz};
  double c[3];
  for (int a = 0; a < 3; ++a)
    c[a] = (o[a] + static_cast<double>(v[a]) * vs) + (static_cast<double>(l[a]) + 0.5) * L.se;
  return make_double4(c[0], c[1], c[2], radius);
}

// K8a: surface IEs to their canonical slot
__global__ void scatter_surface_kernel(Lattice L, double vs, double radius, SurfaceTmp t, uint32_t n_surf,
                                       const uint64_t* __restrict__ extra_keys, uint32_t n_extra, int sub_bits,
                                       FinalOut o) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n_surf; s += gridDim.x * blockDim.x) {
    const uint64_t k = t.vs_key[s];
    const uint32_t pos = s + lower_bound_u64(extra_keys, n_extra, k);
    const uint32_t voxel = static_cast<uint32_t>(k >> sub_bits);
    const uint32_t sub = static_cast<uint32_t>(k & ((1ull << sub_bits) - 1ull));
    o.meta[pos] = kSurface | (t.planar[s] << 2);
    o.label[pos] = t.label[s];
    o.edge[pos] = 0;
    o.rx[pos] = 0;
    o.voxel[pos] = voxel;
    o.sub[pos] = sub;
    o.sc[pos] = subvoxel_center(L, vs, voxel, sub, radius);
    o.rp[pos] = t.centroid[s];
    if (t.planar[s]) {
      o.pp[pos] = t.pp[s];
      o.pn[pos] = t.pn[s];
    } else {
      // IntersectableEntity keeps the first point's plane even when not planar
      o.pp[pos] = t.pp[s];
      o.pn[pos] = t.pn[s];
    }
    o.seg_s[pos] = make_double4(0, 0, 0, 0);
    o.seg_e[pos] = make_double4(0, 0, 0, 0);
    o.range[pos] = t.range[s];
  }
}

// K8b: extra IEs (sorted) to their canonical slot
__global__ void scatter_extra_kernel(Lattice L, double vs, double radius, const ExtraIE* __restrict__ ex,
                                     uint32_t n_extra, const uint64_t* __restrict__ surf_keys, uint32_t n_surf,
                                     const double* __restrict__ rx_pos, const uint32_t* __restrict__ rx_id,
                                     uint32_t n_rx, FinalOut o) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_extra) return;
  const ExtraIE x = ex[r];
  const uint32_t pos = r + upper_bound_u64(surf_keys, n_surf, x.vs_key);
  o.meta[pos] = x.kind;
  o.label[pos] = x.label;
  o.edge[pos] = x.edge;
  o.rx[pos] = x.rx;
  o.voxel[pos] = x.voxel;
  o.sub[pos] = x.sub;
  o.sc[pos] = subvoxel_center(L, vs, x.voxel, x.sub, radius);
  double4 rp = make_double4(0, 0, 0, 0);
  if (x.kind == kEdge) {
    const V3 a{x.ss[0], x.ss[1], x.ss[2]}, b{x.se[0], x.se[1], x.se[2]};
    const V3 m = 0.5 * (a + b);
    rp = make_double4(m.x, m.y, m.z, 0);
  } else {
    // reception_point_of, Receiver: first RX with this id (voxel_grid.cpp:73-77)
    for (uint32_t k = 0; k < n_rx; ++k) {
      if (rx_id[k] == x.rx) {
        rp = make_double4(rx_pos[3 * k], rx_pos[3 * k + 1], rx_pos[3 * k + 2], 0);
        break;
      }
    }
  }
  o.rp[pos] = rp;
  o.pp[pos] = make_double4(0, 0, 0, 0);
  o.pn[pos] = make_double4(0, 0, 1, 0);  // IntersectableEntity default plane_normal = UnitZ
  o.seg_s[pos] = make_double4(x.ss[0], x.ss[1], x.ss[2], 0);
  o.seg_e[pos] = make_double4(x.se[0], x.se[1], x.se[2], 0);
  o.range[pos] = make_uint2(0, 0);
}

// K8c: cells (voxel_grid.cpp:219-223)
__global__ void cells_kernel(const uint32_t* __restrict__ voxel, uint32_t n, int4* __restrict__ cells) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t v = voxel[i];
    if (i == 0 || voxel[i - 1] != v) cells[v].x = static_cast<int>(i);
    if (i + 1 == n || voxel[i + 1] != v) cells[v].y = static_cast<int>(i + 1);
  }
}

// K9: exact L-infinity distance transform, separable (min over axis of max(|d|, f)).
constexpr int kInf = 2147483647;

__global__ void dt_x_kernel(int4* __restrict__ cells, int dx, int dy, int dz, int* __restrict__ g) {
  const int line = blockIdx.x * blockDim.x + threadIdx.x;
  if (line >= dy * dz) return;
  const size_t base = static_cast<size_t>(line) * dx;
  int last = -1;
  for (int x = 0; x < dx; ++x) {
    const int4 c = cells[base + x];
    if (c.x != c.y) last = x;
    g[base + x] = last < 0 ? kInf : x - last;
  }
  last = -1;
  for (int x = dx - 1; x >= 0; --x) {
    const int4 c = cells[base + x];
    if (c.x != c.y) last = x;
    if (last >= 0) g[base + x] = min(g[base + x], last - x);
  }
}

// axis stride s, length n: out[p] = min_r max(r, in[p +- r*s])
__global__ void dt_axis_kernel(const int* __restrict__ in, int* __restrict__ out, int dx, int dy, int dz, int axis,
                               int4* __restrict__ cells_out) {
  const size_t total = static_cast<size_t>(dx) * dy * dz;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int x = static_cast<int>(i % dx);
    const int y = static_cast<int>((i / dx) % dy);
    const int z = static_cast<int>(i / (static_cast<size_t>(dx) * dy));
    const int c = axis == 1 ? y : z;
    const int n = axis == 1 ? dy : dz;
    const size_t stride = axis == 1 ? static_cast<size_t>(dx) : static_cast<size_t>(dx) * dy;
    int best = in[i];
    for (int r = 1; r < best; ++r) {
      const bool lo_ok = c - r >= 0, hi_ok = c + r < n;
      if (!lo_ok && !hi_ok) break;
      if (lo_ok) best = min(best, max(r, in[i - r * stride]));
      if (hi_ok) best = min(best, max(r, in[i + r * stride]));
    }
    (void)x;
    if (cells_out) cells_out[i].z = best;
    else out[i] = best;
  }
}

__global__ void fill_march_kernel(int4* cells, size_t n, int v) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    cells[i].z = v;
}

__global__ void any_occupied_kernel(const int4* cells, size_t n, int* flag) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    if (cells[i].x != cells[i].y) {
      *flag = 1;
      return;
    }
}

__global__ void any_nonplanar_kernel(const uint32_t* __restrict__ meta, uint64_t n, int* __restrict__ flag) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    if ((meta[i] & 3u) == kSurface && !((meta[i] >> 2) & 1u)) *flag = 1;
}
__global__ void gather_payload_kernel(const uint32_t* __restrict__ pidx, uint64_t n, const double* __restrict__ pos,
                                      const double* __restrict__ nrm, uint64_t n_points, double* __restrict__ ppos,
                                      double* __restrict__ pnrm) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t p = pidx[i];
    if (p >= n_points) continue;  // a hand-built grid's index past the scene: never staged reads
    for (int a = 0; a < 3; ++a) {
      ppos[3 * i + a] = pos[3 * p + a];
      pnrm[3 * i + a] = nrm[3 * p + a];
    }
  }
}

}  // namespace

// The grid's view for kernels that evaluate the non-planar SDF on `scene`: the payload
// positions and normals are gathered into point_indices order once (same values, same
// order as estimate_surface's point_indices -> scene reads), when any IE is non-planar.
GridView GridDev::view_for(Ctx& ctx, const SceneDev& scene) const {
  GridView v = view();
  cudaStream_t s = ctx.stream;
  if (has_nonplanar < 0) {
    DBuf<int> f(1, s);
    PCR_CUDA(cudaMemsetAsync(f.get(), 0, sizeof(int), s));
    if (n_ies) {
      count_launch();
      any_nonplanar_kernel<<<blocks_for(n_ies, kThreads), kThreads, 0, s>>>(meta.get(), n_ies, f.get());
      PCR_LAUNCH_CHECK();
    }
    int h = 0;
    d2h(&h, f.get(), 1, s);
    stream_wait(s);
    has_nonplanar = h;
  }
#ifndef PCR_STAGE_PAYLOAD
#define PCR_STAGE_PAYLOAD 1
#endif
  if (!PCR_STAGE_PAYLOAD || !has_nonplanar || !n_pidx) return v;
  if (pay_for != scene.uid) {
    pay_pos.alloc(3 * n_pidx, s);
    pay_nrm.alloc(3 * n_pidx, s);
    count_launch();
    gather_payload_kernel<<<blocks_for(n_pidx, kThreads), kThreads, 0, s>>>(
        pidx.get(), n_pidx, scene.pos.get(), scene.nrm.get(), scene.n_points, pay_pos.get(), pay_nrm.get());
    PCR_LAUNCH_CHECK();
    pay_for = scene.uid;
  }
  v.pay_pos = pay_pos.get();
  v.pay_nrm = pay_nrm.get();
  return v;
}

void compute_march_distances_device(Ctx& ctx, GridDev& grid) {
  cudaStream_t s = ctx.stream;
  const size_t n = grid.n_cells;
  if (n == 0) return;
  DBuf<int> flag(1, s);
  PCR_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), s));
  count_launch();
  any_occupied_kernel<<<blocks_for(n, kThreads), kThreads, 0, s>>>(grid.cells.get(), n, flag.get());
  PCR_LAUNCH_CHECK();
  int any = 0;
  d2h(&any, flag.get(), 1, s);
  stream_wait(s);
  if (!any) {
    count_launch();
    fill_march_kernel<<<blocks_for(n, kThreads), kThreads, 0, s>>>(grid.cells.get(), n, kMarchNoIes);
    PCR_LAUNCH_CHECK();
    grid.march_ok = true;
    return;
  }
  const int dx = grid.dims[0], dy = grid.dims[1], dz = grid.dims[2];
  DBuf<int> g1(n, s), g2(n, s);
  count_launch();
  dt_x_kernel<<<blocks_for(static_cast<uint64_t>(dy) * dz, 128, 1u << 30), 128, 0, s>>>(grid.cells.get(), dx, dy, dz,
                                                                                       g1.get());
  PCR_LAUNCH_CHECK();
  count_launch();
  dt_axis_kernel<<<blocks_for(n, kThreads), kThreads, 0, s>>>(g1.get(), g2.get(), dx, dy, dz, 1, nullptr);
  PCR_LAUNCH_CHECK();
  count_launch();
  dt_axis_kernel<<<blocks_for(n, kThreads), kThreads, 0, s>>>(g2.get(), nullptr, dx, dy, dz, 2, grid.cells.get());
  PCR_LAUNCH_CHECK();
  grid.march_ok = true;
}

void build_grid_device(Ctx& ctx, const SceneDev& scene, double voxel_size, int division_factor,
                       uint64_t max_cells, GridDev& out, const VoxelShard* shard) {
  cudaStream_t s = ctx.stream;
  // voxel_grid.cpp:83-84
  if (!(voxel_size > 0.0)) throw Error(1, "voxel_size must be > 0");
  if (division_factor < 1) throw Error(1, "division_factor must be >= 1");

  // ---- K1: scene_bounds(scene, voxel_size) (scene.cpp:93-106)
  uint64_t N = scene.n_points;  // this build's points (a shard's subset when sharded)
  double mn[3], mx[3];
  for (int a = 0; a < 3; ++a) {
    mn[a] = std::numeric_limits<double>::max();
    mx[a] = std::numeric_limits<double>::lowest();
  }
  uint32_t max_label = 0;
  if (N) {
    const unsigned nb = blocks_for(N, kThreads, 4u * 148u);
    DBuf<BoundsPartial> part(nb, s);
    count_launch();
    bounds_kernel<<<nb, kThreads, 0, s>>>(scene.pos.get(), scene.label.get(), N, part.get());
    PCR_LAUNCH_CHECK();
    std::vector<BoundsPartial> hp(nb);
    d2h(hp.data(), part.get(), nb, s);
    stream_wait(s);
    for (const auto& p : hp) {
      for (int a = 0; a < 3; ++a) {
        mn[a] = smin(mn[a], p.mn[a]);
        mx[a] = smax(mx[a], p.mx[a]);
      }
      max_label = std::max(max_label, p.max_label);
    }
  }
  auto expand = [&](const double* p) {
    for (int a = 0; a < 3; ++a) {
      mn[a] = smin(mn[a], p[a]);  // cwiseMin: std::min(min, p)
      mx[a] = smax(mx[a], p[a]);
    }
  };
  for (uint32_t e = 0; e < scene.n_edges; ++e) {
    expand(&scene.h_edges[12 * e]);
    expand(&scene.h_edges[12 * e + 3]);
  }
  for (size_t i = 0; i < scene.h_tx_id.size(); ++i) expand(&scene.h_tx[3 * i]);
  for (size_t i = 0; i < scene.h_rx_id.size(); ++i) expand(&scene.h_rx[3 * i]);
  if (!(mn[0] <= mx[0] && mn[1] <= mx[1] && mn[2] <= mx[2])) throw Error(4, "empty scene");
  for (int a = 0; a < 3; ++a) {
    mn[a] = mn[a] - voxel_size;
    mx[a] = mx[a] + voxel_size;
  }

  // ---- dims (voxel_grid.cpp:92-101)
  int dims[3];
  double cell_product = 1.0;
  for (int a = 0; a < 3; ++a) {
    const double span = (mx[a] - mn[a]) / voxel_size;
    dims[a] = std::max(1, static_cast<int>(std::ceil(span - 1e-9)));
    cell_product *= dims[a];
  }
  if (cell_product > static_cast<double>(max_cells)) throw Error(4, "grid too large");
  out.set_geometry(V3{mn[0], mn[1], mn[2]}, dims, voxel_size, division_factor);
  const uint64_t n_cells = static_cast<uint64_t>(cell_product);
  out.n_cells = n_cells;
  out.cells.alloc(n_cells ? n_cells : 1, s);
  PCR_CUDA(cudaMemsetAsync(out.cells.get(), 0, sizeof(int4) * (n_cells ? n_cells : 1), s));

  Lattice L;
  L.ox = mn[0];
  L.oy = mn[1];
  L.oz = mn[2];
  L.se = out.sub_edge;
  L.dims[0] = dims[0];
  L.dims[1] = dims[1];
  L.dims[2] = dims[2];
  L.dv = division_factor;
  const int dv = division_factor;
  const int voxel_bits = bit_width(n_cells ? n_cells - 1 : 0);
  const int sub_bits = std::max(1, bit_width(static_cast<uint64_t>(dv) * dv * dv - 1));
  const int label_bits = bit_width(max_label);
  const bool with_label = voxel_bits + sub_bits + label_bits <= 64;

  // ---- sharded build: this shard's contiguous voxel range, its points only
  DBuf<uint32_t> shard_ids;
  uint32_t v_lo = 0, v_hi = static_cast<uint32_t>(n_cells);
  if (shard) {
    if (shard->n_shards == 0 || shard->index >= shard->n_shards) throw Error(1, "voxelize: shard index out of range");
    DBuf<uint32_t> vox(N ? N : 1, s);
    if (N) {
      count_launch();
      voxel_of_kernel<<<blocks_for(N, kThreads), kThreads, 0, s>>>(L, scene.pos.get(), N, vox.get());
      PCR_LAUNCH_CHECK();
    }
    // splitters: voxel ranges of about N / n_shards points each (every shard computes
    // the same histogram of the same replicated scene, so they agree without a message)
    {
      DBuf<uint32_t> hist(n_cells ? n_cells : 1, s), pre(n_cells ? n_cells : 1, s), tot(1, s);
      PCR_CUDA(cudaMemsetAsync(hist.get(), 0, sizeof(uint32_t) * (n_cells ? n_cells : 1), s));
      if (N) {
        count_launch();
        voxel_hist_kernel<<<blocks_for(N, kThreads), kThreads, 0, s>>>(vox.get(), N, hist.get());
        PCR_LAUNCH_CHECK();
      }
      exclusive_scan_u32(hist.get(), pre.get(), n_cells, tot.get(), s);
      std::vector<uint32_t> hp(n_cells);
      d2h(hp.data(), pre.get(), n_cells, s);
      stream_wait(s);
      auto split = [&](uint32_t r) -> uint32_t {  // first voxel whose prefix reaches r N / n
        if (r == 0) return 0;
        if (r >= shard->n_shards) return static_cast<uint32_t>(n_cells);
        const uint64_t want = (N * r + shard->n_shards - 1) / shard->n_shards;
        return static_cast<uint32_t>(std::lower_bound(hp.begin(), hp.end(), want) - hp.begin());
      };
      v_lo = split(shard->index);
      v_hi = std::max(v_lo, split(shard->index + 1));
    }
    DBuf<uint32_t> flag(N ? N : 1, s), fpos(N ? N : 1, s), cnt(1, s);
    uint32_t n_in = 0;
    if (N) {
      count_launch();
      in_range_kernel<<<blocks_for(N, kThreads), kThreads, 0, s>>>(vox.get(), N, v_lo, v_hi, flag.get());
      PCR_LAUNCH_CHECK();
      exclusive_scan_u32(flag.get(), fpos.get(), N, cnt.get(), s);
      d2h(&n_in, cnt.get(), 1, s);
      stream_wait(s);
    }
    shard_ids.alloc(n_in ? n_in : 1, s);
    if (n_in) {
      count_launch();
      compact_ids_kernel<<<blocks_for(N, kThreads), kThreads, 0, s>>>(flag.get(), fpos.get(), N, shard_ids.get());
      PCR_LAUNCH_CHECK();
    }
    N = n_in;
    out.part_voxel_lo = v_lo;
    out.part_voxel_hi = v_hi;
  }

  // ---- K2/K3: keys + stable radix sort
  DBuf<uint64_t> key(N ? N : 1, s);
  DBuf<uint32_t> sidx(N ? N : 1, s);
  DBuf<uint64_t> vs_key(N ? N : 1, s);
  DBuf<uint32_t> slabel(N ? N : 1, s);
  DBuf<uint32_t> head(N ? N : 1, s);
  DBuf<uint32_t> ie_id(N ? N : 1, s);
  DBuf<uint32_t> n_surf_dev(1, s);
  uint32_t n_surf = 0;
  if (N) {
    if (shard)
      PCR_CUDA(cudaMemcpyAsync(sidx.get(), shard_ids.get(), N * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    else
      iota_u32(sidx.get(), N, s);
    if (!with_label) {
      // Keys too wide for one word: stable pass on the label first (LSD order).
      count_launch();
      gather_label_key_kernel<<<blocks_for(N, kThreads), kThreads, 0, s>>>(scene.label.get(), sidx.get(), N,
                                                                           key.get());
      PCR_LAUNCH_CHECK();
      radix_sort_pairs(key.get(), sidx.get(), N, 0, std::max(1, label_bits), s);
    }
    count_launch();
    bin_kernel<<<blocks_for(N, kThreads), kThreads, 0, s>>>(L, scene.pos.get(), scene.label.get(),
                                                            (with_label && !shard) ? nullptr : sidx.get(), N,
                                                            sub_bits, label_bits, with_label, key.get());
    PCR_LAUNCH_CHECK();
    radix_sort_pairs(key.get(), sidx.get(), N, 0,
                     with_label ? voxel_bits + sub_bits + label_bits : voxel_bits + sub_bits, s);
    count_launch();
    unpack_kernel<<<blocks_for(N, kThreads), kThreads, 0, s>>>(key.get(), sidx.get(), scene.label.get(), N,
                                                               label_bits, with_label, vs_key.get(), slabel.get());
    PCR_LAUNCH_CHECK();
    // ---- K4: heads -> IE ids
    count_launch();
    head_kernel<<<blocks_for(N, kThreads), kThreads, 0, s>>>(vs_key.get(), slabel.get(), N, head.get());
    PCR_LAUNCH_CHECK();
    exclusive_scan_u32(head.get(), ie_id.get(), N, n_surf_dev.get(), s);
    d2h(&n_surf, n_surf_dev.get(), 1, s);
    stream_wait(s);
  }
  key.release();

  // ---- K5: SurfacePoints IEs
  const size_t ms = n_surf ? n_surf : 1;
  DBuf<uint32_t> starts(ms, s);
  DBuf<uint64_t> t_key(ms, s);
  DBuf<uint32_t> t_label(ms, s), t_planar(ms, s);
  DBuf<uint2> t_range(ms, s);
  DBuf<double4> t_cent(ms, s), t_pp(ms, s), t_pn(ms, s);
  SurfaceTmp tmp{t_key.get(), t_label.get(), t_range.get(), t_cent.get(), t_pp.get(), t_pn.get(), t_planar.get()};
  if (n_surf) {
    count_launch();
    starts_kernel<<<blocks_for(N, kThreads), kThreads, 0, s>>>(head.get(), ie_id.get(), N, starts.get());
    PCR_LAUNCH_CHECK();
    count_launch();
    surface_ie_kernel<<<blocks_for(static_cast<uint64_t>(n_surf) * 32, kThreads, 148u * 32u), kThreads, 0, s>>>(
        vs_key.get(), slabel.get(), sidx.get(), starts.get(), n_surf, N, scene.pos.get(), scene.nrm.get(), tmp);
    PCR_LAUNCH_CHECK();
  }
  head.release();
  ie_id.release();
  vs_key.release();
  slabel.release();

  // ---- K6/K7a: edge pieces and receivers
  const uint32_t n_edges = scene.n_edges;
  const uint32_t n_rx = static_cast<uint32_t>(scene.h_rx_id.size());
  uint32_t n_pieces = 0;
  DBuf<uint32_t> piece_off(n_edges + 1, s);
  if (n_edges) {
    DBuf<uint32_t> cnt(n_edges, s);
    count_launch();
    edge_count_kernel<<<blocks_for(n_edges, 64, 1u << 30), 64, 0, s>>>(L, scene.edges.get(), n_edges, cnt.get());
    PCR_LAUNCH_CHECK();
    DBuf<uint32_t> tot(1, s);
    exclusive_scan_u32(cnt.get(), piece_off.get(), n_edges, tot.get(), s);
    d2h(&n_pieces, tot.get(), 1, s);
    stream_wait(s);
  }
  uint32_t n_extra = n_pieces + n_rx;
  DBuf<ExtraIE> extra(n_extra ? n_extra : 1, s), extra_sorted(n_extra ? n_extra : 1, s);
  DBuf<uint64_t> extra_keys(n_extra ? n_extra : 1, s);
  if (n_pieces) {
    count_launch();
    edge_emit_kernel<<<blocks_for(n_edges, 64, 1u << 30), 64, 0, s>>>(L, scene.edges.get(), scene.edge_label.get(),
                                                                      n_edges, piece_off.get(), sub_bits,
                                                                      extra.get());
    PCR_LAUNCH_CHECK();
  }
  if (n_rx) {
    count_launch();
    rx_kernel<<<blocks_for(n_rx, 64, 1u << 30), 64, 0, s>>>(L, scene.rx_pos.get(), scene.rx_id.get(), n_rx,
                                                            sub_bits, extra.get() + n_pieces);
    PCR_LAUNCH_CHECK();
  }
  if (n_extra) {
    count_launch();
    extra_rank_kernel<<<blocks_for(n_extra, 128, 1u << 30), 128, 0, s>>>(extra.get(), n_extra, extra_sorted.get());
    PCR_LAUNCH_CHECK();
    if (shard) {  // the shard keeps the edge pieces and receivers of its voxel range (few)
      std::vector<ExtraIE> h(n_extra), k;
      d2h(h.data(), extra_sorted.get(), n_extra, s);
      stream_wait(s);
      for (const ExtraIE& x : h)
        if (x.voxel >= v_lo && x.voxel < v_hi) k.push_back(x);
      n_extra = static_cast<uint32_t>(k.size());
      if (n_extra) h2d(extra_sorted.get(), k.data(), n_extra, s);
    }
  }
  if (n_extra) {
    count_launch();
    extract_keys_kernel<<<blocks_for(n_extra, 128, 1u << 30), 128, 0, s>>>(extra_sorted.get(), n_extra,
                                                                           extra_keys.get());
    PCR_LAUNCH_CHECK();
  }

  // ---- K8: canonical merge, final records, cells
  const uint64_t n_ies = static_cast<uint64_t>(n_surf) + n_extra;
  out.alloc_ies(n_ies, s);
  out.n_pidx = N;
  out.pidx = std::move(sidx);
  FinalOut fo{out.meta.get(), out.label.get(), out.edge.get(), out.rx.get(), out.voxel.get(), out.sub.get(),
              out.sc.get(), out.rp.get(), out.pp.get(), out.pn.get(), out.seg_s.get(), out.seg_e.get(),
              out.range.get()};
  const double radius = out.sub_radius;
  if (n_surf) {
    count_launch();
    scatter_surface_kernel<<<blocks_for(n_surf, kThreads), kThreads, 0, s>>>(
        L, voxel_size, radius, tmp, n_surf, extra_keys.get(), n_extra, sub_bits, fo);
    PCR_LAUNCH_CHECK();
  }
  if (n_extra) {
    count_launch();
    scatter_extra_kernel<<<blocks_for(n_extra, 128, 1u << 30), 128, 0, s>>>(
        L, voxel_size, radius, extra_sorted.get(), n_extra, t_key.get(), n_surf, scene.rx_pos.get(),
        scene.rx_id.get(), n_rx, fo);
    PCR_LAUNCH_CHECK();
  }
  if (shard) {  // a part: cells and march distances come with the assembled grid
    out.cells.release();
    stream_wait(s);
    return;
  }
  if (n_ies) {
    count_launch();
    cells_kernel<<<blocks_for(n_ies, kThreads), kThreads, 0, s>>>(out.voxel.get(), static_cast<uint32_t>(n_ies),
                                                                  out.cells.get());
    PCR_LAUNCH_CHECK();
  }
  // ---- K9
  compute_march_distances_device(ctx, out);
  stream_wait(s);
}

}  // namespace pcr
