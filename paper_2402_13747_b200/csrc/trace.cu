// trace.cu — stage 2: transmission_phase (tracer.cpp:207-255) and propagate
// (tracer.cpp:476-533) as a depth-first wavefront of ray chunks.
//
//   K10 transmission_kernel  one thread per (TX, IE): safe_normalized, segment_visible,
//                            LOS / surface hit / edge hit; ordered compaction by scan
//   materialize_kernel       node (interaction) + fan index -> conical ray (reflect_ray
//                            tracer.cpp:257-267, diffract_rays :269-311 with a host sin/cos table)
//   K12 walk_kernel          voxel_cone_trace walk per ray -> visibility tasks (ray, IE)
//   K13 visibility_kernel    one thread per task: segment_visible + march/project, then
//                            spawn (dfs_trace :418-472): RX -> candidate, surface -> reflection
//                            node, edge -> Keller-fan node
//   K16 kappa                DFS-order keys + group hashes; radix sorts; first kappa per
//                            (rx, label sequence) in DFS order (propagate :513-531)
//
// DFS order: the reference emits candidates task by task, receptions in ascending
// ie_index (:400-401), fans in j order. The key (task, j1, ie2, j2, ..., rx_ie) packed
// MSB-first orders candidates exactly so; keeping the first kappa of each group in
// key order reproduces the merged task-local + global caps. Chunks are processed
// depth first so the frontier stays bounded.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <vector>

#include "host_alloc.hpp"
#include "pipeline.hpp"
#include "shard_rows.cuh"
#include "sort.cuh"
#include "stages.cuh"
#include "trace.cuh"

namespace pcr {

struct TraceCfg {
  int max_interactions, kappa, fan_n, max_diffractions;
  double apex;
};

namespace {

constexpr int kT = 256;

__device__ __forceinline__ uint32_t atomic_append(uint32_t* counter) { return atomicAdd(counter, 1u); }

// Builds ray j of a node's children. Reflection: j == 0. Returns alive.
__device__ __forceinline__ bool make_ray(const Node& nd, uint32_t node_idx, uint32_t j, const GridView& g,
                                         const SceneView& s, const TraceCfg& c, const FanTable& fan, Ray& r) {
  r.node = node_idx;
  r.j = j;
  r.origin_ie = nd.ie;
  r.origin_label = nd.label;
  r.depth = nd.depth;
  r.dc = nd.dc;
  r.apex = c.apex;  // spawn_apex_angle is the identity (tracer.cpp:110-114)
  const V3 pos = load3(nd.pos), n = load3(nd.nrm), inc = load3(nd.inc);
  if (nd.kind == 0) {
    // reflect_ray (tracer.cpp:257-267)
    const double dn = dot(inc, n);
    if (dn >= 0.0) return false;
    r.d = normalized(inc - (2.0 * dn) * n);
    r.o = pos + g.hit_eps * n;
    r.n_planes = 1;
    r.pn[0] = n;
    return true;
  }
  V3 w, e1, e2, na, nb;
  double cos_b, sin_b;
  if (!fan_frame(s.edges + 12ull * nd.edge, inc, w, e1, e2, cos_b, sin_b, na, nb)) return false;
  const double* t = fan.t + 6ull * j;
  const V3 dir = cos_b * w + sin_b * (t[0] * e1 + t[1] * e2);
  if (dot(dir, na) < 0.0 && dot(dir, nb) < 0.0) return false;
  r.o = pos;
  r.d = dir;
  r.n_planes = 2;
  // planes {point, -tangent(phi + dphi/2)}, {point, tangent(phi - dphi/2)}; tangent(psi) = -sin(psi) e1 + cos(psi) e2
  const V3 tp = (-t[2]) * e1 + t[3] * e2;
  r.pn[0] = -tp;
  r.pn[1] = (-t[4]) * e1 + t[5] * e2;
  return true;
}

__global__ void materialize_kernel(const Node* __restrict__ nodes, uint32_t node_begin,
                                   const uint64_t* __restrict__ prefix, uint32_t n_range, uint64_t v_begin,
                                   uint32_t n_rays, const uint64_t* __restrict__ v_total, GridView g, SceneView s,
                                   TraceCfg c, FanTable fan, Ray* __restrict__ rays) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_rays) return;
  const uint64_t vk = v_begin + k;
  if (vk >= *v_total) {  // past the range's last child ray (the host sizes chunks before it knows the total)
    rays[k].alive = 0;
    return;
  }
  uint32_t lo = 0, hi = n_range;  // upper_bound(prefix, vk) - 1
  while (lo < hi) {
    const uint32_t m = (lo + hi) >> 1;
    if (prefix[m] <= vk) lo = m + 1;
    else hi = m;
  }
  const uint32_t local = lo - 1;
  const uint32_t j = static_cast<uint32_t>(vk - prefix[local]);
  Ray r;
  const uint32_t ni = node_begin + local;
  r.alive = make_ray(nodes[ni], ni, j, g, s, c, fan, r) ? 1 : 0;
  rays[k] = r;
}

// K12: cone walk emitting visibility tasks. `filter` drops IEs whose reception
// cannot produce output at this depth (non-RX at depth >= max_interactions,
// edges once the diffraction budget is spent): the reference traces them and
// discards the reception (tracer.cpp:441, 456), so the output is unchanged.
// One warp per ray (warp_cone_walk); surviving IEs are appended with one atomic per
// warp round.
constexpr int kWalkThreads = 128;
// 8 blocks of 128 threads per SM (64 registers): C3 cone walk 9.32 s at the
// compiler's 80 registers, 9.42 s at 72, 8.89 s at 64, 9.55 s at 48 (same box)
#ifndef PCR_WALK_MINB
#define PCR_WALK_MINB 8
#endif
__global__ void __launch_bounds__(kWalkThreads, PCR_WALK_MINB) walk_kernel(const Ray* __restrict__ rays, uint32_t n_rays, GridView g,
                                                            TraceCfg c, bool filter, Task* __restrict__ tasks,
                                                            uint32_t* __restrict__ n_tasks, uint32_t cap,
                                                            unsigned long long* __restrict__ stats) {
  const int lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t cells = 0, ies = 0;
  for (uint32_t k = warp; k < n_rays; k += nwarps) {
    const Ray r = rays[k];
    if (!r.alive) continue;
    const bool can_refl = r.depth < c.max_interactions;
    const bool can_diff = can_refl && r.dc < c.max_diffractions;
    warp_cone_walk(
        g, r, [](uint32_t) {},
        [&](uint32_t i, bool pass) {
          if (pass && filter) {
            const uint32_t kind = g.ie_meta[i] & 3u;
            if ((kind == kSurface && !can_refl) || (kind == kEdge && !can_diff)) pass = false;
          }
          const unsigned m = __ballot_sync(0xffffffffu, pass);
          if (!m) return;
          const int leader = __ffs(m) - 1;
          uint32_t base = 0;
          if (lane == leader) base = atomicAdd(n_tasks, static_cast<uint32_t>(__popc(m)));
          base = __shfl_sync(0xffffffffu, base, leader);
          if (pass) {
            const uint32_t slot = base + __popc(m & lt);
            if (slot < cap) tasks[slot] = Task{k, i};
          }
        },
        &cells, &ies);
  }
  if (stats && lane == 0) {
    atomicAdd(stats, static_cast<unsigned long long>(cells));
    atomicAdd(stats + 1, static_cast<unsigned long long>(ies));
  }
}

// 32 blocks per SM (4 waves at 8 resident): smaller per-warp strides balance the
// rays' uneven walks; same box, C2 cone walk 119.8 / 116.9 / 111.5 ms at 8 / 16 / 32
#ifndef PCR_WALK_GRID_MULT
#define PCR_WALK_GRID_MULT 32
#endif
unsigned walk_blocks(uint64_t n_rays, int sm_count) {
  const uint64_t want = (n_rays * 32 + kWalkThreads - 1) / kWalkThreads;
  const uint64_t cap = static_cast<uint64_t>(sm_count) * PCR_WALK_GRID_MULT;
  return static_cast<unsigned>(want < cap ? (want ? want : 1) : cap);
}

struct SpawnOut {
  Node* nodes;
  uint32_t* n_nodes;
  Cand* cands;
  uint32_t* n_cands;
  uint64_t* n_vis;  // segment_visible calls
};

// K13: visibility + hit + spawn.
// One warp per task: warp_segment_visible, then lane 0 computes the hit and spawns.
__device__ void spawn_reception(const Task tk, const Ray& r, const Node* __restrict__ parent_nodes, const GridView& g,
                                const SceneView& s, const TraceCfg& c, SpawnOut& o);

// 8 blocks of 128 threads per SM (64 registers; the spills stay in L1): C3
// visibility 17.4 s at 168 registers, 13.6 s at 128, 13.4 s at 80, 12.3 s at 64
// and 48 (same box); C2 30.9 -> 27.7 ms
#ifndef PCR_VIS_MINB
#define PCR_VIS_MINB 8
#endif
__global__ void __launch_bounds__(128, PCR_VIS_MINB) visibility_kernel(const Task* __restrict__ tasks,
                                                         const uint32_t* __restrict__ n_tasks_dev, uint32_t cap,
                                                         const Ray* __restrict__ rays,
                                                         const Node* __restrict__ parent_nodes, GridView g,
                                                         SceneView s, TraceCfg c, SpawnOut o) {
  const int lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  // visible tasks are queued one per lane and spawned 32 at a time (one lane each)
  // instead of by lane 0 alone after every test; appends are atomic either way and
  // the node/candidate order is canonicalised downstream
  // the walk's task count stays on the device (no host round trip between the two
  // kernels); a walk that overflowed the buffer left an incomplete list: do nothing,
  // the host sees the count and reruns the chunk with a bigger buffer
  const uint32_t n_tasks = *n_tasks_dev;
  if (n_tasks > cap) return;
  uint32_t mine = 0;
  int queued = 0;
  for (uint32_t t = warp; t < n_tasks; t += nwarps) {
    const Task tk = tasks[t];
    const Ray r = rays[tk.ray];
    const V3 rp = ld3(g.ie_rp[tk.ie]);
    if (!warp_segment_visible(r.o, rp, tk.ie, g, s)) continue;
    if (lane == queued) mine = t;
    if (++queued == 32) {
      const Task q = tasks[mine];
      spawn_reception(q, rays[q.ray], parent_nodes, g, s, c, o);
      queued = 0;
    }
  }
  if (lane < queued) {
    const Task q = tasks[mine];
    spawn_reception(q, rays[q.ray], parent_nodes, g, s, c, o);
  }
}

__device__ void spawn_reception(const Task tk, const Ray& r, const Node* __restrict__ parent_nodes, const GridView& g,
                                const SceneView& s, const TraceCfg& c, SpawnOut& o) {
  (void)c;
  const uint32_t i = tk.ie;
  const V3 rp = ld3(g.ie_rp[i]);
  const uint32_t kind = g.ie_meta[i] & 3u;
  if (kind == kReceiver) {
    const uint32_t slot = atomic_append(o.n_cands);
    o.cands[slot] = Cand{r.node, r.j, i, 0};
    return;
  }
  Node nd;
  nd.parent = r.node;
  nd.parent_j = r.j;
  nd.ie = i;
  nd.label = g.ie_label[i];
  nd.task = parent_nodes[r.node].task;
  nd.depth = static_cast<uint8_t>(r.depth + 1);
  nd.pad = 0;
  if (kind == kSurface) {
    const V3 dir = safe_normalized(rp - r.o);
    SurfaceHit hit;
    bool ok = march_segment(r.o, dir, i, g, s, __longlong_as_double(0x7ff0000000000000ll), &hit);
    if (!ok) {
      ok = project_to_surface(rp, i, g, s, &hit);
      if (ok) hit.distance = norm(hit.position - r.o);
    }
    if (!ok) return;
    const V3 incoming = safe_normalized(hit.position - r.o);
    if (is_zero(incoming)) return;
    if (dot(incoming, hit.normal) >= 0.0) return;  // reflect_ray rejects back-facing incidence
    nd.kind = 0;
    nd.dc = r.dc;
    nd.edge = 0;
    store3(nd.pos, hit.position);
    store3(nd.nrm, hit.normal);
    store3(nd.inc, incoming);
    nd.n_children = 1;
  } else {
    const V3 incoming = safe_normalized(rp - r.o);
    if (is_zero(incoming)) return;
    const uint32_t e = g.ie_edge[i];
    V3 w, e1, e2, na, nb;
    double cos_b, sin_b;
    if (!fan_frame(s.edges + 12ull * e, incoming, w, e1, e2, cos_b, sin_b, na, nb)) return;
    nd.kind = 1;
    nd.dc = static_cast<uint8_t>(r.dc + 1);
    nd.edge = e;
    store3(nd.pos, rp);
    store3(nd.nrm, na);
    store3(nd.inc, incoming);
    nd.n_children = static_cast<uint32_t>(c.fan_n);
  }
  const uint32_t slot = atomic_append(o.n_nodes);
  o.nodes[slot] = nd;
}

// K10: transmission (tracer.cpp:207-255), one thread per IE.
struct TxOut {
  uint8_t* los;
  uint8_t* hit;
  double* hpos;  // n*3
  double* hnrm;
  double* hinc;
};

__device__ void transmission_hit(uint32_t i, const V3& tx, const GridView& g, const SceneView& s, TxOut& o);

// one warp per IE: warp_segment_visible, then lane 0 classifies the reception
__global__ void __launch_bounds__(128, 4) transmission_kernel(GridView g, SceneView s, V3 tx, TxOut o) {
  const int lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t i = warp; i < g.n_ies; i += nwarps) {
    const V3 rp = ld3(g.ie_rp[i]);
    const uint32_t kind = g.ie_meta[i] & 3u;
    const V3 dir = safe_normalized(rp - tx);
    bool go = !(is_zero(dir) && kind != kReceiver);
    if (go) go = warp_segment_visible(tx, rp, i, g, s);
    if (lane == 0) {
      o.los[i] = 0;
      o.hit[i] = 0;
      if (go) transmission_hit(i, tx, g, s, o);
    }
  }
}

__device__ void transmission_hit(uint32_t i, const V3& tx, const GridView& g, const SceneView& s, TxOut& o) {
  const V3 rp = ld3(g.ie_rp[i]);
  const uint32_t kind = g.ie_meta[i] & 3u;
  const V3 dir = safe_normalized(rp - tx);
  if (kind == kReceiver) {
    o.los[i] = 1;
    return;
  }
  if (kind == kSurface) {
    SurfaceHit hit;
    bool ok = march_segment(tx, dir, i, g, s, __longlong_as_double(0x7ff0000000000000ll), &hit);
    if (!ok) ok = project_to_surface(rp, i, g, s, &hit);
    if (!ok) return;
    const V3 incoming = safe_normalized(hit.position - tx);
    if (is_zero(incoming)) return;
    o.hit[i] = 1;
    store3(o.hpos + 3ull * i, hit.position);
    store3(o.hnrm + 3ull * i, hit.normal);
    store3(o.hinc + 3ull * i, incoming);
    return;
  }
  o.hit[i] = 1;
  store3(o.hpos + 3ull * i, rp);
  store3(o.hnrm + 3ull * i, V3{0, 0, 1});
  store3(o.hinc + 3ull * i, dir);
}

// Root nodes from initial hits (propagate :482-509).
__global__ void seed_kernel(const uint32_t* __restrict__ ie_index, const uint8_t* __restrict__ kind,
                            const double* __restrict__ pos, const double* __restrict__ nrm,
                            const double* __restrict__ inc, uint32_t n, uint32_t task_first, uint32_t task_step,
                            GridView g, SceneView s, TraceCfg c, Node* __restrict__ nodes) {
  const uint32_t slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= n) return;
  // this shard's tasks are initial hits task_first, task_first + task_step, ...
  const uint32_t k = task_first + slot * task_step;
  const uint32_t i = ie_index[k];
  Node nd;
  nd.parent = kNoNode;
  nd.parent_j = 0;
  nd.ie = i;
  nd.label = g.ie_label[i];
  nd.task = k;  // the global task index: DFS keys are shard-independent
  nd.depth = 1;
  nd.pad = 0;
  nd.n_children = 0;
  const V3 p = load3(pos + 3ull * k), nn = load3(nrm + 3ull * k), in = load3(inc + 3ull * k);
  store3(nd.pos, p);
  store3(nd.inc, in);
  if (kind[k] == kSurface) {
    nd.kind = 0;
    nd.dc = 0;
    nd.edge = 0;
    store3(nd.nrm, nn);
    nd.n_children = dot(in, nn) < 0.0 ? 1u : 0u;
  } else if (kind[k] == kEdge) {
    const uint32_t e = g.ie_edge[i];
    nd.kind = 1;
    nd.dc = 1;
    nd.edge = e;
    store3(nd.nrm, load3(s.edges + 12ull * e + 6));
    V3 w, e1, e2, na, nb;
    double cb, sb;
    if (c.max_diffractions >= 1 && fan_frame(s.edges + 12ull * e, in, w, e1, e2, cb, sb, na, nb))
      nd.n_children = static_cast<uint32_t>(c.fan_n);
  } else {
    nd.kind = 0;
    nd.dc = 0;
    nd.edge = 0;
    store3(nd.nrm, V3{0, 0, 1});
  }
  nodes[slot] = nd;
}

__global__ void children_kernel(const Node* __restrict__ nodes, uint32_t begin, uint32_t n, uint64_t* __restrict__ cnt) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) cnt[k] = nodes[begin + k].n_children;
}

// ---- kappa: keys and groups --------------------------------------------------------
struct KeyLayout {
  int bits_task, bits_j, bits_ie, levels, total;
};

__device__ __forceinline__ void put_bits(uint64_t* w, int& pos, uint64_t v, int bits) {
  // MSB-first bit stream into 4 words
  for (int b = bits - 1; b >= 0; --b) {
    if ((v >> b) & 1ull) w[pos >> 6] |= 1ull << (63 - (pos & 63));
    ++pos;
  }
}

__device__ __forceinline__ uint64_t mix64(uint64_t h, uint64_t v) {
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  h *= 0xff51afd7ed558ccdull;
  h ^= h >> 33;
  return h;
}

__global__ void key_kernel(const Cand* __restrict__ cands, uint32_t n, const Node* __restrict__ nodes, GridView g,
                           KeyLayout L, uint64_t* __restrict__ keys /* 4 words per cand, word-major */,
                           uint64_t* __restrict__ group_hash) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const Cand cd = cands[k];
  uint32_t chain[kMaxDepth], js[kMaxDepth];
  int d = 0;
  uint32_t nj = cd.j;
  for (uint32_t ni = cd.node; ni != kNoNode; ni = nodes[ni].parent) {
    chain[d] = ni;
    js[d] = nj;
    nj = nodes[ni].parent_j;
    ++d;
  }
  // chain[d-1] is the root
  uint64_t w[4] = {0, 0, 0, 0};
  int pos = 0;
  const Node& root = nodes[chain[d - 1]];
  put_bits(w, pos, root.task, L.bits_task);
  uint64_t h = mix64(0x1234567ull, g.ie_rx[cd.rx_ie]);
  h = mix64(h, static_cast<uint64_t>(d));
  for (int lv = d - 1; lv >= 0; --lv) {
    put_bits(w, pos, js[lv], L.bits_j);
    const uint32_t next_ie = lv > 0 ? nodes[chain[lv - 1]].ie : cd.rx_ie;
    put_bits(w, pos, next_ie, L.bits_ie);
    h = mix64(h, nodes[chain[lv]].label);
  }
  for (int q = 0; q < 4; ++q) keys[static_cast<size_t>(q) * n + k] = w[q];
  group_hash[k] = h;
}

__global__ void gather_u64_kernel(const uint64_t* __restrict__ src, const uint32_t* __restrict__ perm, uint32_t n,
                                  uint64_t* __restrict__ dst) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) dst[k] = src[perm[k]];
}

// same group as the previous element in (hash, key) order? (verifies hash runs)
__device__ bool same_group(const Cand& a, const Cand& b, const Node* nodes, const GridView& g) {
  if (g.ie_rx[a.rx_ie] != g.ie_rx[b.rx_ie]) return false;
  uint32_t x = a.node, y = b.node;
  while (x != kNoNode && y != kNoNode) {
    if (nodes[x].label != nodes[y].label) return false;
    x = nodes[x].parent;
    y = nodes[y].parent;
  }
  return x == kNoNode && y == kNoNode;
}

__global__ void rank_kernel(const uint64_t* __restrict__ hash_sorted, const uint32_t* __restrict__ perm, uint32_t n,
                            const Cand* __restrict__ cands, const Node* __restrict__ nodes, GridView g,
                            uint32_t* __restrict__ run_start, int* __restrict__ collision) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const bool head = k == 0 || hash_sorted[k] != hash_sorted[k - 1];
  run_start[k] = head ? k : 0;
  if (!head && !same_group(cands[perm[k]], cands[perm[k - 1]], nodes, g)) *collision = 1;
}

__global__ void max_scan_small_kernel(uint32_t* v, uint32_t n) {
  // sequential running max within one block of 1 thread per 1024-chunk is too slow for big n;
  // done as a simple single-thread pass when n is small (only used below a threshold)
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    uint32_t m = 0;
    for (uint32_t i = 0; i < n; ++i) {
      m = v[i] > m ? v[i] : m;
      v[i] = m;
    }
  }
}

__global__ void keep_kernel(const uint32_t* __restrict__ run_start, const uint32_t* __restrict__ perm, uint32_t n,
                            int kappa, uint8_t* __restrict__ keep_by_cand) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  keep_by_cand[perm[k]] = (k - run_start[k]) < static_cast<uint32_t>(kappa) ? 1 : 0;
}

__global__ void keep_flags_in_order_kernel(const uint8_t* __restrict__ keep_by_cand, const uint32_t* __restrict__ perm,
                                           uint32_t n, uint32_t* __restrict__ flag) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) flag[k] = keep_by_cand[perm[k]];
}

__global__ void compact_cands_kernel(const Cand* __restrict__ in, const uint32_t* __restrict__ perm,
                                     const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos, uint32_t n,
                                     Cand* __restrict__ out) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n && flag[k]) out[pos[k]] = in[perm[k]];
}

// keys (word-major, 4 words) and group hashes of the kept candidates, in kept order
__global__ void compact_keys_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ hash,
                                    const uint32_t* __restrict__ perm, const uint32_t* __restrict__ flag,
                                    const uint32_t* __restrict__ pos, uint32_t n, uint32_t n_out,
                                    uint64_t* __restrict__ keys_out, uint64_t* __restrict__ hash_out) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n || !flag[k]) return;
  const uint32_t src = perm[k], dst = pos[k];
  for (int q = 0; q < 4; ++q) keys_out[static_cast<size_t>(q) * n_out + dst] = keys[static_cast<size_t>(q) * n + src];
  hash_out[dst] = hash[src];
}

// segmented running max of run starts (heads carry their own index)
__global__ void run_max_block_kernel(uint32_t* v, uint32_t n, uint32_t* block_max) {
  __shared__ uint32_t sh[1024];
  const uint32_t base = blockIdx.x * 1024u;
  const uint32_t i = base + threadIdx.x;
  sh[threadIdx.x] = i < n ? v[i] : 0;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    uint32_t t = threadIdx.x >= static_cast<unsigned>(o) ? sh[threadIdx.x - o] : 0;
    __syncthreads();
    sh[threadIdx.x] = max(sh[threadIdx.x], t);
    __syncthreads();
  }
  if (i < n) v[i] = sh[threadIdx.x];
  if (threadIdx.x == 1023) block_max[blockIdx.x] = sh[1023];
}
__global__ void run_max_fix_kernel(uint32_t* v, uint32_t n, const uint32_t* block_prefix_max) {
  const uint32_t i = blockIdx.x * 1024u + threadIdx.x;
  if (i < n && blockIdx.x > 0) v[i] = max(v[i], block_prefix_max[blockIdx.x - 1]);
}

// ---- materialisation of kept candidates ---------------------------------------------
struct CandOut {
  uint32_t stride;
  uint32_t* rx_id;
  double* rx_pos;
  double* length;
  uint32_t* n_inter;
  uint8_t* kind;
  double* pos;
  uint32_t* label;
  double* nrm;
  uint32_t* ie;
  uint32_t* edge;
};

__global__ void materialize_cands_kernel(const Cand* __restrict__ cands, uint32_t n, const Node* __restrict__ nodes,
                                         GridView g, V3 tx, CandOut o) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const Cand cd = cands[k];
  uint32_t chain[kMaxDepth];
  int d = 0;
  for (uint32_t ni = cd.node; ni != kNoNode; ni = nodes[ni].parent) chain[d++] = ni;
  const V3 rxp = ld3(g.ie_rp[cd.rx_ie]);
  o.rx_id[k] = g.ie_rx[cd.rx_ie];
  store3(o.rx_pos + 3ull * k, rxp);
  o.n_inter[k] = static_cast<uint32_t>(d);
  // chain_length (tracer.cpp:116-125), front to back
  V3 prev = tx;
  double len = 0.0;
  for (int lv = 0; lv < d; ++lv) {
    const Node& nd = nodes[chain[d - 1 - lv]];
    const size_t q = static_cast<size_t>(k) * o.stride + lv;
    const V3 p = load3(nd.pos);
    o.kind[q] = nd.kind;
    store3(o.pos + 3 * q, p);
    o.label[q] = nd.label;
    store3(o.nrm + 3 * q, load3(nd.nrm));
    o.ie[q] = nd.ie;
    o.edge[q] = nd.edge;
    len += norm(p - prev);
    prev = p;
  }
  o.length[k] = len + norm(rxp - prev);
}

// ---- batch primitives (test / API surface) ------------------------------------------------
__global__ void rays_from_desc_kernel(const pcr_ray_desc* __restrict__ d, uint64_t n, Ray* __restrict__ rays) {
  const uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  const pcr_ray_desc x = d[k];
  Ray r;
  r.o = load3(x.origin);
  r.d = load3(x.direction);
  r.apex = x.apex_angle;
  r.n_planes = static_cast<uint8_t>(x.n_planes);
  for (int q = 0; q < 2; ++q) r.pn[q] = load3(x.plane_normal[q]);
  r.node = kNoNode;
  r.j = 0;
  r.origin_ie = x.origin_ie;
  r.origin_label = x.origin_label;
  r.depth = 0;
  r.dc = 0;
  r.alive = 1;
  rays[k] = r;
}

__global__ void evaluated_kernel(const Ray* __restrict__ rays, uint32_t n, GridView g,
                                 const uint64_t* __restrict__ offset, uint32_t* __restrict__ count,
                                 uint32_t* __restrict__ out) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  uint32_t c = 0;
  const Ray r = rays[k];
  cone_walk(
      g, r,
      [&](uint32_t cell) {
        if (out) out[offset[k] + c] = cell;
        ++c;
      },
      [](uint32_t) {});
  if (count) count[k] = c;
}

// TraceDebug::visited (tracer.cpp:333-335, 391-397): the walker's voxels, jumps
// over empty space (march >= 2) included, in walk order
__global__ void visited_kernel(const Ray* __restrict__ rays, uint32_t n, GridView g,
                               const uint64_t* __restrict__ offset, uint32_t* __restrict__ count,
                               uint32_t* __restrict__ out) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  uint32_t c = 0;
  if (g.n_ies) {
    const Ray r = rays[k];
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    Walker w;
    w.init(g, r.o, r.d, 0.0, inf);
    while (w.active) {
      const uint32_t vi = linear_index(g, w.v[0], w.v[1], w.v[2]);
      if (out) out[offset[k] + c] = vi;
      ++c;
      const int march = g.cells[vi].z;
      if (march >= 2)
        w.init_at(g, w.t_entry + static_cast<double>(march - 1) * g.voxel_size, inf);
      else
        w.advance(g);
    }
  }
  if (count) count[k] = c;
}

struct RecOut {
  uint8_t* ok;
  uint8_t* hit_valid;
  double* hpos;
  double* hnrm;
  uint32_t* hlabel;
  double* hdist;
};

__global__ void reception_kernel(const Task* __restrict__ tasks, uint32_t n, const Ray* __restrict__ rays, GridView g,
                                 SceneView s, RecOut o) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const Task tk = tasks[t];
  const Ray r = rays[tk.ray];
  const uint32_t i = tk.ie;
  const V3 rp = ld3(g.ie_rp[i]);
  o.ok[t] = 0;
  o.hit_valid[t] = 0;
  if (!segment_visible(r.o, rp, i, g, s)) return;
  if ((g.ie_meta[i] & 3u) == kSurface) {
    const V3 dir = safe_normalized(rp - r.o);
    SurfaceHit hit;
    bool ok = march_segment(r.o, dir, i, g, s, __longlong_as_double(0x7ff0000000000000ll), &hit);
    if (!ok) {
      ok = project_to_surface(rp, i, g, s, &hit);
      if (ok) hit.distance = norm(hit.position - r.o);
    }
    if (!ok) return;
    o.hit_valid[t] = 1;
    store3(o.hpos + 3ull * t, hit.position);
    store3(o.hnrm + 3ull * t, hit.normal);
    o.hlabel[t] = hit.label;
    o.hdist[t] = hit.distance;
  }
  o.ok[t] = 1;
}

__global__ void segvis_kernel(const double* __restrict__ o, const double* __restrict__ tgt,
                              const uint32_t* __restrict__ tie, uint64_t n, GridView g, SceneView s,
                              uint8_t* __restrict__ out) {
  // even segments through the warp-cooperative walk, odd ones through the per-thread
  // walk (refinement's final check): both must agree with the reference
  const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (uint64_t k = 2 * warp; k < n; k += 2 * nwarps) {
    const bool v = warp_segment_visible(load3(o + 3 * k), load3(tgt + 3 * k), tie[k], g, s);
    if (lane == 0) out[k] = v ? 1 : 0;
    if (lane == 1 && k + 1 < n)
      out[k + 1] = segment_visible(load3(o + 3 * (k + 1)), load3(tgt + 3 * (k + 1)), tie[k + 1], g, s) ? 1 : 0;
  }
}

unsigned nb(uint64_t n, unsigned t = kT) { return static_cast<unsigned>((n + t - 1) / t ? (n + t - 1) / t : 1); }

}  // namespace

// ========================================================================================
// host side

void ensure_fan(Ctx& ctx, int n) {
  if (ctx.fan_n == n && ctx.fan_table.get()) return;
  // diffract_rays (tracer.cpp:288-301): phi = j * dphi, dphi = 2 pi / n; the sines and
  // cosines depend on (j, n) only and are evaluated once here with the host libm.
  const double pi = 3.141592653589793238462643383279502884;
  const double dphi = 2.0 * pi / n;
  std::vector<double> t(6ull * (n > 0 ? n : 1));
  for (int j = 0; j < n; ++j) {
    const double phi = j * dphi;
    t[6 * j + 0] = std::cos(phi);
    t[6 * j + 1] = std::sin(phi);
    t[6 * j + 2] = std::sin(phi + 0.5 * dphi);
    t[6 * j + 3] = std::cos(phi + 0.5 * dphi);
    t[6 * j + 4] = std::sin(phi - 0.5 * dphi);
    t[6 * j + 5] = std::cos(phi - 0.5 * dphi);
  }
  ctx.fan_table.alloc(t.size(), ctx.stream);
  h2d(ctx.fan_table.get(), t.data(), t.size(), ctx.stream);
  ctx.fan_n = n;
}

static TraceCfg make_cfg(const pcr_trace_params& p) {
  TraceCfg c;
  c.max_interactions = p.max_interactions;
  c.kappa = p.kappa;
  c.fan_n = p.diffraction_ray_count;
  c.max_diffractions = p.max_diffractions;
  c.apex = p.cone_apex_angle;
  return c;
}

__global__ void compact_tx_kernel(const uint8_t* __restrict__ los, const uint8_t* __restrict__ hit,
                                  const uint32_t* __restrict__ los_pos, const uint32_t* __restrict__ hit_pos_idx,
                                  uint32_t n, const double* __restrict__ hp, const double* __restrict__ hn,
                                  const double* __restrict__ hi, GridView g, uint32_t* __restrict__ los_ie,
                                  uint32_t* __restrict__ hit_ie, uint8_t* __restrict__ hit_kind,
                                  double* __restrict__ op, double* __restrict__ on, double* __restrict__ oi) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (los[i]) los_ie[los_pos[i]] = i;
  if (hit[i]) {
    const uint32_t q = hit_pos_idx[i];
    hit_ie[q] = i;
    hit_kind[q] = static_cast<uint8_t>(g.ie_meta[i] & 3u);
    for (int a = 0; a < 3; ++a) {
      op[3ull * q + a] = hp[3ull * i + a];
      on[3ull * q + a] = hn[3ull * i + a];
      oi[3ull * q + a] = hi[3ull * i + a];
    }
  }
}

__global__ void flags_u32_kernel(const uint8_t* __restrict__ f, uint32_t n, uint32_t* __restrict__ o) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = f[i];
}

void transmission_device(Ctx& ctx, const GridDev& grid, const SceneDev& scene, uint32_t tx_index, TxDev& out) {
  cudaStream_t s = ctx.stream;
  const uint32_t n = static_cast<uint32_t>(grid.n_ies);
  const V3 tx = load3(&scene.h_tx[3ull * tx_index]);
  const size_t m = n ? n : 1;
  DBuf<uint8_t> los(m, s), hit(m, s);
  DBuf<double> hp(3 * m, s), hn(3 * m, s), hi(3 * m, s);
  if (n) {
    count_launch();
    {
      KTimer kt(ctx, "transmission");
      transmission_kernel<<<walk_blocks(n, ctx.sm_count), 128, 0, s>>>(grid.view_for(ctx, scene), scene.view(), tx,
                                                     TxOut{los.get(), hit.get(), hp.get(), hn.get(), hi.get()});
    }
    PCR_LAUNCH_CHECK();
  }
  DBuf<uint32_t> f(m, s), lpos(m, s), hpos(m, s), tot(2, s);
  if (n) {
    count_launch();
    flags_u32_kernel<<<nb(n), kT, 0, s>>>(los.get(), n, f.get());
    exclusive_scan_u32(f.get(), lpos.get(), n, tot.get(), s);
    count_launch();
    flags_u32_kernel<<<nb(n), kT, 0, s>>>(hit.get(), n, f.get());
    exclusive_scan_u32(f.get(), hpos.get(), n, tot.get() + 1, s);
  } else {
    PCR_CUDA(cudaMemsetAsync(tot.get(), 0, 2 * sizeof(uint32_t), s));
  }
  uint32_t h_tot[2];
  d2h(h_tot, tot.get(), 2, s);
  stream_wait(s);
  out.n_los = h_tot[0];
  out.n_hits = h_tot[1];
  out.los_ie.alloc(out.n_los + 1, s);
  out.hit_ie.alloc(out.n_hits + 1, s);
  out.hit_kind.alloc(out.n_hits + 1, s);
  out.hit_pos.alloc(3ull * out.n_hits + 3, s);
  out.hit_nrm.alloc(3ull * out.n_hits + 3, s);
  out.hit_inc.alloc(3ull * out.n_hits + 3, s);
  if (n) {
    count_launch();
    compact_tx_kernel<<<nb(n), kT, 0, s>>>(los.get(), hit.get(), lpos.get(), hpos.get(), n, hp.get(), hn.get(),
                                           hi.get(), grid.view(), out.los_ie.get(), out.hit_ie.get(),
                                           out.hit_kind.get(), out.hit_pos.get(), out.hit_nrm.get(),
                                           out.hit_inc.get());
    PCR_LAUNCH_CHECK();
  }
}

namespace {

struct StackEntry {
  uint32_t node_begin, n_nodes;
  DBuf<uint64_t> prefix;
  DBuf<uint64_t> total;  // child rays of the range (device; read with the chunk's counters)
  uint64_t v_total, v_done;
  bool known;            // v_total read back yet
};

__global__ void count_alive_kernel(const Ray* __restrict__ rays, uint32_t n, unsigned long long* __restrict__ c) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  const bool a = k < n && rays[k].alive;
  const unsigned b = __ballot_sync(0xffffffffu, a);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(c, static_cast<unsigned long long>(__popc(b)));
}

}  // namespace

// First-kappa selection in DFS order; returns kept candidates (key order) in `out`.
static void kappa_select(Ctx& ctx, const GridDev& grid, const DBuf<Cand>& cands, uint32_t n, const Node* nodes,
                         const KeyLayout& L, int kappa, DBuf<Cand>& out, uint32_t& n_out,
                         DBuf<uint64_t>* keys_out = nullptr, DBuf<uint64_t>* hash_out = nullptr) {
  cudaStream_t s = ctx.stream;
  if (n == 0) {
    n_out = 0;
    return;
  }
  DBuf<uint64_t> keys(4ull * n, s), hash(n, s), tmp(n, s);
  count_launch();
  key_kernel<<<nb(n), kT, 0, s>>>(cands.get(), n, nodes, grid.view(), L, keys.get(), hash.get());
  PCR_LAUNCH_CHECK();
  DBuf<uint32_t> perm(n, s);
  iota_u32(perm.get(), n, s);
  // LSD over the key words, least significant first
  const int words = (L.total + 63) / 64;
  for (int q = words - 1; q >= 0; --q) {
    const int used = std::min(64, L.total - 64 * q);
    count_launch();
    gather_u64_kernel<<<nb(n), kT, 0, s>>>(keys.get() + static_cast<size_t>(q) * n, perm.get(), n, tmp.get());
    radix_sort_pairs(tmp.get(), perm.get(), n, 64 - used, 64, s);
  }
  DBuf<uint32_t> perm_key(n, s);
  PCR_CUDA(cudaMemcpyAsync(perm_key.get(), perm.get(), n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  count_launch();
  gather_u64_kernel<<<nb(n), kT, 0, s>>>(hash.get(), perm.get(), n, tmp.get());
  radix_sort_pairs(tmp.get(), perm.get(), n, 0, 64, s);
  DBuf<uint32_t> run_start(n, s);
  DBuf<int> collision(1, s);
  PCR_CUDA(cudaMemsetAsync(collision.get(), 0, sizeof(int), s));
  count_launch();
  rank_kernel<<<nb(n), kT, 0, s>>>(tmp.get(), perm.get(), n, cands.get(), nodes, grid.view(), run_start.get(),
                                   collision.get());
  PCR_LAUNCH_CHECK();
  // running max of run starts = start of each element's run
  {
    const uint32_t nblk = (n + 1023) / 1024;
    DBuf<uint32_t> bm(nblk, s);
    count_launch();
    run_max_block_kernel<<<nblk, 1024, 0, s>>>(run_start.get(), n, bm.get());
    if (nblk > 1) {
      count_launch();
      max_scan_small_kernel<<<1, 1, 0, s>>>(bm.get(), nblk);
      count_launch();
      run_max_fix_kernel<<<nblk, 1024, 0, s>>>(run_start.get(), n, bm.get());
    }
    PCR_LAUNCH_CHECK();
  }
  DBuf<uint8_t> keep(n, s);
  count_launch();
  keep_kernel<<<nb(n), kT, 0, s>>>(run_start.get(), perm.get(), n, kappa, keep.get());
  DBuf<uint32_t> flag(n, s), pos(n, s), tot(1, s);
  count_launch();
  keep_flags_in_order_kernel<<<nb(n), kT, 0, s>>>(keep.get(), perm_key.get(), n, flag.get());
  PCR_LAUNCH_CHECK();
  exclusive_scan_u32(flag.get(), pos.get(), n, tot.get(), s);
  int coll = 0;
  d2h(&coll, collision.get(), 1, s);
  d2h(&n_out, tot.get(), 1, s);
  stream_wait(s);
  if (coll) throw Error(4, "trace: group hash collision in kappa selection");
  DBuf<Cand> o(n_out ? n_out : 1, s);
  count_launch();
  compact_cands_kernel<<<nb(n), kT, 0, s>>>(cands.get(), perm_key.get(), flag.get(), pos.get(), n, o.get());
  PCR_LAUNCH_CHECK();
  if (keys_out && hash_out) {
    keys_out->alloc(4ull * (n_out ? n_out : 1), s);
    hash_out->alloc(n_out ? n_out : 1, s);
    count_launch();
    compact_keys_kernel<<<nb(n), kT, 0, s>>>(keys.get(), hash.get(), perm_key.get(), flag.get(), pos.get(), n, n_out,
                                             keys_out->get(), hash_out->get());
    PCR_LAUNCH_CHECK();
  }
  out = std::move(o);
}

// propagate for one TX from device initial hits; kept candidates materialised.
struct TraceWs {
  DBuf<Node> nodes;
  DBuf<Cand> cands;
  DBuf<Task> tasks;
};
static TraceWs& trace_ws(Ctx& ctx) {
  if (!ctx.trace_ws) ctx.trace_ws = std::shared_ptr<void>(new TraceWs(), [](void* p) { delete static_cast<TraceWs*>(p); });
  return *static_cast<TraceWs*>(ctx.trace_ws.get());
}

void propagate_device(Ctx& ctx, const GridDev& grid, const SceneDev& scene, uint32_t tx_index, const uint32_t* hit_ie,
                      const uint8_t* hit_kind, const double* hit_pos, const double* hit_nrm, const double* hit_inc,
                      uint32_t n_hits, const pcr_trace_params& p, CandDev& out, TraceStats& stats,
                      uint32_t shard, uint32_t n_shards, bool want_keys) {
  cudaStream_t s = ctx.stream;
  const TraceCfg c = make_cfg(p);
  out.n = 0;
  out.stride = static_cast<uint32_t>(std::max(1, p.max_interactions));
  if (n_shards == 0 || shard >= n_shards) throw Error(1, "trace: shard index out of range");
  // this shard's tasks: initial hits shard, shard + n_shards, ... (SURVEY 8e cyclic split)
  const uint32_t n_local = n_hits > shard ? (n_hits - shard + n_shards - 1) / n_shards : 0;
  if (p.max_interactions < 1 || n_local == 0) return;
  if (p.max_interactions > kMaxDepth) throw Error(1, "trace: max_interactions above the supported 8");
  if (p.max_diffractions >= 1 || true) ensure_fan(ctx, std::max(1, c.fan_n));
  const FanTable fan{ctx.fan_table.get(), c.fan_n};
  const GridView gv = grid.view_for(ctx, scene);
  const SceneView sv = scene.view();

  KeyLayout L;
  L.bits_task = std::max(1, bit_width(n_hits));
  L.bits_j = std::max(1, bit_width(static_cast<uint64_t>(std::max(1, c.fan_n))));
  L.bits_ie = std::max(1, bit_width(grid.n_ies));
  L.levels = c.max_interactions;
  L.total = L.bits_task + c.max_interactions * (L.bits_j + L.bits_ie);
  if (L.total > 256) throw Error(1, "trace: DFS key wider than 256 bits");

  // node arena
  size_t node_cap = std::max<size_t>(1u << 20, 2ull * n_local);
  // the node arena, candidate list and task buffer persist in the context across calls
  // (TraceWs): growing them inside the chunk loop maps new pool memory now and then,
  // measured as single 150-330 ms host stalls in a C2 trace stage of 1.3 s
  TraceWs& ws = trace_ws(ctx);
  struct Return {
    TraceWs& ws;
    DBuf<Node>& nodes;
    DBuf<Cand>& cands;
    DBuf<Task>& tasks;
    ~Return() {
      ws.nodes = std::move(nodes);
      ws.cands = std::move(cands);
      ws.tasks = std::move(tasks);
    }
  };
  DBuf<Node> nodes = std::move(ws.nodes);
  if (nodes.size() < node_cap) nodes.alloc(node_cap, s);
  node_cap = nodes.size();
  DBuf<uint32_t> counters(3, s);  // n_tasks, n_nodes, n_cands
  uint32_t n_nodes = n_local;
  count_launch();
  seed_kernel<<<nb(n_local), kT, 0, s>>>(hit_ie, hit_kind, hit_pos, hit_nrm, hit_inc, n_local, shard, n_shards, gv, sv,
                                         c, nodes.get());
  PCR_LAUNCH_CHECK();
  size_t cand_cap = 1u << 20;
  DBuf<Cand> cands = std::move(ws.cands);
  if (cands.size() < cand_cap) cands.alloc(cand_cap, s);
  cand_cap = cands.size();
  uint32_t n_cands = 0;
  const size_t kappa_trigger = 1u << 26;

  const uint32_t chunk = 1u << 18;
  DBuf<Ray> rays(chunk, s);
  size_t task_cap = 8ull * chunk;
  DBuf<Task> tasks = std::move(ws.tasks);
  if (tasks.size() < task_cap) tasks.alloc(task_cap, s);
  task_cap = tasks.size();
  Return give_back{ws, nodes, cands, tasks};
  DBuf<unsigned long long> alive(1, s);
  DBuf<unsigned long long> walk_stats(2, s);
  PCR_CUDA(cudaMemsetAsync(walk_stats.get(), 0, 2 * sizeof(unsigned long long), s));
  {
    const unsigned long long zero = 0;
    PCR_CUDA(cudaMemcpyToSymbolAsync(g_libm_unresolved, &zero, sizeof(zero), 0, cudaMemcpyHostToDevice, s));
  }

  std::vector<StackEntry> stack;
  auto push_range = [&](uint32_t begin, uint32_t count) {
    if (!count) return;
    StackEntry e;
    e.node_begin = begin;
    e.n_nodes = count;
    DBuf<uint64_t> cnt(count, s);
    e.prefix.alloc(count, s);
    count_launch();
    children_kernel<<<nb(count), kT, 0, s>>>(nodes.get(), begin, count, cnt.get());
    PCR_LAUNCH_CHECK();
    e.total.alloc(1, s);
    exclusive_scan_u64(cnt.get(), e.prefix.get(), count, e.total.get(), s);
    // the total is read with the next chunk's counters (no round trip here): until then
    // chunks are sized at the chunk bound and materialize clamps on the device total
    e.v_total = 0;
    e.known = false;
    e.v_done = 0;
    stack.push_back(std::move(e));
  };
  push_range(0, n_local);

  // development aid (PCR_TRACE_HOSTSTATS=1): host time of the chunk loop split into
  // time blocked in stream_wait and the rest, chunk and rerun counts, to stderr
  static const bool host_stats = std::getenv("PCR_TRACE_HOSTSTATS") != nullptr;
  using clk = std::chrono::steady_clock;
  double hs_wait = 0, hs_kappa = 0;
  uint64_t hs_chunks = 0, hs_reruns = 0, hs_grow = 0;
  const auto hs_t0 = clk::now();
  double hs_max_pre = 0, hs_max_post = 0, hs_pre = 0, hs_post = 0;
  auto hs_mark = clk::now();
  while (!stack.empty()) {
    StackEntry& top = stack.back();
    if (top.known && top.v_done >= top.v_total) {
      stack.pop_back();
      continue;
    }
    const uint32_t nr =
        static_cast<uint32_t>(top.known ? std::min<uint64_t>(chunk, top.v_total - top.v_done) : chunk);
    count_launch();
    {
      KTimer kt(ctx, "materialize");
      materialize_kernel<<<nb(nr), kT, 0, s>>>(nodes.get(), top.node_begin, top.prefix.get(), top.n_nodes,
                                               top.v_done, nr, top.total.get(), gv, sv, c, fan, rays.get());
    }
    PCR_LAUNCH_CHECK();
    const bool was_known = top.known;
    PCR_CUDA(cudaMemsetAsync(alive.get(), 0, sizeof(unsigned long long), s));
    count_launch();
    count_alive_kernel<<<nb(nr), kT, 0, s>>>(rays.get(), nr, alive.get());
    // walk -> tasks -> visibility with one host round trip: capacity for the worst case
    // (every task spawns) is reserved up front, the visibility kernel reads the task
    // count from the device, and an overflowing walk reruns with a bigger buffer
    uint32_t n_tasks = 0;
    unsigned long long h_alive = 0;
    const uint32_t before_nodes = n_nodes;
    for (;;) {
      if (n_nodes + task_cap > node_cap) {
        const size_t nc = std::max(node_cap * 2, n_nodes + task_cap + (1u << 20));
        if (nc > 0xfffffff0ull) throw Error(3, "trace: interaction arena exceeds 2^32 nodes");
        nodes.reserve(nc, n_nodes, s);
        node_cap = nc;
        ++hs_grow;
      }
      if (n_cands + task_cap > cand_cap) {
        const size_t nc = std::max(cand_cap * 2, n_cands + task_cap);
        cands.reserve(nc, n_cands, s);
        cand_cap = nc;
      }
      // tasks, nodes, candidates through the context's pinned scratch (see Ctx::pin)
      uint32_t* h_in = reinterpret_cast<uint32_t*>(ctx.pin);
      uint32_t* h_cnt = reinterpret_cast<uint32_t*>(ctx.pin + 8);
      unsigned long long* h_out = reinterpret_cast<unsigned long long*>(ctx.pin + 10);
      h_in[0] = 0;
      h_in[1] = n_nodes;
      h_in[2] = n_cands;
      h2d(counters.get(), h_in, 3, s);
      count_launch();
      {
        KTimer kt(ctx, "cone_walk");
        walk_kernel<<<walk_blocks(nr, ctx.sm_count), kWalkThreads, 0, s>>>(rays.get(), nr, gv, c, true,
                                                                            tasks.get(), counters.get(),
                                                static_cast<uint32_t>(task_cap), walk_stats.get());
      }
      PCR_LAUNCH_CHECK();
      count_launch();
      {
        KTimer kt(ctx, "visibility");
        visibility_kernel<<<walk_blocks(task_cap, ctx.sm_count), 128, 0, s>>>(
            tasks.get(), counters.get(), static_cast<uint32_t>(task_cap), rays.get(), nodes.get(), gv, sv, c,
            SpawnOut{nodes.get(), counters.get() + 1, cands.get(), counters.get() + 2, nullptr});
      }
      PCR_LAUNCH_CHECK();
      d2h(h_cnt, counters.get(), 3, s);
      d2h(h_out, alive.get(), 1, s);
      if (!top.known) d2h(reinterpret_cast<uint64_t*>(h_out + 1), top.total.get(), 1, s);
      const auto w0 = host_stats ? clk::now() : clk::time_point{};
      if (host_stats) {
        const double pre = std::chrono::duration<double>(w0 - hs_mark).count();
        hs_pre += pre;
        hs_max_pre = std::max(hs_max_pre, pre);
      }
      stream_wait(s);
      if (host_stats) {
        hs_mark = clk::now();
        hs_wait += std::chrono::duration<double>(hs_mark - w0).count();
        ++hs_chunks;
      }
      h_alive = h_out[0];
      if (!top.known) top.v_total = h_out[1];
      top.known = true;
      n_tasks = h_cnt[0];
      if (n_tasks <= task_cap) {
        n_nodes = h_cnt[1];
        n_cands = h_cnt[2];
        break;
      }
      task_cap = static_cast<size_t>(n_tasks) * 5 / 4 + 1024;  // visibility did nothing: rerun the chunk
      ++hs_reruns;
      tasks.alloc(task_cap, s);
    }
    top.v_done += was_known ? nr : std::min<uint64_t>(nr, top.v_total);
    stats.cone_traces += h_alive;
    stats.visibility_tests += n_tasks;
    if (n_tasks == 0) continue;
    if (n_cands > kappa_trigger) {
      const auto k0 = host_stats ? clk::now() : clk::time_point{};
      // exact pre-cap (a subset's first-kappa is a superset of its share of the global one)
      DBuf<Cand> kept;
      uint32_t nk = 0;
      kappa_select(ctx, grid, cands, n_cands, nodes.get(), L, c.kappa, kept, nk);
      cands.reserve(std::max<size_t>(cand_cap, nk), 0, s);
      PCR_CUDA(cudaMemcpyAsync(cands.get(), kept.get(), nk * sizeof(Cand), cudaMemcpyDeviceToDevice, s));
      n_cands = nk;
      if (host_stats) hs_kappa += std::chrono::duration<double>(clk::now() - k0).count();
    }
    // `top` may be invalidated by push_range; nothing below uses it.
    push_range(before_nodes, n_nodes - before_nodes);
    if (host_stats) {
      const auto now = clk::now();
      const double post = std::chrono::duration<double>(now - hs_mark).count();
      hs_post += post;
      hs_max_post = std::max(hs_max_post, post);
      hs_mark = now;
    }
  }

  if (host_stats)
    std::fprintf(stderr, "trace loop: %.3f s, in stream_wait %.3f s, before waits %.3f s (max %.4f), after %.3f s (max %.4f), kappa pre-cap %.3f s, chunks %llu, reruns %llu, arena grows %llu\n",
                 std::chrono::duration<double>(clk::now() - hs_t0).count(), hs_wait, hs_pre, hs_max_pre, hs_post, hs_max_post, hs_kappa,
                 static_cast<unsigned long long>(hs_chunks), static_cast<unsigned long long>(hs_reruns),
                 static_cast<unsigned long long>(hs_grow));
  DBuf<Cand> kept;
  uint32_t nk = 0;
  {
    KTimer kt(ctx, "kappa_select");
    kappa_select(ctx, grid, cands, n_cands, nodes.get(), L, c.kappa, kept, nk, want_keys ? &out.keys : nullptr,
                 want_keys ? &out.hash : nullptr);
  }
  out.n = nk;
  const size_t m = nk ? nk : 1;
  const size_t ms = m * out.stride;
  out.rx_id.alloc(m, s);
  out.n_inter.alloc(m, s);
  out.rx_pos.alloc(3 * m, s);
  out.length.alloc(m, s);
  out.kind.alloc(ms, s);
  out.pos.alloc(3 * ms, s);
  out.label.alloc(ms, s);
  out.nrm.alloc(3 * ms, s);
  out.ie.alloc(ms, s);
  out.edge.alloc(ms, s);
  PCR_CUDA(cudaMemsetAsync(out.kind.get(), 0, ms, s));
  PCR_CUDA(cudaMemsetAsync(out.pos.get(), 0, 3 * ms * sizeof(double), s));
  PCR_CUDA(cudaMemsetAsync(out.nrm.get(), 0, 3 * ms * sizeof(double), s));
  PCR_CUDA(cudaMemsetAsync(out.label.get(), 0, ms * sizeof(uint32_t), s));
  PCR_CUDA(cudaMemsetAsync(out.ie.get(), 0, ms * sizeof(uint32_t), s));
  PCR_CUDA(cudaMemsetAsync(out.edge.get(), 0, ms * sizeof(uint32_t), s));
  if (nk) {
    CandOut co{out.stride,     out.rx_id.get(), out.rx_pos.get(), out.length.get(), out.n_inter.get(),
               out.kind.get(), out.pos.get(),   out.label.get(),  out.nrm.get(),    out.ie.get(),
               out.edge.get()};
    count_launch();
    materialize_cands_kernel<<<nb(nk), kT, 0, s>>>(kept.get(), nk, nodes.get(), gv, load3(&scene.h_tx[3ull * tx_index]),
                                                   co);
    PCR_LAUNCH_CHECK();
  }
  unsigned long long wst[2] = {0, 0}, unresolved = 0;
  d2h(wst, walk_stats.get(), 2, s);
  PCR_CUDA(cudaMemcpyFromSymbolAsync(&unresolved, g_libm_unresolved, sizeof(unresolved), 0, cudaMemcpyDeviceToHost, s));
  stream_wait(s);
  stats.walk_cells += wst[0];
  stats.walk_ies += wst[1];
  stats.libm_unresolved += unresolved;
}

// ---- sharded propagation: candidate rows and the global kappa merge ---------
namespace {

__global__ void pack_rows_kernel(uint32_t n, uint32_t stride, uint32_t tx_index, const uint32_t* __restrict__ rx_id,
                                 const uint32_t* __restrict__ n_inter, const double* __restrict__ rx_pos,
                                 const double* __restrict__ length, const uint8_t* __restrict__ kind,
                                 const double* __restrict__ pos, const uint32_t* __restrict__ label,
                                 const double* __restrict__ nrm, const uint32_t* __restrict__ ie,
                                 const uint32_t* __restrict__ edge, const uint64_t* __restrict__ keys,
                                 const uint64_t* __restrict__ hash, uint8_t* __restrict__ rows) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  uint8_t* r = rows + static_cast<size_t>(k) * cand_row_bytes(stride);
  CandRowHead h;
  for (int q = 0; q < 4; ++q) h.key[q] = keys[static_cast<size_t>(q) * n + k];
  h.hash = hash[k];
  h.tx_index = tx_index;
  h.rx_id = rx_id[k];
  h.n_inter = n_inter[k];
  h.pad0 = 0;
  for (int a = 0; a < 3; ++a) h.rx_pos[a] = rx_pos[3ull * k + a];
  h.length = length[k];
  h.pad1 = 0.0;
  *reinterpret_cast<CandRowHead*>(r) = h;
  CandRowLevel* lv = reinterpret_cast<CandRowLevel*>(r + sizeof(CandRowHead));
  for (uint32_t q = 0; q < stride; ++q) {
    const size_t j = static_cast<size_t>(k) * stride + q;
    CandRowLevel l;
    for (int a = 0; a < 3; ++a) {
      l.pos[a] = pos[3 * j + a];
      l.nrm[a] = nrm[3 * j + a];
    }
    l.label = label[j];
    l.ie = ie[j];
    l.edge = edge[j];
    l.kind = kind[j];
    lv[q] = l;
  }
}

__device__ __forceinline__ const CandRowHead& row_head(const uint8_t* rows, size_t bytes, uint32_t i) {
  return *reinterpret_cast<const CandRowHead*>(rows + static_cast<size_t>(i) * bytes);
}

// word q of every row's key (q = 4: tx index), through perm
__global__ void row_word_kernel(const uint8_t* __restrict__ rows, size_t bytes, const uint32_t* __restrict__ perm,
                                uint32_t n, int q, uint64_t* __restrict__ out) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const CandRowHead& h = row_head(rows, bytes, perm[k]);
  out[k] = q < 4 ? h.key[q] : q == 4 ? static_cast<uint64_t>(h.tx_index) : h.hash;
}

__device__ bool same_row_group(const uint8_t* rows, size_t bytes, uint32_t a, uint32_t b) {
  const CandRowHead& x = row_head(rows, bytes, a);
  const CandRowHead& y = row_head(rows, bytes, b);
  if (x.tx_index != y.tx_index || x.rx_id != y.rx_id || x.n_inter != y.n_inter) return false;
  const CandRowLevel* lx = reinterpret_cast<const CandRowLevel*>(rows + static_cast<size_t>(a) * bytes + sizeof(CandRowHead));
  const CandRowLevel* ly = reinterpret_cast<const CandRowLevel*>(rows + static_cast<size_t>(b) * bytes + sizeof(CandRowHead));
  for (uint32_t q = 0; q < x.n_inter; ++q)
    if (lx[q].label != ly[q].label) return false;
  return true;
}

// rows in (tx, hash, key) order: run heads, with every non-head checked to be in the
// same (tx, rx, labels) group as its predecessor (a hash collision is an error)
__global__ void row_rank_kernel(const uint8_t* __restrict__ rows, size_t bytes, const uint32_t* __restrict__ perm,
                                uint32_t n, uint32_t* __restrict__ run_start, int* __restrict__ collision) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  bool head = k == 0;
  if (!head) {
    const CandRowHead& a = row_head(rows, bytes, perm[k]);
    const CandRowHead& b = row_head(rows, bytes, perm[k - 1]);
    head = a.tx_index != b.tx_index || a.hash != b.hash;
    if (!head && !same_row_group(rows, bytes, perm[k], perm[k - 1])) *collision = 1;
  }
  run_start[k] = head ? k : 0;
}

__global__ void unpack_rows_kernel(const uint8_t* __restrict__ rows, uint32_t stride, const uint32_t* __restrict__ perm,
                                   const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos, uint32_t n,
                                   CandOut o, uint32_t* __restrict__ per_tx) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n || !flag[k]) return;
  const size_t bytes = cand_row_bytes(stride);
  const uint8_t* r = rows + static_cast<size_t>(perm[k]) * bytes;
  const CandRowHead& h = *reinterpret_cast<const CandRowHead*>(r);
  const CandRowLevel* lv = reinterpret_cast<const CandRowLevel*>(r + sizeof(CandRowHead));
  const uint32_t d = pos[k];
  o.rx_id[d] = h.rx_id;
  o.n_inter[d] = h.n_inter;
  for (int a = 0; a < 3; ++a) o.rx_pos[3ull * d + a] = h.rx_pos[a];
  o.length[d] = h.length;
  for (uint32_t q = 0; q < stride; ++q) {
    const size_t j = static_cast<size_t>(d) * stride + q;
    for (int a = 0; a < 3; ++a) {
      o.pos[3 * j + a] = lv[q].pos[a];
      o.nrm[3 * j + a] = lv[q].nrm[a];
    }
    o.label[j] = lv[q].label;
    o.ie[j] = lv[q].ie;
    o.edge[j] = lv[q].edge;
    o.kind[j] = static_cast<uint8_t>(lv[q].kind);
  }
  atomicAdd(per_tx + h.tx_index, 1u);
}

}  // namespace

void pack_cand_rows(Ctx& ctx, const CandDev& c, uint32_t tx_index, uint8_t* rows) {
  if (!c.n) return;
  if (!c.keys.get() || !c.hash.get()) throw Error(1, "trace: candidate rows need DFS keys");
  count_launch();
  pack_rows_kernel<<<nb(c.n), kT, 0, ctx.stream>>>(c.n, c.stride, tx_index, c.rx_id.get(), c.n_inter.get(),
                                                   c.rx_pos.get(), c.length.get(), c.kind.get(), c.pos.get(),
                                                   c.label.get(), c.nrm.get(), c.ie.get(), c.edge.get(),
                                                   c.keys.get(), c.hash.get(), rows);
  PCR_LAUNCH_CHECK();
}

// Global first-kappa over every shard's rows, concatenated in any order: the rows are
// put in (tx, DFS key) order — the reference's emission order per TX — and grouped by
// (tx, rx, label sequence); the first kappa of each group survive. Every shard kept the
// first kappa of its own subset of each group, a superset of its share of the global
// first kappa (T9), so the result equals the unsharded propagate. Output: all TXs'
// kept candidates in (tx, key) order and the number per TX.
void kappa_merge_rows(Ctx& ctx, const uint8_t* rows, uint64_t n64, uint32_t stride, int kappa, uint32_t n_tx,
                      CandDev& out, std::vector<uint32_t>& per_tx) {
  cudaStream_t s = ctx.stream;
  per_tx.assign(n_tx, 0);
  out.n = 0;
  out.stride = stride;
  if (n64 > 0xffffffffull) throw Error(PCR_ERR_NOMEM, "trace: too many candidate rows");
  const uint32_t n = static_cast<uint32_t>(n64);
  const size_t bytes = cand_row_bytes(stride);
  const size_t m = n ? n : 1, ms = m * stride;
  out.rx_id.alloc(m, s);
  out.n_inter.alloc(m, s);
  out.rx_pos.alloc(3 * m, s);
  out.length.alloc(m, s);
  out.kind.alloc(ms, s);
  out.pos.alloc(3 * ms, s);
  out.label.alloc(ms, s);
  out.nrm.alloc(3 * ms, s);
  out.ie.alloc(ms, s);
  out.edge.alloc(ms, s);
  if (!n) return;
  KTimer kt(ctx, "kappa_merge");
  DBuf<uint32_t> perm_key(n, s), perm(n, s);
  DBuf<uint64_t> tmp(n, s);
  iota_u32(perm_key.get(), n, s);
  // LSD: key words least significant first, then the TX index
  const int order[5] = {3, 2, 1, 0, 4};
  for (int w : order) {
    count_launch();
    row_word_kernel<<<nb(n), kT, 0, s>>>(rows, bytes, perm_key.get(), n, w, tmp.get());
    PCR_LAUNCH_CHECK();
    radix_sort_pairs(tmp.get(), perm_key.get(), n, 0, w == 4 ? 32 : 64, s);
  }
  // group order (tx, hash, key): stable sorts of the key order by hash, then by tx
  PCR_CUDA(cudaMemcpyAsync(perm.get(), perm_key.get(), n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  for (int w : {5, 4}) {
    count_launch();
    row_word_kernel<<<nb(n), kT, 0, s>>>(rows, bytes, perm.get(), n, w, tmp.get());
    PCR_LAUNCH_CHECK();
    radix_sort_pairs(tmp.get(), perm.get(), n, 0, w == 4 ? 32 : 64, s);
  }
  DBuf<uint32_t> run_start(n, s);
  DBuf<int> collision(1, s);
  PCR_CUDA(cudaMemsetAsync(collision.get(), 0, sizeof(int), s));
  count_launch();
  row_rank_kernel<<<nb(n), kT, 0, s>>>(rows, bytes, perm.get(), n, run_start.get(), collision.get());
  PCR_LAUNCH_CHECK();
  {
    const uint32_t nblk = (n + 1023) / 1024;
    DBuf<uint32_t> bm(nblk, s);
    count_launch();
    run_max_block_kernel<<<nblk, 1024, 0, s>>>(run_start.get(), n, bm.get());
    if (nblk > 1) {
      count_launch();
      max_scan_small_kernel<<<1, 1, 0, s>>>(bm.get(), nblk);
      count_launch();
      run_max_fix_kernel<<<nblk, 1024, 0, s>>>(run_start.get(), n, bm.get());
    }
    PCR_LAUNCH_CHECK();
  }
  DBuf<uint8_t> keep(n, s);
  count_launch();
  keep_kernel<<<nb(n), kT, 0, s>>>(run_start.get(), perm.get(), n, kappa, keep.get());
  DBuf<uint32_t> flag(n, s), pos(n, s), tot(1, s);
  count_launch();
  keep_flags_in_order_kernel<<<nb(n), kT, 0, s>>>(keep.get(), perm_key.get(), n, flag.get());
  PCR_LAUNCH_CHECK();
  exclusive_scan_u32(flag.get(), pos.get(), n, tot.get(), s);
  DBuf<uint32_t> cnt(n_tx ? n_tx : 1, s);
  PCR_CUDA(cudaMemsetAsync(cnt.get(), 0, (n_tx ? n_tx : 1) * sizeof(uint32_t), s));
  CandOut co{stride,         out.rx_id.get(), out.rx_pos.get(), out.length.get(), out.n_inter.get(),
             out.kind.get(), out.pos.get(),   out.label.get(),  out.nrm.get(),    out.ie.get(),
             out.edge.get()};
  count_launch();
  unpack_rows_kernel<<<nb(n), kT, 0, s>>>(rows, stride, perm_key.get(), flag.get(), pos.get(), n, co, cnt.get());
  PCR_LAUNCH_CHECK();
  int coll = 0;
  uint32_t n_out = 0;
  d2h(&coll, collision.get(), 1, s);
  d2h(&n_out, tot.get(), 1, s);
  if (n_tx) d2h(per_tx.data(), cnt.get(), n_tx, s);
  stream_wait(s);
  if (coll) throw Error(4, "trace: group hash collision in kappa selection");
  out.n = n_out;
}

// ---- C-ABI adapters ---------------------------------------------------------------------
static void fill_paths_from_cands(const CandDev& cd, uint32_t tx_id, const double* txp, pcr_paths* p, size_t row0,
                                  cudaStream_t s) {
  const size_t n = cd.n;
  if (!n) return;
  std::vector<uint32_t> rx(n), ni(n), lab(n * cd.stride), ie(n * cd.stride), ed(n * cd.stride);
  std::vector<uint8_t> kind(n * cd.stride);
  std::vector<double> rxp(3 * n), len(n), pos(3 * n * cd.stride), nrm(3 * n * cd.stride);
  d2h(rx.data(), cd.rx_id.get(), n, s);
  d2h(ni.data(), cd.n_inter.get(), n, s);
  d2h(lab.data(), cd.label.get(), lab.size(), s);
  d2h(ie.data(), cd.ie.get(), ie.size(), s);
  d2h(ed.data(), cd.edge.get(), ed.size(), s);
  d2h(kind.data(), cd.kind.get(), kind.size(), s);
  d2h(rxp.data(), cd.rx_pos.get(), rxp.size(), s);
  d2h(len.data(), cd.length.get(), n, s);
  d2h(pos.data(), cd.pos.get(), pos.size(), s);
  d2h(nrm.data(), cd.nrm.get(), nrm.size(), s);
  stream_wait(s);
  for (size_t k = 0; k < n; ++k) {
    const size_t r = row0 + k;
    p->tx_id[r] = tx_id;
    p->rx_id[r] = rx[k];
    std::memcpy(p->tx_position + 3 * r, txp, 3 * sizeof(double));
    std::memcpy(p->rx_position + 3 * r, &rxp[3 * k], 3 * sizeof(double));
    p->length[r] = len[k];
    p->n_inter[r] = ni[k];
    for (uint32_t l = 0; l < ni[k] && l < p->stride; ++l) {
      const size_t q = r * p->stride + l, src = k * cd.stride + l;
      p->kind[q] = kind[src];
      std::memcpy(p->position + 3 * q, &pos[3 * src], 3 * sizeof(double));
      p->label[q] = lab[src];
      std::memcpy(p->normal + 3 * q, &nrm[3 * src], 3 * sizeof(double));
      p->ie_index[q] = ie[src];
      p->edge_index[q] = ed[src];
    }
  }
}

void api_transmission(Ctx& ctx, const GridDev& grid, const SceneDev& scene, uint32_t tx_index,
                      const pcr_trace_params& p, pcr_paths** los_out, pcr_initial_hits** hits_out) {
  (void)p;
  if (tx_index >= scene.h_tx_id.size()) throw Error(1, "trace: tx index out of range");
  cudaStream_t s = ctx.stream;
  TxDev t;
  transmission_device(ctx, grid, scene, tx_index, t);
  std::vector<uint32_t> los_ie(t.n_los);
  d2h(los_ie.data(), t.los_ie.get(), t.n_los, s);
  pcr_initial_hits* h = halloc<pcr_initial_hits>(1);
  h->n = t.n_hits;
  h->ie_index = halloc<uint32_t>(t.n_hits);
  h->kind = halloc<uint8_t>(t.n_hits);
  h->position = halloc<double>(3ull * t.n_hits);
  h->normal = halloc<double>(3ull * t.n_hits);
  h->incoming = halloc<double>(3ull * t.n_hits);
  d2h(h->ie_index, t.hit_ie.get(), t.n_hits, s);
  d2h(h->kind, t.hit_kind.get(), t.n_hits, s);
  d2h(h->position, t.hit_pos.get(), 3ull * t.n_hits, s);
  d2h(h->normal, t.hit_nrm.get(), 3ull * t.n_hits, s);
  d2h(h->incoming, t.hit_inc.get(), 3ull * t.n_hits, s);
  std::vector<double4> rp(grid.n_ies);
  std::vector<uint32_t> rxid(grid.n_ies);
  d2h(rp.data(), grid.rp.get(), grid.n_ies, s);
  d2h(rxid.data(), grid.rx.get(), grid.n_ies, s);
  stream_wait(s);
  pcr_paths* los = alloc_paths(t.n_los, 1);
  const double* txp = &scene.h_tx[3ull * tx_index];
  for (uint32_t k = 0; k < t.n_los; ++k) {
    const uint32_t i = los_ie[k];
    los->tx_id[k] = scene.h_tx_id[tx_index];
    los->rx_id[k] = rxid[i];
    std::memcpy(los->tx_position + 3 * k, txp, 3 * sizeof(double));
    const double r3[3] = {rp[i].x, rp[i].y, rp[i].z};
    std::memcpy(los->rx_position + 3 * k, r3, 3 * sizeof(double));
    const V3 d = V3{r3[0], r3[1], r3[2]} - V3{txp[0], txp[1], txp[2]};
    los->length[k] = norm(d);
  }
  *los_out = los;
  *hits_out = h;
}

void api_propagate(Ctx& ctx, const GridDev& grid, const SceneDev& scene, uint32_t tx_index,
                   const pcr_initial_hits& hits, const pcr_trace_params& p, pcr_paths** out) {
  if (tx_index >= scene.h_tx_id.size()) throw Error(1, "trace: tx index out of range");
  cudaStream_t s = ctx.stream;
  const size_t n = hits.n;
  const size_t m = n ? n : 1;
  DBuf<uint32_t> ie(m, s);
  DBuf<uint8_t> kind(m, s);
  DBuf<double> pos(3 * m, s), nrm(3 * m, s), inc(3 * m, s);
  h2d(ie.get(), hits.ie_index, n, s);
  h2d(kind.get(), hits.kind, n, s);
  h2d(pos.get(), hits.position, 3 * n, s);
  h2d(nrm.get(), hits.normal, 3 * n, s);
  h2d(inc.get(), hits.incoming, 3 * n, s);
  CandDev cd;
  TraceStats st;
  propagate_device(ctx, grid, scene, tx_index, ie.get(), kind.get(), pos.get(), nrm.get(), inc.get(),
                   static_cast<uint32_t>(n), p, cd, st);
  ctx.last_trace[0] = st.cone_traces;
  ctx.last_trace[1] = st.visibility_tests;
  ctx.last_trace[2] = st.walk_cells;
  ctx.last_trace[3] = st.walk_ies;
  ctx.last_trace[4] = st.libm_unresolved;
  pcr_paths* r = alloc_paths(cd.n, cd.stride);
  fill_paths_from_cands(cd, scene.h_tx_id[tx_index], &scene.h_tx[3ull * tx_index], r, 0, s);
  *out = r;
}

void api_cone_trace_batch(Ctx& ctx, const GridDev& grid, const SceneDev& scene, const pcr_ray_desc* rays_h,
                          uint64_t n_rays, bool want_debug, pcr_receptions** out) {
  cudaStream_t s = ctx.stream;
  const size_t m = n_rays ? n_rays : 1;
  DBuf<pcr_ray_desc> desc(m, s);
  h2d(desc.get(), rays_h, n_rays, s);
  DBuf<Ray> rays(m, s);
  TraceCfg c{};
  c.max_interactions = 1 << 20;
  c.max_diffractions = 1 << 20;
  if (n_rays) {
    count_launch();
    rays_from_desc_kernel<<<nb(n_rays), kT, 0, s>>>(desc.get(), n_rays, rays.get());
    PCR_LAUNCH_CHECK();
  }
  const GridView gv = grid.view_for(ctx, scene);
  const SceneView sv = scene.view();
  size_t cap = std::max<size_t>(1024, 64 * m);
  DBuf<Task> tasks(cap, s);
  DBuf<uint32_t> cnt(1, s);
  uint32_t nt = 0;
  for (;;) {
    PCR_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(uint32_t), s));
    if (n_rays) {
      count_launch();
      walk_kernel<<<walk_blocks(n_rays, ctx.sm_count), kWalkThreads, 0, s>>>(rays.get(),
                                                                              static_cast<uint32_t>(n_rays), gv, c,
                                                                              false,
                                                  tasks.get(), cnt.get(), static_cast<uint32_t>(cap), nullptr);
      PCR_LAUNCH_CHECK();
    }
    d2h(&nt, cnt.get(), 1, s);
    stream_wait(s);
    if (nt <= cap) break;
    cap = nt + 1024;
    tasks.alloc(cap, s);
  }
  const size_t mt = nt ? nt : 1;
  DBuf<uint8_t> ok(mt, s), hv(mt, s);
  DBuf<double> hp(3 * mt, s), hn(3 * mt, s), hd(mt, s);
  DBuf<uint32_t> hl(mt, s);
  if (nt) {
    count_launch();
    reception_kernel<<<nb(nt, 128), 128, 0, s>>>(tasks.get(), nt, rays.get(), gv, sv,
                                                 RecOut{ok.get(), hv.get(), hp.get(), hn.get(), hl.get(), hd.get()});
    PCR_LAUNCH_CHECK();
  }
  std::vector<Task> ht(nt);
  std::vector<uint8_t> hok(nt), hhv(nt);
  std::vector<double> hhp(3 * nt), hhn(3 * nt), hhd(nt);
  std::vector<uint32_t> hhl(nt);
  d2h(ht.data(), tasks.get(), nt, s);
  d2h(hok.data(), ok.get(), nt, s);
  d2h(hhv.data(), hv.get(), nt, s);
  d2h(hhp.data(), hp.get(), 3 * nt, s);
  d2h(hhn.data(), hn.get(), 3 * nt, s);
  d2h(hhd.data(), hd.get(), nt, s);
  d2h(hhl.data(), hl.get(), nt, s);
  std::vector<double4> rp(grid.n_ies);
  d2h(rp.data(), grid.rp.get(), grid.n_ies, s);
  // evaluated cells (TraceDebug)
  std::vector<uint64_t> eoff(n_rays + 1, 0);
  std::vector<uint32_t> ev;
  if (want_debug && n_rays) {
    DBuf<uint32_t> ecnt(m, s);
    count_launch();
    evaluated_kernel<<<nb(n_rays, 128), 128, 0, s>>>(rays.get(), static_cast<uint32_t>(n_rays), gv, nullptr,
                                                     ecnt.get(), nullptr);
    PCR_LAUNCH_CHECK();
    std::vector<uint32_t> hc(n_rays);
    d2h(hc.data(), ecnt.get(), n_rays, s);
    stream_wait(s);
    for (size_t k = 0; k < n_rays; ++k) eoff[k + 1] = eoff[k] + hc[k];
    DBuf<uint64_t> doff(n_rays + 1, s);
    h2d(doff.get(), eoff.data(), n_rays + 1, s);
    DBuf<uint32_t> dev(eoff[n_rays] ? eoff[n_rays] : 1, s);
    count_launch();
    evaluated_kernel<<<nb(n_rays, 128), 128, 0, s>>>(rays.get(), static_cast<uint32_t>(n_rays), gv, doff.get(),
                                                     nullptr, dev.get());
    PCR_LAUNCH_CHECK();
    ev.resize(eoff[n_rays]);
    d2h(ev.data(), dev.get(), ev.size(), s);
  }
  // visited voxels (TraceDebug)
  std::vector<uint64_t> voff(n_rays + 1, 0);
  std::vector<uint32_t> vv;
  if (want_debug && n_rays) {
    DBuf<uint32_t> vcnt(m, s);
    count_launch();
    visited_kernel<<<nb(n_rays, 128), 128, 0, s>>>(rays.get(), static_cast<uint32_t>(n_rays), gv, nullptr,
                                                   vcnt.get(), nullptr);
    PCR_LAUNCH_CHECK();
    std::vector<uint32_t> hc(n_rays);
    d2h(hc.data(), vcnt.get(), n_rays, s);
    stream_wait(s);
    for (size_t k = 0; k < n_rays; ++k) voff[k + 1] = voff[k] + hc[k];
    DBuf<uint64_t> doff(n_rays + 1, s);
    h2d(doff.get(), voff.data(), n_rays + 1, s);
    DBuf<uint32_t> dvv(voff[n_rays] ? voff[n_rays] : 1, s);
    count_launch();
    visited_kernel<<<nb(n_rays, 128), 128, 0, s>>>(rays.get(), static_cast<uint32_t>(n_rays), gv, doff.get(),
                                                   nullptr, dvv.get());
    PCR_LAUNCH_CHECK();
    vv.resize(voff[n_rays]);
    d2h(vv.data(), dvv.get(), vv.size(), s);
  }
  stream_wait(s);
  // group by ray, ascending ie (tracer.cpp:400-401)
  std::vector<uint32_t> order;
  order.reserve(nt);
  for (uint32_t t = 0; t < nt; ++t)
    if (hok[t]) order.push_back(t);
  std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
    return ht[a].ray != ht[b].ray ? ht[a].ray < ht[b].ray : ht[a].ie < ht[b].ie;
  });
  pcr_receptions* r = halloc<pcr_receptions>(1);
  const size_t nrec = order.size();
  r->n_rays = n_rays;
  r->n = nrec;
  r->ray_offset = halloc<uint64_t>(n_rays + 1);
  r->ie_index = halloc<uint32_t>(nrec);
  r->reception_point = halloc<double>(3 * nrec);
  r->hit_valid = halloc<uint8_t>(nrec);
  r->hit_position = halloc<double>(3 * nrec);
  r->hit_normal = halloc<double>(3 * nrec);
  r->hit_label = halloc<uint32_t>(nrec);
  r->hit_distance = halloc<double>(nrec);
  r->evaluated_offset = halloc<uint64_t>(n_rays + 1);
  r->evaluated = halloc<uint32_t>(ev.size());
  r->visited_offset = halloc<uint64_t>(n_rays + 1);
  r->visited = halloc<uint32_t>(vv.size());
  size_t k = 0;
  for (uint64_t ray = 0; ray < n_rays; ++ray) {
    r->ray_offset[ray] = k;
    while (k < nrec && ht[order[k]].ray == ray) {
      const uint32_t t = order[k];
      const uint32_t i = ht[t].ie;
      r->ie_index[k] = i;
      r->reception_point[3 * k] = rp[i].x;
      r->reception_point[3 * k + 1] = rp[i].y;
      r->reception_point[3 * k + 2] = rp[i].z;
      r->hit_valid[k] = hhv[t];
      if (hhv[t]) {
        std::memcpy(r->hit_position + 3 * k, &hhp[3 * t], 3 * sizeof(double));
        std::memcpy(r->hit_normal + 3 * k, &hhn[3 * t], 3 * sizeof(double));
        r->hit_label[k] = hhl[t];
        r->hit_distance[k] = hhd[t];
      } else {
        r->hit_normal[3 * k + 2] = 1.0;  // SurfaceHit default normal UnitZ
      }
      ++k;
    }
  }
  r->ray_offset[n_rays] = k;
  for (uint64_t ray = 0; ray <= n_rays; ++ray) r->evaluated_offset[ray] = eoff[ray];
  if (!ev.empty()) std::memcpy(r->evaluated, ev.data(), ev.size() * sizeof(uint32_t));
  for (uint64_t ray = 0; ray <= n_rays; ++ray) r->visited_offset[ray] = voff[ray];
  if (!vv.empty()) std::memcpy(r->visited, vv.data(), vv.size() * sizeof(uint32_t));
  *out = r;
}

void api_segment_visible_batch(Ctx& ctx, const GridDev& grid, const SceneDev& scene, const double* origin,
                               const double* target, const uint32_t* target_ie, uint64_t n, uint8_t* visible_out) {
  if (!n) return;
  cudaStream_t s = ctx.stream;
  DBuf<double> o(3 * n, s), t(3 * n, s);
  DBuf<uint32_t> ti(n, s);
  DBuf<uint8_t> vis(n, s);
  h2d(o.get(), origin, 3 * n, s);
  h2d(t.get(), target, 3 * n, s);
  h2d(ti.get(), target_ie, n, s);
  count_launch();
  segvis_kernel<<<walk_blocks((n + 1) / 2, ctx.sm_count), 128, 0, s>>>(o.get(), t.get(), ti.get(), n, grid.view_for(ctx, scene),
                                                                       scene.view(), vis.get());
  PCR_LAUNCH_CHECK();
  d2h(visible_out, vis.get(), n, s);
  stream_wait(s);
}

}  // namespace pcr
