// pipeline.cu — run_pipeline_on_scene (proj/src/pipeline.cpp:99-212) over the
// device stages: validate_scene (scene.cpp:31-91) on the device, the stage calls,
// dedup_by_label / dedup_by_fresnel (refine.cpp:288-372) and the final output order
// (pipeline.cpp:194-207) on the device, config_hash (pipeline.cpp:89-97); plus the
// sharded variant of the same run.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <unordered_set>
#include <vector>

#include "host_alloc.hpp"
#include "pipeline.hpp"
#include "shard_rows.cuh"
#include "sort.cuh"
#include "stages.cuh"
#include "trace.cuh"

namespace pcr {

namespace {

constexpr double kC = 299792458.0;
using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

// ---- config -----------------------------------------------------------------------------
uint64_t fnv1a(const char* s) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (; *s; ++s) {
    h ^= static_cast<unsigned char>(*s);
    h *= 0x100000001b3ull;
  }
  return h;
}

// ---- validate_scene (scene.cpp:31-91) ---------------------------------------------------------
// The O(N) point checks run on the device (SURVEY §8f "next" #1): the first offending
// point index (atomicMin) and, per edge, whether any point carries its label. Edges and
// radios are few and are checked on the host in the reference's report order.
struct Violation {
  std::string rule, detail;
  size_t index;
};

__global__ void validate_points_kernel(const double* __restrict__ pos, const double* __restrict__ nrm,
                                       const uint32_t* __restrict__ label, uint64_t n,
                                       const uint32_t* __restrict__ edge_label, uint32_t n_edges,
                                       unsigned long long* __restrict__ first_bad, uint32_t* __restrict__ label_hit) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const V3 p = load3(pos + 3 * i), q = load3(nrm + 3 * i);
    const bool finite = isfinite(p.x) && isfinite(p.y) && isfinite(p.z);
    const double nn = norm(q);
    if (!finite || fabs(nn - 1.0) > 1e-6) atomicMin(first_bad, static_cast<unsigned long long>(i));
    const uint32_t l = label[i];
    for (uint32_t e = 0; e < n_edges; ++e)
      if (edge_label[e] == l && !label_hit[e]) label_hit[e] = 1;
  }
}

bool first_violation_device(Ctx& ctx, const SceneDev& S, Violation& v) {
  cudaStream_t s = ctx.stream;
  DBuf<unsigned long long> first(1, s);
  DBuf<uint32_t> hit(S.n_edges + 1ull, s);
  const unsigned long long none = ~0ull;
  h2d(first.get(), &none, 1, s);
  PCR_CUDA(cudaMemsetAsync(hit.get(), 0, (S.n_edges + 1ull) * sizeof(uint32_t), s));
  if (S.n_points) {
    count_launch();
    KTimer kt(ctx, "validate");
    validate_points_kernel<<<blocks_for(S.n_points, 256, 148u * 8u), 256, 0, s>>>(
        S.pos.get(), S.nrm.get(), S.label.get(), S.n_points, S.edge_label.get(), S.n_edges, first.get(), hit.get());
    PCR_LAUNCH_CHECK();
  }
  unsigned long long fb = none;
  std::vector<uint32_t> lh(S.n_edges + 1ull);
  d2h(&fb, first.get(), 1, s);
  d2h(lh.data(), hit.get(), lh.size(), s);
  stream_wait(s);
  std::vector<Violation> out;
  auto add = [&](const std::string& rule, size_t i, const std::string& detail) {
    if (out.empty()) out.push_back({rule, detail, i});
  };
  if (fb != none) {
    double p[3], q[3];
    d2h(p, S.pos.get() + 3 * fb, 3, s);
    d2h(q, S.nrm.get() + 3 * fb, 3, s);
    stream_wait(s);
    if (!(std::isfinite(p[0]) && std::isfinite(p[1]) && std::isfinite(p[2])))
      add("point_position_finite", fb, "non-finite position");
    const double nn = norm(load3(q));
    if (std::abs(nn - 1.0) > 1e-6) add("point_normal_unit", fb, "normal length " + std::to_string(nn));
  }
  for (uint32_t i = 0; i < S.n_edges; ++i) {
    const double* g = &S.h_edges[12ull * i];
    const V3 st = load3(g), e = load3(g + 3), na = load3(g + 6), nb = load3(g + 9);
    const double len = norm(e - st);
    if (!(len > 0.0)) {
      add("edge_nondegenerate", i, "zero-length edge");
      continue;
    }
    const V3 w = (e - st) / len;
    if (std::abs(norm(na) - 1.0) > 1e-6) add("edge_normal_a_unit", i, "normal_a not unit");
    if (std::abs(norm(nb) - 1.0) > 1e-6) add("edge_normal_b_unit", i, "normal_b not unit");
    if (std::abs(dot(w, na)) > 1e-3) add("edge_normal_a_perpendicular", i, "w.n_a = " + std::to_string(dot(w, na)));
    if (std::abs(dot(w, nb)) > 1e-3) add("edge_normal_b_perpendicular", i, "w.n_b = " + std::to_string(dot(w, nb)));
    if (norm(na - nb) < 1e-9) add("edge_wedge_defined", i, "adjacent normals coincide");
    if (lh[i])
      add("edge_label_disjoint", i,
          "edge label " + std::to_string(S.h_edge_label[i]) + " collides with a surface label");
  }
  auto radios = [&](const std::vector<double>& pos, const std::vector<uint32_t>& id, const char* kind) {
    std::unordered_set<uint32_t> ids;
    for (size_t i = 0; i < id.size(); ++i) {
      const double* p = &pos[3 * i];
      if (!(std::isfinite(p[0]) && std::isfinite(p[1]) && std::isfinite(p[2])))
        add(std::string(kind) + "_position_finite", i, "non-finite position");
      if (!ids.insert(id[i]).second) add(std::string(kind) + "_id_unique", i, "duplicate id " + std::to_string(id[i]));
    }
  };
  radios(S.h_tx, S.h_tx_id, "tx");
  radios(S.h_rx, S.h_rx_id, "rx");
  if (S.h_tx_id.empty()) add("has_transmitter", 0, "no transmitters");
  if (S.h_rx_id.empty()) add("has_receiver", 0, "no receivers");
  if (!(S.carrier_frequency_hz > 0.0)) add("carrier_frequency_positive", 0, "frequency must be > 0");
  if (out.empty()) return false;
  v = out.front();
  return true;
}

// ---- exact paths, dedup, final order ----------------------------------------------------------
struct It {
  uint8_t kind;
  V3 pos, nrm;
  uint32_t label, ie, edge;
};
struct EP {
  uint32_t tx_id, rx_id;
  V3 tx, rx;
  std::vector<It> its;
  double total_length, delay, gnorm;
  bool converged;
};

// ---- combined candidate set on the device -----------------------------------------------------
struct CandSet {
  uint32_t n = 0, stride = 1;
  DBuf<uint32_t> tx_id, rx_id, n_inter, label, ie, edge;
  DBuf<uint8_t> kind;
  DBuf<double> tx_pos, rx_pos, length, pos, nrm;
};

__global__ void los_rows_kernel(const uint32_t* __restrict__ los_ie, uint32_t n, GridView g, V3 tx, uint32_t tx_id,
                                uint32_t row0, uint32_t* rx_id, double* rx_pos, double* length, uint32_t* n_inter,
                                uint32_t* txid, double* txpos) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint32_t i = los_ie[k];
  const V3 rp = ld3(g.ie_rp[i]);
  const uint32_t r = row0 + k;
  rx_id[r] = g.ie_rx[i];
  store3(rx_pos + 3ull * r, rp);
  length[r] = norm(rp - tx);
  n_inter[r] = 0;
  txid[r] = tx_id;
  store3(txpos + 3ull * r, tx);
}

__global__ void tx_rows_kernel(uint32_t n, uint32_t row0, V3 tx, uint32_t tx_id, uint32_t* txid, double* txpos) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  txid[row0 + k] = tx_id;
  store3(txpos + 3ull * (row0 + k), tx);
}

unsigned nb(uint64_t n, unsigned t = 256) { return static_cast<unsigned>((n + t - 1) / t ? (n + t - 1) / t : 1); }

void put_paths(pcr_paths* P, const std::vector<EP>& v) {
  for (size_t i = 0; i < v.size(); ++i) {
    const EP& e = v[i];
    P->tx_id[i] = e.tx_id;
    P->rx_id[i] = e.rx_id;
    store3(P->tx_position + 3 * i, e.tx);
    store3(P->rx_position + 3 * i, e.rx);
    P->length[i] = e.total_length;
    P->delay[i] = e.delay;
    P->converged[i] = e.converged ? 1 : 0;
    P->gradient_norm[i] = e.gnorm;
    P->n_inter[i] = static_cast<uint32_t>(e.its.size());
    for (size_t k = 0; k < e.its.size(); ++k) {
      const size_t j = i * P->stride + k;
      P->kind[j] = e.its[k].kind;
      store3(P->position + 3 * j, e.its[k].pos);
      P->label[j] = e.its[k].label;
      store3(P->normal + 3 * j, e.its[k].nrm);
      P->ie_index[j] = e.its[k].ie;
      P->edge_index[j] = e.its[k].edge;
    }
  }
}

}  // namespace

uint64_t config_hash(const pcr_run_config& c) {
  char buf[512];
  std::snprintf(buf, sizeof(buf), "%.17g|%.17g|%d|%d|%d|%d|%.17g|%d|%.17g|%d|%.17g|%d", c.carrier_frequency_hz,
                c.voxel_size_m, c.division_factor, c.kappa, c.max_interactions, c.max_diffractions,
                c.cone_apex_angle_deg, c.diffraction_ray_count, c.delta, c.rho, c.step_size,
                c.fresnel_enabled ? 1 : 0);
  return fnv1a(buf);
}

void run_config_defaults(pcr_run_config* c) {
  c->carrier_frequency_hz = 60e9;
  c->voxel_size_m = 0.5;
  c->division_factor = 2;
  c->kappa = 100;
  c->max_interactions = 5;
  c->max_diffractions = 1;
  c->cone_apex_angle_deg = 1.0;
  c->diffraction_ray_count = 360;
  c->delta = 1e-4;
  c->rho = 2000;
  c->step_size = 0.5;
  c->seed = 1;
  c->thread_count = 0;
  c->fresnel_enabled = 1;
}

void run_pipeline_core(Ctx& ctx, const SceneDev& scene, const pcr_run_config& cfg, pcr_summary** out,
                       double upload_seconds);

void upload_scene(Ctx& ctx, const pcr_scene_desc& d, SceneDev& S) {
  cudaStream_t s = ctx.stream;
  const size_t n = d.n_points;
  S.n_points = n;
  S.pos.alloc(3 * n + 3, s);
  S.nrm.alloc(3 * n + 3, s);
  S.label.alloc(n + 1, s);
  h2d(S.pos.get(), d.point_position, 3 * n, s);
  h2d(S.nrm.get(), d.point_normal, 3 * n, s);
  h2d(S.label.get(), d.point_label, n, s);
  S.n_edges = d.n_edges;
  S.h_edges.assign(d.edge_geometry, d.edge_geometry + 12ull * d.n_edges);
  S.h_edge_label.assign(d.edge_label, d.edge_label + d.n_edges);
  S.edges.alloc(12ull * d.n_edges + 12, s);
  S.edge_label.alloc(d.n_edges + 1ull, s);
  h2d(S.edges.get(), S.h_edges.data(), S.h_edges.size(), s);
  h2d(S.edge_label.get(), S.h_edge_label.data(), S.h_edge_label.size(), s);
  S.h_tx.assign(d.tx_position, d.tx_position + 3ull * d.n_tx);
  S.h_tx_id.assign(d.tx_id, d.tx_id + d.n_tx);
  S.h_rx.assign(d.rx_position, d.rx_position + 3ull * d.n_rx);
  S.h_rx_id.assign(d.rx_id, d.rx_id + d.n_rx);
  S.rx_pos.alloc(3ull * d.n_rx + 3, s);
  S.rx_id.alloc(d.n_rx + 1ull, s);
  h2d(S.rx_pos.get(), S.h_rx.data(), S.h_rx.size(), s);
  h2d(S.rx_id.get(), S.h_rx_id.data(), S.h_rx_id.size(), s);
  S.carrier_frequency_hz = d.carrier_frequency_hz;
  stream_wait(s);
}

void api_run_pipeline_on_scene(Ctx& ctx, const pcr_scene_desc& desc, const pcr_run_config& cfg, pcr_summary** out) {
  auto t0 = Clock::now();
  SceneDev scene;
  upload_scene(ctx, desc, scene);
  run_pipeline_core(ctx, scene, cfg, out, since(t0));
}

void api_run_pipeline_device(Ctx& ctx, const SceneDev& scene, const pcr_run_config& cfg, pcr_summary** out) {
  run_pipeline_core(ctx, scene, cfg, out, 0.0);
}

namespace {

// One pipeline run's summary under construction (stage timings in reference order).
struct Run {
  pcr_summary* S;
  explicit Run(pcr_summary* s) : S(s) {}
  explicit Run(const pcr_run_config& cfg, const SceneDev& scene) : S(halloc<pcr_summary>(1)) {
    S->hash = config_hash(cfg);
    S->point_count = scene.n_points;
    S->edge_count = scene.n_edges;
  }
  ~Run() { std::free(S); }
  pcr_summary* release() {
    pcr_summary* r = S;
    S = nullptr;
    return r;
  }
  void timing(const char* name, double sec) {
    if (S->n_timings < PCR_MAX_STAGES) {
      std::snprintf(S->timing_stage[S->n_timings], 16, "%s", name);
      S->timing_seconds[S->n_timings++] = sec;
    }
  }
};

// Rethrow a stage failure with the reference's "stage: " prefix (pipeline.cpp:30-32).
[[noreturn]] void stage_fail(const char* stage, const std::exception& e) {
  const Error* pe = dynamic_cast<const Error*>(&e);
  std::string msg = e.what();
  // device stages already prefix "trace: " style messages for their own errors
  if (msg.rfind(std::string(stage) + ": ", 0) != 0) msg = std::string(stage) + ": " + msg;
  throw Error(pe ? pe->code : PCR_ERR_RUNTIME, msg);
}

void stage_validate(Ctx& ctx, const SceneDev& scene) {
  Violation v;
  bool bad = false;
  try {
    bad = first_violation_device(ctx, scene, v);
  } catch (const std::exception& e) {
    stage_fail("validate", e);
  }
  if (bad) throw Error(PCR_ERR_RUNTIME, "validate: " + v.rule + " (" + v.detail + ")");
}

void stage_voxelize(Ctx& ctx, const SceneDev& scene, const pcr_run_config& cfg, GridDev& grid, pcr_summary* S) {
  try {
    KTimer kt(ctx, "build_grid");
    build_grid_device(ctx, scene, cfg.voxel_size_m, cfg.division_factor, uint64_t(1) << 27, grid);
  } catch (const std::exception& e) {
    stage_fail("voxelize", e);
  }
  S->ie_count = grid.n_ies;
  for (int a = 0; a < 3; ++a) S->grid_dims[a] = grid.dims[a];
}

pcr_trace_params trace_params_of(const pcr_run_config& cfg) {
  pcr_trace_params tp;
  tp.max_interactions = cfg.max_interactions;
  tp.kappa = cfg.kappa;
  tp.cone_apex_angle = cfg.cone_apex_angle_deg * 3.141592653589793238462643383279502884 / 180.0;
  tp.diffraction_ray_count = cfg.diffraction_ray_count;
  tp.max_diffractions = cfg.max_diffractions;
  return tp;
}

uint32_t stride_of(const pcr_run_config& cfg) { return static_cast<uint32_t>(std::max(1, cfg.max_interactions)); }

// transmission_phase for every TX (full IE range on every shard: it is O(n_IE) and
// its LOS list heads each TX's candidates).
void stage_transmission(Ctx& ctx, const GridDev& grid, const SceneDev& scene, std::vector<TxDev>& txs,
                        pcr_summary* S) {
  const uint32_t n_tx = static_cast<uint32_t>(scene.h_tx_id.size());
  txs.resize(n_tx);
  for (uint32_t t = 0; t < n_tx; ++t) {
    transmission_device(ctx, grid, scene, t, txs[t]);
    S->transmission_rays += grid.n_ies;
    S->visibility_tests += grid.n_ies;
  }
}

void release_hits(TxDev& t) {
  t.hit_ie.release();
  t.hit_kind.release();
  t.hit_pos.release();
  t.hit_nrm.release();
  t.hit_inc.release();
}

// One TX's propagated candidates: rows [off, off + n) of a CandDev.
struct PropSlice {
  const CandDev* c;
  uint32_t off, n;
};

// The candidate list of run_pipeline (pipeline.cpp:136-146): per TX, LOS in IE order,
// then the propagated candidates in output order.
void assemble_cands(Ctx& ctx, const SceneDev& scene, const GridDev& grid, const std::vector<TxDev>& txs,
                    const std::vector<PropSlice>& props, uint32_t stride, CandSet& cs) {
  cudaStream_t s = ctx.stream;
  const uint32_t n_tx = static_cast<uint32_t>(txs.size());
  uint64_t total = 0;
  for (uint32_t t = 0; t < n_tx; ++t) total += txs[t].n_los + props[t].n;
  if (total > 0xffffffffull) throw Error(PCR_ERR_NOMEM, "too many candidates");
  cs.stride = stride;
  cs.n = static_cast<uint32_t>(total);
  const size_t m = total ? total : 1, ms = m * stride;
  cs.tx_id.alloc(m, s);
  cs.rx_id.alloc(m, s);
  cs.n_inter.alloc(m, s);
  cs.label.alloc(ms, s);
  cs.ie.alloc(ms, s);
  cs.edge.alloc(ms, s);
  cs.kind.alloc(ms, s);
  cs.tx_pos.alloc(3 * m, s);
  cs.rx_pos.alloc(3 * m, s);
  cs.length.alloc(m, s);
  cs.pos.alloc(3 * ms, s);
  cs.nrm.alloc(3 * ms, s);
  PCR_CUDA(cudaMemsetAsync(cs.label.get(), 0, ms * sizeof(uint32_t), s));
  PCR_CUDA(cudaMemsetAsync(cs.ie.get(), 0, ms * sizeof(uint32_t), s));
  PCR_CUDA(cudaMemsetAsync(cs.edge.get(), 0, ms * sizeof(uint32_t), s));
  PCR_CUDA(cudaMemsetAsync(cs.kind.get(), 0, ms, s));
  PCR_CUDA(cudaMemsetAsync(cs.pos.get(), 0, 3 * ms * sizeof(double), s));
  PCR_CUDA(cudaMemsetAsync(cs.nrm.get(), 0, 3 * ms * sizeof(double), s));
  uint32_t row = 0;
  const GridView gv = grid.view();
  for (uint32_t t = 0; t < n_tx; ++t) {
    const V3 txp = load3(&scene.h_tx[3ull * t]);
    if (txs[t].n_los) {
      count_launch();
      los_rows_kernel<<<nb(txs[t].n_los), 256, 0, s>>>(txs[t].los_ie.get(), txs[t].n_los, gv, txp, scene.h_tx_id[t], row,
                                                        cs.rx_id.get(), cs.rx_pos.get(), cs.length.get(),
                                                        cs.n_inter.get(), cs.tx_id.get(), cs.tx_pos.get());
      PCR_LAUNCH_CHECK();
      row += txs[t].n_los;
    }
    const PropSlice& p = props[t];
    if (p.n) {
      const CandDev& c = *p.c;
      const size_t o = p.off, n = p.n;
      auto cp = [&](auto* dst, const auto* src, size_t count) {
        PCR_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(*src), cudaMemcpyDeviceToDevice, s));
      };
      cp(cs.rx_id.get() + row, c.rx_id.get() + o, n);
      cp(cs.n_inter.get() + row, c.n_inter.get() + o, n);
      cp(cs.rx_pos.get() + 3ull * row, c.rx_pos.get() + 3 * o, 3 * n);
      cp(cs.length.get() + row, c.length.get() + o, n);
      const size_t q = static_cast<size_t>(row) * stride, qo = o * c.stride, cnt = n * stride;
      if (c.stride != stride) throw Error(PCR_ERR_RUNTIME, "trace: candidate stride mismatch");
      cp(cs.label.get() + q, c.label.get() + qo, cnt);
      cp(cs.ie.get() + q, c.ie.get() + qo, cnt);
      cp(cs.edge.get() + q, c.edge.get() + qo, cnt);
      cp(cs.kind.get() + q, c.kind.get() + qo, cnt);
      cp(cs.pos.get() + 3 * q, c.pos.get() + 3 * qo, 3 * cnt);
      cp(cs.nrm.get() + 3 * q, c.nrm.get() + 3 * qo, 3 * cnt);
      count_launch();
      tx_rows_kernel<<<nb(p.n), 256, 0, s>>>(p.n, row, txp, scene.h_tx_id[t], cs.tx_id.get(), cs.tx_pos.get());
      PCR_LAUNCH_CHECK();
      row += p.n;
    }
  }
  stream_wait(s);
}

void refine_cands(Ctx& ctx, const GridDev& grid, const SceneDev& scene, const CandSet& cs, const pcr_run_config& cfg,
                  uint32_t first, uint32_t step, RefineDevOut& ro) {
  pcr_refine_params rp{cfg.delta, cfg.rho, cfg.step_size, cfg.fresnel_enabled};
  RefineDevIn in{cs.n,         cs.stride,       cs.tx_pos.get(), cs.rx_pos.get(), cs.pos.get(), cs.nrm.get(),
                 cs.length.get(), cs.n_inter.get(), cs.label.get(), cs.edge.get(), cs.kind.get()};
  in.first = first;
  in.step = step;
  refine_device(ctx, grid, scene, in, rp, ro);
}

// ---- dedup + final order on the device --------------------------------------
// dedup_by_label (refine.cpp:324-343), dedup_by_fresnel (:345-372) and the final order
// (pipeline.cpp:194-207) over the refinement outcomes in HBM; only the surviving paths
// come back to the host. Orders are stable LSD radix sorts on (delay, tx, rx) keys; the
// comparators' last fields (size, positions_lex_less) order the rare runs whose keys
// tie exactly. Only paths equal in every compared field can come out in another order
// than the reference's std::sort (whose order for them is unspecified).
struct ExactView {
  uint32_t stride;
  const uint32_t *src, *tx, *rx, *ni, *label;
  const uint8_t* kind;
  const double *pos, *txp, *len, *delay;
  __device__ uint32_t k(uint32_t e) const { return src[e]; }
};

__device__ __forceinline__ uint64_t mix64d(uint64_t h, uint64_t v) {
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  h *= 0xff51afd7ed558ccdull;
  h ^= h >> 33;
  return h;
}

// has_path -> exact-path list in candidate order; reject histogram; iteration sum
__global__ void exact_flags_kernel(const uint8_t* __restrict__ has, const int32_t* __restrict__ reason,
                                   const uint32_t* __restrict__ iters, uint32_t n, uint32_t* __restrict__ flag,
                                   unsigned long long* __restrict__ counts /* 4 rejects, iterations */) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long it = 0;
  if (i < n) {
    flag[i] = has[i] ? 1u : 0u;
    if (!has[i]) atomicAdd(counts + (reason[i] & 3), 1ull);
    it = iters[i];
  }
  for (int o = 16; o > 0; o >>= 1) it += __shfl_down_sync(0xffffffffu, it, o);
  if ((threadIdx.x & 31) == 0 && it) atomicAdd(counts + 4, it);
}

__global__ void compact_idx_kernel(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos, uint32_t n,
                                   const uint32_t* __restrict__ in, uint32_t* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && flag[i]) out[pos[i]] = in ? in[i] : i;
}

// group keys of the exact paths listed in `ord`: 0 = (tx, rx, kinds, labels),
// 1 = (tx, rx, kinds), 2 = delay bits, 3 = rx, 4 = tx
__global__ void exact_key_kernel(ExactView v, const uint32_t* __restrict__ ord, uint32_t m, int what,
                                 uint64_t* __restrict__ key) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const uint32_t k = v.k(ord[j]);
  uint64_t r;
  if (what <= 1) {
    r = mix64d(mix64d(mix64d(0x51ed270b27u, v.tx[k]), v.rx[k]), v.ni[k]);
    for (uint32_t q = 0; q < v.ni[k]; ++q) {
      const size_t x = static_cast<size_t>(k) * v.stride + q;
      r = mix64d(r, v.kind[x]);
      if (what == 0) r = mix64d(r, v.label[x]);
    }
  } else if (what == 2) {
    r = static_cast<uint64_t>(__double_as_longlong(v.delay[k]));  // delay >= 0: bits are ordered
  } else {
    r = what == 3 ? v.rx[k] : v.tx[k];
  }
  key[j] = r;
}

__device__ bool same_group(const ExactView& v, uint32_t ka, uint32_t kb, bool labels) {
  if (v.tx[ka] != v.tx[kb] || v.rx[ka] != v.rx[kb] || v.ni[ka] != v.ni[kb]) return false;
  for (uint32_t q = 0; q < v.ni[ka]; ++q) {
    const size_t a = static_cast<size_t>(ka) * v.stride + q, b = static_cast<size_t>(kb) * v.stride + q;
    if (v.kind[a] != v.kind[b]) return false;
    if (labels && v.label[a] != v.label[b]) return false;
  }
  return true;
}

// run heads of equal keys in `ord` order; a key run that mixes groups is a hash collision
__global__ void group_heads_kernel(ExactView v, const uint32_t* __restrict__ ord, const uint64_t* __restrict__ key,
                                   uint32_t m, bool labels, uint32_t* __restrict__ head, int* __restrict__ collision) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const bool h = j == 0 || key[j] != key[j - 1];
  head[j] = h ? 1u : 0u;
  if (!h && !same_group(v, v.k(ord[j]), v.k(ord[j - 1]), labels)) *collision = 1;
}

// positions_lex_less (refine.cpp:304-311)
__device__ bool dev_positions_lex_less(const ExactView& v, uint32_t ka, uint32_t kb) {
  const uint32_t na = v.ni[ka], nb = v.ni[kb];
  for (uint32_t q = 0; q < (na < nb ? na : nb); ++q) {
    const double* a = v.pos + 3 * (static_cast<size_t>(ka) * v.stride + q);
    const double* b = v.pos + 3 * (static_cast<size_t>(kb) * v.stride + q);
    if (a[0] != b[0] || a[1] != b[1] || a[2] != b[2]) {
      if (a[0] != b[0]) return a[0] < b[0];
      if (a[1] != b[1]) return a[1] < b[1];
      return a[2] < b[2];
    }
  }
  return na < nb;
}

// dedup_by_label's winner per group: runs are in candidate order, the candidate
// replaces the current best only when strictly better (length, then positions)
__global__ void label_winner_kernel(ExactView v, const uint32_t* __restrict__ ord, const uint32_t* __restrict__ head_pos,
                                    uint32_t n_groups, uint32_t m, uint32_t* __restrict__ winner) {
  const uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= n_groups) return;
  const uint32_t b = head_pos[gi], e = gi + 1 < n_groups ? head_pos[gi + 1] : m;
  uint32_t best = ord[b];
  for (uint32_t j = b + 1; j < e; ++j) {
    const uint32_t c = ord[j];
    const uint32_t kc = v.k(c), kb = v.k(best);
    if (v.len[kc] < v.len[kb] || (v.len[kc] == v.len[kb] && dev_positions_lex_less(v, kc, kb))) best = c;
  }
  winner[gi] = best;
}

// dedup_by_fresnel within one (tx, rx, kinds) bucket, members in delay order: a path
// is a duplicate when all its points lie inside the first-Fresnel ellipsoids of an
// earlier kept path's incoming legs (refine.cpp:356-366)
__global__ void fresnel_kernel(ExactView v, const uint32_t* __restrict__ ord, const uint32_t* __restrict__ head_pos,
                               uint32_t n_groups, uint32_t m, double half_lambda, uint8_t* __restrict__ kept) {
  const uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= n_groups) return;
  const uint32_t b = head_pos[gi], e = gi + 1 < n_groups ? head_pos[gi + 1] : m;
  for (uint32_t j = b; j < e; ++j) {
    const uint32_t kp = v.k(ord[j]);
    bool dup = false;
    for (uint32_t i = b; i < j && !dup; ++i) {
      if (!kept[i]) continue;
      const uint32_t kq = v.k(ord[i]);
      bool inside = true;
      for (uint32_t q = 0; q < v.ni[kp] && inside; ++q) {
        const V3 a = q == 0 ? load3(v.txp + 3ull * kq) : load3(v.pos + 3 * (static_cast<size_t>(kq) * v.stride + q - 1));
        const V3 bq = load3(v.pos + 3 * (static_cast<size_t>(kq) * v.stride + q));
        const V3 pt = load3(v.pos + 3 * (static_cast<size_t>(kp) * v.stride + q));
        inside = norm(pt - a) + norm(pt - bq) <= norm(bq - a) + half_lambda;
      }
      dup = inside;
    }
    kept[j] = dup ? 0 : 1;
  }
}

__global__ void gather_u32_kernel(const uint32_t* __restrict__ src, const uint32_t* __restrict__ perm, uint32_t n,
                                  uint32_t* __restrict__ dst) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[perm[i]];
}

__global__ void u8_to_u32_kernel(const uint8_t* __restrict__ a, uint32_t n, uint32_t* __restrict__ b) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

// Runs of exactly tied sort keys get the comparator's remaining fields by an
// insertion sort (runs are tiny): mode 0 = sort_by_delay's positions_lex_less over
// equal (delay, tx, rx); mode 1 = the final order's (size, positions) over equal
// (tx, rx, delay).
__device__ __forceinline__ bool same_delay_key(const ExactView& v, uint32_t a, uint32_t b) {
  const uint32_t ka = v.k(a), kb = v.k(b);
  return v.delay[ka] == v.delay[kb] && v.tx[ka] == v.tx[kb] && v.rx[ka] == v.rx[kb];
}

// run heads of exactly tied (delay, tx, rx) keys, computed before any run is reordered
__global__ void tie_heads_kernel(ExactView v, const uint32_t* __restrict__ ord, uint32_t m,
                                 uint8_t* __restrict__ head) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  head[j] = (j == 0 || !same_delay_key(v, ord[j - 1], ord[j])) ? 1 : 0;
}

__global__ void tie_sort_kernel(ExactView v, uint32_t* __restrict__ ord, const uint8_t* __restrict__ head, uint32_t m,
                                int mode) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m || !head[j]) return;
  uint32_t e = j + 1;
  while (e < m && !head[e]) ++e;
  if (e - j < 2) return;
  for (uint32_t x = j + 1; x < e; ++x) {
    const uint32_t c = ord[x];
    const uint32_t kc = v.k(c);
    uint32_t y = x;
    while (y > j) {
      const uint32_t kp = v.k(ord[y - 1]);
      const bool less = (mode == 1 && v.ni[kc] != v.ni[kp]) ? v.ni[kc] < v.ni[kp] : dev_positions_lex_less(v, kc, kp);
      if (!less) break;
      ord[y] = ord[y - 1];
      --y;
    }
    ord[y] = c;
  }
}

// Order runs of exactly tied (delay, tx, rx) keys by the comparator's remaining fields
// (mode 0: positions_lex_less of sort_by_delay; mode 1: size then positions, final order).
void sort_ties(Ctx& ctx, const ExactView& v, DBuf<uint32_t>& ord, uint32_t m, int mode) {
  if (m < 2) return;
  cudaStream_t s = ctx.stream;
  DBuf<uint8_t> head(m, s);
  count_launch();
  tie_heads_kernel<<<nb(m), 256, 0, s>>>(v, ord.get(), m, head.get());
  PCR_LAUNCH_CHECK();
  count_launch();
  tie_sort_kernel<<<nb(m), 256, 0, s>>>(v, ord.get(), head.get(), m, mode);
  PCR_LAUNCH_CHECK();
}

__global__ void scatter_flag_kernel(const uint32_t* __restrict__ ord, const uint32_t* __restrict__ f, uint32_t n,
                                    uint32_t* __restrict__ by_id) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) by_id[ord[i]] = f[i];
}

__global__ void gather_exact_kernel(const uint32_t* __restrict__ rows, uint32_t m, uint32_t st,
                                    const uint32_t* tx, const uint32_t* rx, const uint32_t* ni, const double* txp,
                                    const double* rxp, const double* len, const double* del, const double* gn,
                                    const uint8_t* kind, const double* pos, const double* nrm, const uint32_t* lab,
                                    const uint32_t* ie, const uint32_t* ed, uint32_t* o_tx, uint32_t* o_rx,
                                    uint32_t* o_ni, double* o_txp, double* o_rxp, double* o_len, double* o_del,
                                    double* o_gn, uint8_t* o_kind, double* o_pos, double* o_nrm, uint32_t* o_lab,
                                    uint32_t* o_ie, uint32_t* o_ed) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint32_t k = rows[i];
  o_tx[i] = tx[k];
  o_rx[i] = rx[k];
  o_ni[i] = ni[k];
  for (int a = 0; a < 3; ++a) {
    o_txp[3ull * i + a] = txp[3ull * k + a];
    o_rxp[3ull * i + a] = rxp[3ull * k + a];
  }
  o_len[i] = len[k];
  o_del[i] = del[k];
  o_gn[i] = gn[k];
  for (uint32_t q = 0; q < st; ++q) {
    const size_t d = static_cast<size_t>(i) * st + q, sidx = static_cast<size_t>(k) * st + q;
    o_kind[d] = kind[sidx];
    o_lab[d] = lab[sidx];
    o_ie[d] = ie[sidx];
    o_ed[d] = ed[sidx];
    for (int a = 0; a < 3; ++a) {
      o_pos[3 * d + a] = pos[3 * sidx + a];
      o_nrm[3 * d + a] = nrm[3 * sidx + a];
    }
  }
}

// Stable sort of `ord` (m exact-path ids) by key `what` (see exact_key_kernel).
void sort_by(Ctx& ctx, const ExactView& v, DBuf<uint32_t>& ord, uint32_t m, int what, int bits) {
  if (m < 2) return;
  cudaStream_t s = ctx.stream;
  DBuf<uint64_t> key(m, s);
  count_launch();
  exact_key_kernel<<<nb(m), 256, 0, s>>>(v, ord.get(), m, what, key.get());
  PCR_LAUNCH_CHECK();
  radix_sort_pairs(key.get(), ord.get(), m, 0, bits, s);
}

// Group `ord` (already in the wanted in-group order) by key `what`, stable: returns
// the group head positions.
std::vector<uint32_t> group_by(Ctx& ctx, const ExactView& v, DBuf<uint32_t>& ord, uint32_t m, int what,
                               DBuf<uint32_t>& heads) {
  cudaStream_t s = ctx.stream;
  DBuf<uint64_t> key(m ? m : 1, s);
  if (m) {
    count_launch();
    exact_key_kernel<<<nb(m), 256, 0, s>>>(v, ord.get(), m, what, key.get());
    PCR_LAUNCH_CHECK();
    radix_sort_pairs(key.get(), ord.get(), m, 0, 64, s);
  }
  DBuf<uint32_t> head(m ? m : 1, s), pos(m ? m : 1, s), tot(1, s);
  DBuf<int> coll(1, s);
  PCR_CUDA(cudaMemsetAsync(coll.get(), 0, sizeof(int), s));
  PCR_CUDA(cudaMemsetAsync(tot.get(), 0, sizeof(uint32_t), s));
  if (m) {
    count_launch();
    group_heads_kernel<<<nb(m), 256, 0, s>>>(v, ord.get(), key.get(), m, what == 0, head.get(), coll.get());
    PCR_LAUNCH_CHECK();
    exclusive_scan_u32(head.get(), pos.get(), m, tot.get(), s);
  }
  uint32_t ng = 0;
  int c = 0;
  d2h(&ng, tot.get(), 1, s);
  d2h(&c, coll.get(), 1, s);
  stream_wait(s);
  if (c) throw Error(4, "dedup: group hash collision");
  heads.alloc(ng ? ng : 1, s);
  if (m) {
    count_launch();
    compact_idx_kernel<<<nb(m), 256, 0, s>>>(head.get(), pos.get(), m, nullptr, heads.get());
    PCR_LAUNCH_CHECK();
  }
  return {ng};
}

// Refinement outcomes -> deduplicated exact paths in the final order (host EPs), with
// the refine counters (refined_paths, rejected, refine_iterations).
std::vector<EP> dedup_device(Ctx& ctx, const CandSet& cs, const RefineDevOut& ro, const pcr_run_config& cfg,
                             pcr_summary* S) {
  cudaStream_t s = ctx.stream;
  const uint32_t n = cs.n;
  // exact paths (has_path) in candidate order
  DBuf<uint32_t> flag(n ? n : 1, s), fpos(n ? n : 1, s), tot(1, s);
  DBuf<unsigned long long> counts(5, s);
  PCR_CUDA(cudaMemsetAsync(counts.get(), 0, 5 * sizeof(unsigned long long), s));
  PCR_CUDA(cudaMemsetAsync(tot.get(), 0, sizeof(uint32_t), s));
  if (n) {
    count_launch();
    exact_flags_kernel<<<nb(n), 256, 0, s>>>(ro.has_path.get(), ro.reason.get(), ro.iters.get(), n, flag.get(),
                                              counts.get());
    PCR_LAUNCH_CHECK();
    exclusive_scan_u32(flag.get(), fpos.get(), n, tot.get(), s);
  }
  uint32_t m = 0;
  unsigned long long hc[5];
  d2h(&m, tot.get(), 1, s);
  d2h(hc, counts.get(), 5, s);
  stream_wait(s);
  for (int r = 0; r < 4; ++r) S->rejected[r] = hc[r];
  S->refine_iterations = hc[4];
  S->refined_paths = m;
  DBuf<uint32_t> src(m ? m : 1, s);
  if (n) {
    count_launch();
    compact_idx_kernel<<<nb(n), 256, 0, s>>>(flag.get(), fpos.get(), n, nullptr, src.get());
    PCR_LAUNCH_CHECK();
  }
  const ExactView v{cs.stride,      src.get(),     cs.tx_id.get(), cs.rx_id.get(), cs.n_inter.get(),
                    ro.label.get(), cs.kind.get(), ro.pos.get(),   cs.tx_pos.get(), ro.length.get(),
                    ro.delay.get()};
  // dedup_by_label: groups in candidate order, strict-improvement winner per group
  DBuf<uint32_t> ord(m ? m : 1, s), heads;
  iota_u32(ord.get(), m, s);
  uint32_t ng = group_by(ctx, v, ord, m, 0, heads)[0];
  DBuf<uint32_t> kept(ng ? ng : 1, s);
  if (ng) {
    count_launch();
    label_winner_kernel<<<nb(ng), 256, 0, s>>>(v, ord.get(), heads.get(), ng, m, kept.get());
    PCR_LAUNCH_CHECK();
  }
  // sort_by_delay: (delay, tx, rx) by stable LSD passes, positions on the host below
  sort_by(ctx, v, kept, ng, 3, 32);
  sort_by(ctx, v, kept, ng, 4, 32);
  sort_by(ctx, v, kept, ng, 2, 64);
  sort_ties(ctx, v, kept, ng, 0);
  uint32_t mf = ng;
  DBuf<uint32_t> fin;
  if (cfg.fresnel_enabled && ng) {
    // dedup_by_fresnel: buckets (tx, rx, kinds), members in delay order
    DBuf<uint32_t> b_ord(ng, s), b_heads;
    PCR_CUDA(cudaMemcpyAsync(b_ord.get(), kept.get(), ng * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    const uint32_t nb_ = group_by(ctx, v, b_ord, ng, 1, b_heads)[0];
    DBuf<uint8_t> keep8(ng, s);
    count_launch();
    fresnel_kernel<<<nb(nb_, 128), 128, 0, s>>>(v, b_ord.get(), b_heads.get(), nb_, ng,
                                                 0.5 * (kC / cfg.carrier_frequency_hz), keep8.get());
    PCR_LAUNCH_CHECK();
    // survivors back in delay order: flag by path id, then compact the delay order
    DBuf<uint32_t> k32(ng, s), by_id(m ? m : 1, s), f2(ng, s), p2(ng, s), t2(1, s);
    PCR_CUDA(cudaMemsetAsync(by_id.get(), 0, (m ? m : 1) * sizeof(uint32_t), s));
    count_launch();
    u8_to_u32_kernel<<<nb(ng), 256, 0, s>>>(keep8.get(), ng, k32.get());
    PCR_LAUNCH_CHECK();
    count_launch();
    scatter_flag_kernel<<<nb(ng), 256, 0, s>>>(b_ord.get(), k32.get(), ng, by_id.get());
    PCR_LAUNCH_CHECK();
    count_launch();
    gather_u32_kernel<<<nb(ng), 256, 0, s>>>(by_id.get(), kept.get(), ng, f2.get());
    PCR_LAUNCH_CHECK();
    exclusive_scan_u32(f2.get(), p2.get(), ng, t2.get(), s);
    d2h(&mf, t2.get(), 1, s);
    stream_wait(s);
    fin.alloc(mf ? mf : 1, s);
    count_launch();
    compact_idx_kernel<<<nb(ng), 256, 0, s>>>(f2.get(), p2.get(), ng, kept.get(), fin.get());
    PCR_LAUNCH_CHECK();
  } else {
    fin.swap(kept);
  }
  // final order (pipeline.cpp:194-207): (tx, rx, delay) by stable passes over the
  // delay-ordered survivors; (size, positions) on the host for exact key ties
  sort_by(ctx, v, fin, mf, 3, 32);
  sort_by(ctx, v, fin, mf, 4, 32);
  sort_ties(ctx, v, fin, mf, 1);
  // download only the survivors
  std::vector<uint32_t> ids(mf);
  d2h(ids.data(), fin.get(), mf, s);
  std::vector<uint32_t> hsrc(m);
  d2h(hsrc.data(), src.get(), m, s);
  stream_wait(s);
  const uint32_t stv = cs.stride;
  std::vector<EP> out(mf);
  {
    // gather the survivors' rows on the device, then one copy per field
    DBuf<uint32_t> rows(mf ? mf : 1, s);
    std::vector<uint32_t> hrows(mf);
    for (uint32_t i = 0; i < mf; ++i) hrows[i] = hsrc[ids[i]];
    h2d(rows.get(), hrows.data(), mf, s);
    DBuf<uint32_t> g_tx(mf + 1, s), g_rx(mf + 1, s), g_ni(mf + 1, s), g_lab(mf * stv + 1, s), g_ie(mf * stv + 1, s),
        g_ed(mf * stv + 1, s);
    DBuf<uint8_t> g_kind(mf * stv + 1, s);
    DBuf<double> g_txp(3 * mf + 3, s), g_rxp(3 * mf + 3, s), g_len(mf + 1, s), g_del(mf + 1, s), g_gn(mf + 1, s),
        g_pos(3 * mf * stv + 3, s), g_nrm(3 * mf * stv + 3, s);
    if (mf) {
      count_launch();
      gather_exact_kernel<<<nb(mf), 256, 0, s>>>(
          rows.get(), mf, stv, cs.tx_id.get(), cs.rx_id.get(), cs.n_inter.get(), cs.tx_pos.get(), cs.rx_pos.get(),
          ro.length.get(), ro.delay.get(), ro.gnorm.get(), cs.kind.get(), ro.pos.get(), ro.nrm.get(), ro.label.get(),
          cs.ie.get(), cs.edge.get(), g_tx.get(), g_rx.get(), g_ni.get(), g_txp.get(), g_rxp.get(), g_len.get(),
          g_del.get(), g_gn.get(), g_kind.get(), g_pos.get(), g_nrm.get(), g_lab.get(), g_ie.get(), g_ed.get());
      PCR_LAUNCH_CHECK();
    }
    std::vector<uint32_t> tx(mf), rx(mf), ni(mf), lab(mf * stv), ie(mf * stv), ed(mf * stv);
    std::vector<uint8_t> kind(mf * stv);
    std::vector<double> txp(3 * mf), rxp(3 * mf), len(mf), del(mf), gn(mf), pos(3 * mf * stv), nrm(3 * mf * stv);
    d2h(tx.data(), g_tx.get(), mf, s);
    d2h(rx.data(), g_rx.get(), mf, s);
    d2h(ni.data(), g_ni.get(), mf, s);
    d2h(txp.data(), g_txp.get(), 3 * mf, s);
    d2h(rxp.data(), g_rxp.get(), 3 * mf, s);
    d2h(len.data(), g_len.get(), mf, s);
    d2h(del.data(), g_del.get(), mf, s);
    d2h(gn.data(), g_gn.get(), mf, s);
    d2h(kind.data(), g_kind.get(), mf * stv, s);
    d2h(pos.data(), g_pos.get(), 3 * mf * stv, s);
    d2h(nrm.data(), g_nrm.get(), 3 * mf * stv, s);
    d2h(lab.data(), g_lab.get(), mf * stv, s);
    d2h(ie.data(), g_ie.get(), mf * stv, s);
    d2h(ed.data(), g_ed.get(), mf * stv, s);
    stream_wait(s);
    for (uint32_t i = 0; i < mf; ++i) {
      EP& e = out[i];
      e.tx_id = tx[i];
      e.rx_id = rx[i];
      e.tx = load3(&txp[3 * i]);
      e.rx = load3(&rxp[3 * i]);
      e.total_length = len[i];
      e.delay = del[i];
      e.gnorm = gn[i];
      e.converged = true;
      for (uint32_t q = 0; q < ni[i]; ++q) {
        const size_t j = static_cast<size_t>(i) * stv + q;
        e.its.push_back(It{kind[j], load3(&pos[3 * j]), load3(&nrm[3 * j]), lab[j], ie[j], ed[j]});
      }
    }
  }
  return out;
}

// the final paths -> S->paths
void emit_paths(const std::vector<EP>& exact, pcr_summary* S) {
  S->exact_paths = exact.size();
  size_t st = 1;
  for (const EP& e : exact) st = std::max(st, e.its.size());
  pcr_paths* P = alloc_paths(exact.size(), static_cast<uint32_t>(st));
  put_paths(P, exact);
  S->paths = *P;
  std::free(P);
}

}  // namespace

void run_pipeline_core(Ctx& ctx, const SceneDev& scene, const pcr_run_config& cfg, pcr_summary** out,
                       double upload_seconds) {
  Run run(cfg, scene);
  pcr_summary* S = run.S;
  const uint32_t n_tx = static_cast<uint32_t>(scene.h_tx_id.size());

  auto t0 = Clock::now();
  stage_validate(ctx, scene);
  run.timing("validate", since(t0) + upload_seconds);

  t0 = Clock::now();
  GridDev grid;
  stage_voxelize(ctx, scene, cfg, grid, S);
  run.timing("voxelize", since(t0));

  // trace
  t0 = Clock::now();
  const pcr_trace_params tp = trace_params_of(cfg);
  CandSet cs;
  try {
    std::vector<TxDev> txs;
    std::vector<CandDev> props(n_tx);
    std::vector<PropSlice> slices(n_tx);
    stage_transmission(ctx, grid, scene, txs, S);
    TraceStats st;
    for (uint32_t t = 0; t < n_tx; ++t) {
      propagate_device(ctx, grid, scene, t, txs[t].hit_ie.get(), txs[t].hit_kind.get(), txs[t].hit_pos.get(),
                       txs[t].hit_nrm.get(), txs[t].hit_inc.get(), txs[t].n_hits, tp, props[t], st);
      release_hits(txs[t]);
      slices[t] = PropSlice{&props[t], 0, props[t].n};
    }
    S->cone_traces = st.cone_traces;
    S->walk_cells = st.walk_cells;
    S->walk_ies = st.walk_ies;
    S->libm_unresolved = st.libm_unresolved;
    S->visibility_tests += st.visibility_tests;
    assemble_cands(ctx, scene, grid, txs, slices, stride_of(cfg), cs);
  } catch (const std::exception& e) {
    stage_fail("trace", e);
  }
  S->coarse_paths = cs.n;
  run.timing("trace", since(t0));

  // refine
  t0 = Clock::now();
  RefineDevOut ro;
  try {
    refine_cands(ctx, grid, scene, cs, cfg, 0, 1, ro);
    S->refine_trials = ro.trials;
    S->refine_marches = ro.marches;
    S->refine_trial_nodes = ro.trial_nodes;
    S->refine_iter_nodes = ro.iter_nodes;
  } catch (const std::exception& e) {
    stage_fail("refine", e);
  }
  run.timing("refine", since(t0));

  // dedup_by_label, dedup_by_fresnel and the final order, on the device
  t0 = Clock::now();
  try {
    emit_paths(dedup_device(ctx, cs, ro, cfg, S), S);
  } catch (const std::exception& e) {
    stage_fail("refine", e);
  }
  run.timing("dedup", since(t0));
  *out = run.release();
}

// ---- sharded pipeline ---------------------------------------------------------
// A shard traces the initial hits t ≡ shard (mod n_shards) of every TX and keeps its
// own first-kappa (exact pre-cap); the rows of every shard are merged by DFS key into
// the global candidate list (identical on every shard); a shard refines candidates
// i ≡ shard (mod n_shards); one shard collects every outcome row and finishes.
struct ShardState {
  pcr_run_config cfg{};
  uint32_t shard = 0, n_shards = 1;
  GridDev grid;
  const GridDev* ext = nullptr;  // a grid the caller built / assembled (pcr_shard_trace_grid)
  const GridDev& g() const { return ext ? *ext : grid; }
  std::vector<TxDev> txs;
  pcr_summary head{};  // counts and timings of this shard so far
  double trace_s = 0, refine_s = 0;
  pcr_shard_stats stats{};
  DBuf<uint8_t> rows;
  uint64_t n_rows = 0;
  CandSet cs;
  bool merged = false;
  DBuf<uint8_t> out_rows;
  uint64_t n_out = 0;
};

namespace {

ShardState& shard_state(Ctx& ctx) {
  if (!ctx.shard) throw Error(PCR_ERR_INVALID, "shard: pcr_shard_trace has not run on this context");
  return *ctx.shard;
}

void head_timing(pcr_summary& S, const char* name, double sec) {
  if (S.n_timings < PCR_MAX_STAGES) {
    std::snprintf(S.timing_stage[S.n_timings], 16, "%s", name);
    S.timing_seconds[S.n_timings++] = sec;
  }
}

__global__ void pack_outcomes_kernel(uint32_t n_sub, uint32_t first, uint32_t step, uint32_t stride,
                                     const int32_t* __restrict__ reason, const uint8_t* __restrict__ has,
                                     const uint32_t* __restrict__ iters, const double* __restrict__ length,
                                     const double* __restrict__ delay, const double* __restrict__ gnorm,
                                     const double* __restrict__ pos, const double* __restrict__ nrm,
                                     const uint32_t* __restrict__ label, uint8_t* __restrict__ rows) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_sub) return;
  const uint32_t k = first + i * step;
  uint8_t* r = rows + static_cast<size_t>(i) * out_row_bytes(stride);
  OutRowHead h{k, reason[k], iters[k], has[k], length[k], delay[k], gnorm[k]};
  *reinterpret_cast<OutRowHead*>(r) = h;
  OutRowLevel* lv = reinterpret_cast<OutRowLevel*>(r + sizeof(OutRowHead));
  for (uint32_t q = 0; q < stride; ++q) {
    const size_t j = static_cast<size_t>(k) * stride + q;
    OutRowLevel l;
    for (int a = 0; a < 3; ++a) {
      l.pos[a] = pos[3 * j + a];
      l.nrm[a] = nrm[3 * j + a];
    }
    l.label = label[j];
    l.pad = 0;
    lv[q] = l;
  }
}

__global__ void unpack_outcomes_kernel(const uint8_t* __restrict__ rows, uint64_t n_rows, uint32_t n, uint32_t stride,
                                       int32_t* reason, uint8_t* has, uint32_t* iters, double* length, double* delay,
                                       double* gnorm, double* pos, double* nrm, uint32_t* label, uint32_t* seen,
                                       int* bad) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_rows) return;
  const uint8_t* r = rows + i * out_row_bytes(stride);
  const OutRowHead& h = *reinterpret_cast<const OutRowHead*>(r);
  const uint32_t k = h.cand;
  if (k >= n || atomicAdd(seen + k, 1u) != 0) {
    *bad = 1;
    return;
  }
  reason[k] = h.reason;
  has[k] = static_cast<uint8_t>(h.has_path);
  iters[k] = h.iters;
  length[k] = h.length;
  delay[k] = h.delay;
  gnorm[k] = h.gnorm;
  const OutRowLevel* lv = reinterpret_cast<const OutRowLevel*>(r + sizeof(OutRowHead));
  for (uint32_t q = 0; q < stride; ++q) {
    const size_t j = static_cast<size_t>(k) * stride + q;
    for (int a = 0; a < 3; ++a) {
      pos[3 * j + a] = lv[q].pos[a];
      nrm[3 * j + a] = lv[q].nrm[a];
    }
    label[j] = lv[q].label;
  }
}

}  // namespace

void api_shard_trace(Ctx& ctx, const SceneDev& scene, const pcr_run_config& cfg, uint32_t shard, uint32_t n_shards,
                     uint64_t* n_rows, uint64_t* row_bytes, const GridDev* grid) {
  if (n_shards == 0 || shard >= n_shards) throw Error(PCR_ERR_INVALID, "shard: index out of range");
  ctx.shard = std::make_shared<ShardState>();
  ShardState& st = *ctx.shard;
  st.cfg = cfg;
  st.shard = shard;
  st.n_shards = n_shards;
  pcr_summary& S = st.head;
  S.hash = config_hash(cfg);
  S.point_count = scene.n_points;
  S.edge_count = scene.n_edges;
  const uint32_t n_tx = static_cast<uint32_t>(scene.h_tx_id.size());
  const uint32_t stride = stride_of(cfg);

  auto t0 = Clock::now();
  stage_validate(ctx, scene);
  head_timing(S, "validate", since(t0));
  t0 = Clock::now();
  if (grid) {  // replicated by the caller (NCCL broadcast or sharded build + all-gather)
    if (grid->voxel_size != cfg.voxel_size_m || grid->dv != cfg.division_factor)
      throw Error(PCR_ERR_INVALID, "shard: grid built with other voxel parameters");
    st.ext = grid;
    S.ie_count = grid->n_ies;
    for (int a = 0; a < 3; ++a) S.grid_dims[a] = grid->dims[a];
  } else {
    stage_voxelize(ctx, scene, cfg, st.grid, &S);
  }
  head_timing(S, "voxelize", since(t0));

  t0 = Clock::now();
  try {
    cudaStream_t s = ctx.stream;
    const pcr_trace_params tp = trace_params_of(cfg);
    stage_transmission(ctx, st.g(), scene, st.txs, &S);
    std::vector<CandDev> props(n_tx);
    TraceStats ts;
    uint64_t total = 0;
    for (uint32_t t = 0; t < n_tx; ++t) {
      TxDev& x = st.txs[t];
      propagate_device(ctx, st.g(), scene, t, x.hit_ie.get(), x.hit_kind.get(), x.hit_pos.get(), x.hit_nrm.get(),
                       x.hit_inc.get(), x.n_hits, tp, props[t], ts, shard, n_shards, true);
      release_hits(x);
      total += props[t].n;
    }
    st.stats.cone_traces = ts.cone_traces;
    st.stats.visibility_tests = ts.visibility_tests;
    st.stats.walk_cells = ts.walk_cells;
    st.stats.walk_ies = ts.walk_ies;
    st.stats.libm_unresolved = ts.libm_unresolved;
    const size_t bytes = cand_row_bytes(stride);
    st.rows.alloc(total ? total * bytes : 1, s);
    uint64_t row = 0;
    for (uint32_t t = 0; t < n_tx; ++t) {
      pack_cand_rows(ctx, props[t], t, st.rows.get() + row * bytes);
      row += props[t].n;
    }
    st.n_rows = total;
    stream_wait(s);
  } catch (const std::exception& e) {
    stage_fail("trace", e);
  }
  st.trace_s = since(t0);
  *n_rows = st.n_rows;
  *row_bytes = cand_row_bytes(stride);
}

void api_shard_rows(Ctx& ctx, void* dst) {
  ShardState& st = shard_state(ctx);
  if (st.n_rows)
    PCR_CUDA(cudaMemcpyAsync(dst, st.rows.get(), st.n_rows * cand_row_bytes(stride_of(st.cfg)),
                             cudaMemcpyDeviceToDevice, ctx.stream));
  PCR_CUDA(cudaStreamSynchronize(ctx.stream));
}

void api_shard_refine(Ctx& ctx, const SceneDev& scene, const void* rows, uint64_t n_rows, uint64_t* n_out,
                      uint64_t* out_bytes) {
  ShardState& st = shard_state(ctx);
  cudaStream_t s = ctx.stream;
  const uint32_t stride = stride_of(st.cfg);
  const uint32_t n_tx = static_cast<uint32_t>(scene.h_tx_id.size());
  auto t0 = Clock::now();
  try {
    CandDev merged;
    std::vector<uint32_t> per_tx;
    kappa_merge_rows(ctx, static_cast<const uint8_t*>(rows), n_rows, stride, st.cfg.kappa, n_tx, merged, per_tx);
    std::vector<PropSlice> slices(n_tx);
    uint32_t off = 0;
    for (uint32_t t = 0; t < n_tx; ++t) {
      slices[t] = PropSlice{&merged, off, per_tx[t]};
      off += per_tx[t];
    }
    assemble_cands(ctx, scene, st.g(), st.txs, slices, stride, st.cs);
    st.merged = true;
  } catch (const std::exception& e) {
    stage_fail("trace", e);
  }
  st.trace_s += since(t0);
  st.head.coarse_paths = st.cs.n;

  t0 = Clock::now();
  try {
    RefineDevOut ro;
    refine_cands(ctx, st.g(), scene, st.cs, st.cfg, st.shard, st.n_shards, ro);
    st.stats.refine_trials = ro.trials;
    st.stats.refine_marches = ro.marches;
    st.stats.refine_trial_nodes = ro.trial_nodes;
    st.stats.refine_iter_nodes = ro.iter_nodes;
    const uint32_t n = st.cs.n;
    const uint32_t n_sub = n > st.shard ? (n - st.shard + st.n_shards - 1) / st.n_shards : 0;
    const size_t bytes = out_row_bytes(stride);
    st.out_rows.alloc(n_sub ? n_sub * bytes : 1, s);
    st.n_out = n_sub;
    if (n_sub) {
      count_launch();
      pack_outcomes_kernel<<<nb(n_sub), 256, 0, s>>>(n_sub, st.shard, st.n_shards, stride, ro.reason.get(),
                                                      ro.has_path.get(), ro.iters.get(), ro.length.get(),
                                                      ro.delay.get(), ro.gnorm.get(), ro.pos.get(), ro.nrm.get(),
                                                      ro.label.get(), st.out_rows.get());
      PCR_LAUNCH_CHECK();
      // iterations of this shard's candidates (a work counter, summed over shards)
      std::vector<uint32_t> all(n);
      d2h(all.data(), ro.iters.get(), n, s);
      stream_wait(s);
      uint64_t sum = 0;
      for (uint32_t i = 0; i < n_sub; ++i) sum += all[st.shard + static_cast<size_t>(i) * st.n_shards];
      st.stats.refine_iterations = sum;
    }
    stream_wait(s);
  } catch (const std::exception& e) {
    stage_fail("refine", e);
  }
  st.refine_s = since(t0);
  *n_out = st.n_out;
  *out_bytes = out_row_bytes(stride);
}

void api_shard_outcomes(Ctx& ctx, void* dst) {
  ShardState& st = shard_state(ctx);
  if (st.n_out)
    PCR_CUDA(cudaMemcpyAsync(dst, st.out_rows.get(), st.n_out * out_row_bytes(stride_of(st.cfg)),
                             cudaMemcpyDeviceToDevice, ctx.stream));
  PCR_CUDA(cudaStreamSynchronize(ctx.stream));
}

void api_shard_stats(Ctx& ctx, pcr_shard_stats* out) { *out = shard_state(ctx).stats; }

void api_shard_finish(Ctx& ctx, const void* rows, uint64_t n_rows, const pcr_shard_stats& totals,
                      pcr_summary** out) {
  ShardState& st = shard_state(ctx);
  if (!st.merged) throw Error(PCR_ERR_INVALID, "shard: pcr_shard_refine has not run on this context");
  cudaStream_t s = ctx.stream;
  const CandSet& cs = st.cs;
  const uint32_t stride = cs.stride;
  auto t0 = Clock::now();
  Run run(halloc<pcr_summary>(1));
  pcr_summary* S = run.S;
  *S = st.head;  // hash, sizes, transmission counts, validate + voxelize timings
  S->cone_traces = totals.cone_traces;
  S->walk_cells = totals.walk_cells;
  S->walk_ies = totals.walk_ies;
  S->libm_unresolved = totals.libm_unresolved;
  S->refine_trial_nodes = totals.refine_trial_nodes;
  S->refine_iter_nodes = totals.refine_iter_nodes;
  S->visibility_tests += totals.visibility_tests;
  S->refine_trials = totals.refine_trials;
  S->refine_marches = totals.refine_marches;
  run.timing("trace", st.trace_s);
  RefineDevOut ro;
  try {
    if (n_rows != cs.n) throw Error(PCR_ERR_INVALID, "shard: outcome rows do not cover the candidate list");
    const size_t m = cs.n ? cs.n : 1, ms = m * stride;
    ro.reason.alloc(m, s);
    ro.has_path.alloc(m, s);
    ro.iters.alloc(m, s);
    ro.length.alloc(m, s);
    ro.delay.alloc(m, s);
    ro.gnorm.alloc(m, s);
    ro.pos.alloc(3 * ms, s);
    ro.nrm.alloc(3 * ms, s);
    ro.label.alloc(ms, s);
    DBuf<uint32_t> seen(m, s);
    DBuf<int> bad(1, s);
    PCR_CUDA(cudaMemsetAsync(seen.get(), 0, m * sizeof(uint32_t), s));
    PCR_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
    if (n_rows) {
      count_launch();
      unpack_outcomes_kernel<<<nb(n_rows), 256, 0, s>>>(static_cast<const uint8_t*>(rows), n_rows, cs.n, stride,
                                                         ro.reason.get(), ro.has_path.get(), ro.iters.get(),
                                                         ro.length.get(), ro.delay.get(), ro.gnorm.get(),
                                                         ro.pos.get(), ro.nrm.get(), ro.label.get(), seen.get(),
                                                         bad.get());
      PCR_LAUNCH_CHECK();
    }
    int h_bad = 0;
    d2h(&h_bad, bad.get(), 1, s);
    stream_wait(s);
    if (h_bad) throw Error(PCR_ERR_INVALID, "shard: outcome rows do not cover the candidate list");
  } catch (const std::exception& e) {
    stage_fail("refine", e);
  }
  run.timing("refine", st.refine_s + since(t0));
  t0 = Clock::now();
  try {
    emit_paths(dedup_device(ctx, cs, ro, st.cfg, S), S);
  } catch (const std::exception& e) {
    stage_fail("refine", e);
  }
  run.timing("dedup", since(t0));
  *out = run.release();
}

}  // namespace pcr
