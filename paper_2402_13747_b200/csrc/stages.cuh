// stages.cuh — device-resident stage results passed between trace.cu, refine.cu
// and pipeline.cu.
#pragma once

#include <vector>

#include "../../include/pcray_b200.h"
#include "device_state.cuh"

namespace pcr {

// transmission_phase result for one TX (tracer.hpp:66-69), IE order kept.
struct TxDev {
  uint32_t n_los = 0, n_hits = 0;
  DBuf<uint32_t> los_ie;  // IE index of each LOS candidate
  DBuf<uint32_t> hit_ie;  // initial hits
  DBuf<uint8_t> hit_kind;
  DBuf<double> hit_pos, hit_nrm, hit_inc;
};

// Work counters of a propagate call (SURVEY §8d units).
struct TraceStats {
  uint64_t cone_traces = 0, visibility_tests = 0, walk_cells = 0, walk_ies = 0;
  uint64_t libm_unresolved = 0;  // knife-edge atan2/asin decisions not certified (trace.cuh libm_le)
};

// Kept propagation candidates of one TX in output (DFS) order; interaction
// arrays are row-major [n][stride].
struct CandDev {
  uint32_t n = 0;
  uint32_t stride = 1;
  DBuf<uint32_t> rx_id, n_inter, label, ie, edge;
  DBuf<uint8_t> kind;
  DBuf<double> rx_pos, length, pos, nrm;
  // with want_keys: DFS keys (4 words, word-major [4][n]) and group hashes, output order
  DBuf<uint64_t> keys, hash;
};

struct RefineDevIn {
  uint32_t n, stride;
  const double *tx, *rx, *pos, *nrm, *coarse_length;
  const uint32_t *n_inter, *label, *edge;
  const uint8_t* kind;
  uint32_t first = 0, step = 1;  // refine only candidates first + i * step (shards)
};

struct RefineDevOut {
  DBuf<int32_t> reason;
  DBuf<uint8_t> has_path;
  DBuf<double> pos, nrm, length, delay, gnorm;
  DBuf<uint32_t> label, iters;
  uint64_t trials = 0, marches = 0;  // work counters (summed over candidates)
  uint64_t trial_nodes = 0, iter_nodes = 0;  // the same weighted by the path's node count
};

void transmission_device(Ctx& ctx, const GridDev& grid, const SceneDev& scene, uint32_t tx_index, TxDev& out);
void propagate_device(Ctx& ctx, const GridDev& grid, const SceneDev& scene, uint32_t tx_index, const uint32_t* hit_ie,
                      const uint8_t* hit_kind, const double* hit_pos, const double* hit_nrm, const double* hit_inc,
                      uint32_t n_hits, const pcr_trace_params& p, CandDev& out, TraceStats& stats,
                      uint32_t shard = 0, uint32_t n_shards = 1, bool want_keys = false);
// Sharded pipeline: a shard's kept candidates of one TX as exchange rows
// (shard_rows.cuh; `rows` holds c.n * cand_row_bytes(c.stride) bytes), and the global
// first-kappa over the rows of every shard.
void pack_cand_rows(Ctx& ctx, const CandDev& c, uint32_t tx_index, uint8_t* rows);
void kappa_merge_rows(Ctx& ctx, const uint8_t* rows, uint64_t n, uint32_t stride, int kappa, uint32_t n_tx,
                      CandDev& out, std::vector<uint32_t>& per_tx);
void refine_device(Ctx& ctx, const GridDev& grid, const SceneDev& scene, const RefineDevIn& in,
                   const pcr_refine_params& p, RefineDevOut& out);

}  // namespace pcr
