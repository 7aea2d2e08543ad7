// shard_rows.cuh — the fixed-layout records ranks exchange when the pipeline is
// sharded: propagated candidates with their DFS keys (trace → κ merge)
// and refinement outcomes (refine → final dedup). Plain bytes, so any transport
// (NCCL all-gather of a uint8 tensor, a host copy) moves them unchanged.
#pragma once

#include <cstddef>
#include <cstdint>

namespace pcr {

// One propagated candidate: header + `stride` interaction levels.
struct CandRowHead {
  uint64_t key[4];  // DFS-order key, MSB-first (task, j1, ie2, j2, ..., rx_ie)
  uint64_t hash;    // group hash of (rx, label sequence)
  uint32_t tx_index, rx_id, n_inter, pad0;
  double rx_pos[3];
  double length;  // coarse chain length
  double pad1;
};
struct CandRowLevel {
  double pos[3];
  double nrm[3];
  uint32_t label, ie, edge, kind;
};
static_assert(sizeof(CandRowHead) == 96, "CandRowHead layout");
static_assert(sizeof(CandRowLevel) == 64, "CandRowLevel layout");
__host__ __device__ inline size_t cand_row_bytes(uint32_t stride) {
  return sizeof(CandRowHead) + sizeof(CandRowLevel) * stride;
}

// One refinement outcome of candidate `cand` (index into the merged candidate list).
struct OutRowHead {
  uint32_t cand;
  int32_t reason;
  uint32_t iters;
  uint32_t has_path;
  double length, delay, gnorm;
};
struct OutRowLevel {
  double pos[3];
  double nrm[3];
  uint32_t label, pad;
};
static_assert(sizeof(OutRowHead) == 40, "OutRowHead layout");
static_assert(sizeof(OutRowLevel) == 56, "OutRowLevel layout");
__host__ __device__ inline size_t out_row_bytes(uint32_t stride) {
  return sizeof(OutRowHead) + sizeof(OutRowLevel) * stride;
}

}  // namespace pcr
