// sort.cuh — device-wide primitives written for this library: exclusive scan and a
// stable LSD radix sort of (u64 key, u32 value) pairs. Stability is what makes
// the voxelization order (voxel, subvoxel, label, point) reproducible: the
// values start as point indices in ascending order, so ties keep index order
// (voxel_grid.cpp:121-124 sorts full tuples with unique keys; same result).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace pcr {

// out[i] = sum(in[0..i)); *total_dev (optional, device) = sum(in). in == out allowed.
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t n, uint32_t* total_dev, cudaStream_t s);
void exclusive_scan_u64(const uint64_t* in, uint64_t* out, size_t n, uint64_t* total_dev, cudaStream_t s);

// Stable sort by bits [begin_bit, end_bit) of keys; vals permuted alongside.
void radix_sort_pairs(uint64_t* keys, uint32_t* vals, size_t n, int begin_bit, int end_bit, cudaStream_t s);

// vals[i] = i
void iota_u32(uint32_t* vals, size_t n, cudaStream_t s);

// Number of significant bits of x (0 for x == 0).
inline int bit_width(uint64_t x) {
  int b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

}  // namespace pcr
