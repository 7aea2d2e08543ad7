// sort.cu — exclusive scan (reduce-then-scan) and a stable LSD radix sort.
//
// Radix pass (8-bit digits, 2048-key tiles, 256 threads = 8 warps, 8 keys/thread):
//   upsweep   : per-tile digit histogram -> counts[digit * n_tiles + tile]
//   scan      : exclusive scan of counts (digit-major = global stable offsets)
//   downsweep : each warp walks a contiguous 256-key run in 32-key chunks; peers
//               with the same digit are found with __match_any_sync, ranked by
//               lane, and the warp's running per-digit count lives in shared
//               memory; a per-digit prefix over warps makes the tile order
//               stable; the tile is placed digit-sorted in shared memory and
//               written out run by run (coalesced). Keys are read twice
//               (histogram + scatter) and written once.
#include "common.cuh"
#include "sort.cuh"

namespace pcr {

uint64_t g_launch_count = 0, g_h2d_bytes = 0, g_d2h_bytes = 0;

bool sync_launches() {
  static const bool on = [] {
    const char* e = std::getenv("PCR_SYNC_LAUNCHES");
    return e && e[0] == '1';
  }();
  return on;
}

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// Block-wide exclusive scan of per-thread values; returns the block total.
template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T& excl) {
  __shared__ T warp_tot[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const T inc = warp_inclusive_scan(v);
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    T t = lane < nw ? warp_tot[lane] : T(0);
    t = warp_inclusive_scan(t);
    if (lane < nw) warp_tot[lane] = t;
  }
  __syncthreads();
  const T warp_base = wid ? warp_tot[wid - 1] : T(0);
  excl = warp_base + inc - v;
  const T total = warp_tot[(blockDim.x >> 5) - 1];
  __syncthreads();
  return total;
}

template <typename T>
__global__ void scan_reduce_kernel(const T* __restrict__ in, size_t n, T* __restrict__ partial) {
  const size_t base = static_cast<size_t>(blockIdx.x) * kScanTile;
  T s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const size_t i = base + static_cast<size_t>(k) * kScanThreads + threadIdx.x;
    if (i < n) s += in[i];
  }
  T excl;
  const T tot = block_exclusive_scan(s, excl);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

template <typename T>
__global__ void scan_tile_kernel(const T* __restrict__ in, T* __restrict__ out, size_t n,
                                 const T* __restrict__ tile_offset, T* __restrict__ total) {
  const size_t base = static_cast<size_t>(blockIdx.x) * kScanTile + static_cast<size_t>(threadIdx.x) * kScanItems;
  T v[kScanItems];
  T s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const size_t i = base + k;
    v[k] = i < n ? in[i] : T(0);
    s += v[k];
  }
  T excl;
  const T tot = block_exclusive_scan(s, excl);
  T run = excl + (tile_offset ? tile_offset[blockIdx.x] : T(0));
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const size_t i = base + k;
    if (i < n) out[i] = run;
    run += v[k];
  }
  if (total && threadIdx.x == blockDim.x - 1 && blockIdx.x == gridDim.x - 1) *total = run;
  (void)tot;
}

template <typename T>
void exclusive_scan_impl(const T* in, T* out, size_t n, T* total_dev, cudaStream_t s) {
  if (n == 0) {
    if (total_dev) PCR_CUDA(cudaMemsetAsync(total_dev, 0, sizeof(T), s));
    return;
  }
  const size_t tiles = (n + kScanTile - 1) / kScanTile;
  if (tiles == 1) {
    count_launch();
    scan_tile_kernel<T><<<1, kScanThreads, 0, s>>>(in, out, n, nullptr, total_dev);
    PCR_LAUNCH_CHECK();
    return;
  }
  DBuf<T> partial(tiles, s);
  count_launch();
  scan_reduce_kernel<T><<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(in, n, partial.get());
  PCR_LAUNCH_CHECK();
  exclusive_scan_impl<T>(partial.get(), partial.get(), tiles, nullptr, s);
  count_launch();
  scan_tile_kernel<T><<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(in, out, n, partial.get(), total_dev);
  PCR_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------
constexpr int kRadixThreads = 256;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixIpt = 8;  // keys per thread
constexpr int kRadixTile = kRadixThreads * kRadixIpt;
constexpr int kRadixDigits = 256;

__global__ void __launch_bounds__(kRadixThreads) radix_upsweep(const uint64_t* __restrict__ keys, size_t n,
                                                                 int shift, uint32_t* __restrict__ counts,
                                                                 uint32_t n_tiles) {
  __shared__ uint32_t hist[kRadixDigits];
  hist[threadIdx.x] = 0;
  __syncthreads();
  const size_t base = static_cast<size_t>(blockIdx.x) * kRadixTile;
#pragma unroll 4
  for (int k = 0; k < kRadixIpt; ++k) {
    const size_t i = base + static_cast<size_t>(k) * kRadixThreads + threadIdx.x;
    if (i < n) atomicAdd(&hist[(keys[i] >> shift) & 0xffu], 1u);
  }
  __syncthreads();
  counts[static_cast<size_t>(threadIdx.x) * n_tiles + blockIdx.x] = hist[threadIdx.x];
}

// One tile: rank every key within its digit (warp match + per-warp counters), place
// the tile digit-sorted in shared memory, then write it out run by run so consecutive
// threads store consecutive addresses of one digit's output range (coalesced). The
// order within a digit stays the input order: the sort is stable.
__global__ void __launch_bounds__(kRadixThreads) radix_downsweep(
    const uint64_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, uint64_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, size_t n, int shift, const uint32_t* __restrict__ offsets, uint32_t n_tiles) {
  __shared__ uint32_t cnt[kRadixWarps][kRadixDigits];
  __shared__ uint32_t dstart[kRadixDigits];
  __shared__ uint64_t stage[kRadixTile];  // keys, then (reused) values
  __shared__ uint8_t sdig[kRadixTile];
  for (int i = threadIdx.x; i < kRadixWarps * kRadixDigits; i += kRadixThreads) (&cnt[0][0])[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const size_t tile0 = static_cast<size_t>(blockIdx.x) * kRadixTile;
  const size_t base = tile0 + static_cast<size_t>(wid) * 32 * kRadixIpt;
  const uint32_t tile_n = static_cast<uint32_t>(n - tile0 < static_cast<size_t>(kRadixTile) ? n - tile0 : kRadixTile);
  uint64_t key[kRadixIpt];
  uint32_t loc[kRadixIpt];
#pragma unroll
  for (int k = 0; k < kRadixIpt; ++k) {
    const size_t i = base + static_cast<size_t>(k) * 32 + lane;
    const bool ok = i < n;
    key[k] = ok ? keys_in[i] : 0ull;
    const uint32_t d = ok ? static_cast<uint32_t>((key[k] >> shift) & 0xffu) : (0x100u + lane);
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t rank = __popc(peers & lt_mask);
    uint32_t before = 0;
    if (ok) before = cnt[wid][d];
    __syncwarp();
    if (ok && (peers & lt_mask) == 0) cnt[wid][d] = before + __popc(peers);
    __syncwarp();
    loc[k] = before + rank;
  }
  __syncthreads();
  {
    // per digit: exclusive over warps, then the digit's start within the tile
    const int d = threadIdx.x;  // one digit per thread
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w) {
      const uint32_t t = cnt[w][d];
      cnt[w][d] = run;
      run += t;
    }
    // block exclusive scan of the digit totals (256 threads = 256 digits)
    uint32_t incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    __shared__ uint32_t wsum[kRadixWarps];
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    uint32_t woff = 0;
    for (int w = 0; w < wid; ++w) woff += wsum[w];
    dstart[d] = woff + incl - run;
  }
  __syncthreads();
  uint32_t lpos[kRadixIpt];
#pragma unroll
  for (int k = 0; k < kRadixIpt; ++k) {
    const size_t i = base + static_cast<size_t>(k) * 32 + lane;
    if (i < n) {
      const uint32_t d = static_cast<uint32_t>((key[k] >> shift) & 0xffu);
      lpos[k] = dstart[d] + cnt[wid][d] + loc[k];
      stage[lpos[k]] = key[k];
      sdig[lpos[k]] = static_cast<uint8_t>(d);
    }
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < tile_n; j += kRadixThreads) {
    const uint32_t d = sdig[j];
    keys_out[static_cast<size_t>(offsets[static_cast<size_t>(d) * n_tiles + blockIdx.x]) + (j - dstart[d])] = stage[j];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kRadixIpt; ++k) {
    const size_t i = base + static_cast<size_t>(k) * 32 + lane;
    if (i < n) reinterpret_cast<uint32_t*>(stage)[lpos[k]] = vals_in[i];
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < tile_n; j += kRadixThreads) {
    const uint32_t d = sdig[j];
    vals_out[static_cast<size_t>(offsets[static_cast<size_t>(d) * n_tiles + blockIdx.x]) + (j - dstart[d])] =
        reinterpret_cast<const uint32_t*>(stage)[j];
  }
}

__global__ void iota_kernel(uint32_t* v, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    v[i] = static_cast<uint32_t>(i);
}

}  // namespace

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t n, uint32_t* total_dev, cudaStream_t s) {
  exclusive_scan_impl<uint32_t>(in, out, n, total_dev, s);
}
void exclusive_scan_u64(const uint64_t* in, uint64_t* out, size_t n, uint64_t* total_dev, cudaStream_t s) {
  exclusive_scan_impl<uint64_t>(in, out, n, total_dev, s);
}

void iota_u32(uint32_t* vals, size_t n, cudaStream_t s) {
  if (!n) return;
  count_launch();
  iota_kernel<<<blocks_for(n, 256), 256, 0, s>>>(vals, n);
  PCR_LAUNCH_CHECK();
}

void radix_sort_pairs(uint64_t* keys, uint32_t* vals, size_t n, int begin_bit, int end_bit, cudaStream_t s) {
  if (n <= 1 || end_bit <= begin_bit) return;
  if (n >= (size_t(1) << 32)) throw Error(1, "radix_sort_pairs: too many keys");
  const uint32_t n_tiles = static_cast<uint32_t>((n + kRadixTile - 1) / kRadixTile);
  DBuf<uint64_t> k2(n, s);
  DBuf<uint32_t> v2(n, s);
  DBuf<uint32_t> counts(static_cast<size_t>(kRadixDigits) * n_tiles, s);
  uint64_t* kin = keys;
  uint32_t* vin = vals;
  uint64_t* kout = k2.get();
  uint32_t* vout = v2.get();
  for (int shift = begin_bit; shift < end_bit; shift += 8) {
    count_launch();
    radix_upsweep<<<n_tiles, kRadixThreads, 0, s>>>(kin, n, shift, counts.get(), n_tiles);
    PCR_LAUNCH_CHECK();
    exclusive_scan_u32(counts.get(), counts.get(), counts.size(), nullptr, s);
    count_launch();
    radix_downsweep<<<n_tiles, kRadixThreads, 0, s>>>(kin, vin, kout, vout, n, shift, counts.get(), n_tiles);
    PCR_LAUNCH_CHECK();
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  if (kin != keys) {
    PCR_CUDA(cudaMemcpyAsync(keys, kin, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
    PCR_CUDA(cudaMemcpyAsync(vals, vin, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  }
}

}  // namespace pcr
