// gridparts.cu — sharded voxelization: grid parts as bytes, and the
// assembly of the whole VoxelGrid from every shard's part.
//
// Shard r builds the IEs of its contiguous voxel range [v_r, v_{r+1}) (voxelize.cu,
// build_grid_device with a VoxelShard): splitters put about N / n points in each range,
// the shard sorts and groups only its own points, and keeps the edge pieces and
// receivers that fall in its voxels. Because the canonical IE order (voxel_grid.cpp:
// 50-57, :210) is voxel-major and point_indices lists the surface IEs' payloads in IE
// order, the whole grid is the concatenation of the parts in shard order: IE records
// unchanged, point ranges shifted by the points of the earlier parts, then cells from
// the concatenated voxel column and the Chebyshev transform — bit for bit the grid of
// the unsharded build. The parts travel as flat byte buffers (all-gathered over NCCL
// by the caller; shard.py / the C++ driver), so assembly reads them from device memory.
//
// Part layout: 128-byte header {magic, n_ies, n_pidx, voxel_lo, voxel_hi, origin xyz,
// voxel_size, dims xyz, division_factor}, then meta, label, edge, rx, voxel, sub
// (u32 x n_ies each), sc, rp, pp, pn, seg_s, seg_e (double4 x n_ies), range (uint2 x
// n_ies), point_indices (u32 x n_pidx); every array starts on a 16-byte boundary.
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "device_state.cuh"
#include "sort.cuh"

namespace pcr {
namespace {

constexpr uint64_t kPartMagic = 0x3154524150524350ull;  // "PCRPART1"

struct PartHeader {
  uint64_t magic, n_ies, n_pidx, voxel_lo, voxel_hi;
  double origin[3], voxel_size;
  int32_t dims[3], dv;
  uint64_t pad[5];
};
static_assert(sizeof(PartHeader) == 128, "part header");

uint64_t a16(uint64_t x) { return (x + 15) & ~15ull; }

// byte offsets of the arrays inside a part with n IEs and m point indices
struct PartLayout {
  uint64_t u32[6], d4[6], range, pidx, total;
  PartLayout(uint64_t n, uint64_t m) {
    uint64_t o = sizeof(PartHeader);
    for (int k = 0; k < 6; ++k) {
      u32[k] = o;
      o = a16(o + 4 * n);
    }
    for (int k = 0; k < 6; ++k) {
      d4[k] = o;
      o = a16(o + 32 * n);
    }
    range = o;
    o = a16(o + 8 * n);
    pidx = o;
    total = a16(o + 4 * m);
  }
};

__global__ void shift_range_kernel(uint2* range, const uint32_t* meta, uint64_t n, uint32_t shift) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    if ((meta[i] & 3u) == 0) {  // SurfacePoints: payload range into point_indices
      range[i].x += shift;
      range[i].y += shift;
    }
}

__global__ void cells_from_voxels_kernel(const uint32_t* __restrict__ voxel, uint32_t n, int4* __restrict__ cells) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t v = voxel[i];
    if (i == 0 || voxel[i - 1] != v) cells[v].x = static_cast<int>(i);
    if (i + 1 == n || voxel[i + 1] != v) cells[v].y = static_cast<int>(i + 1);
  }
}

unsigned grid_blocks(uint64_t n) {
  const uint64_t b = (n + 255) / 256;
  return static_cast<unsigned>(b < 1 ? 1 : (b > 148ull * 64 ? 148ull * 64 : b));
}

}  // namespace

uint64_t grid_part_bytes(const GridDev& part) { return PartLayout(part.n_ies, part.n_pidx).total; }

void grid_part_serialize(Ctx& ctx, const GridDev& p, void* dst_device) {
  cudaStream_t s = ctx.stream;
  uint8_t* d = static_cast<uint8_t*>(dst_device);
  const PartLayout L(p.n_ies, p.n_pidx);
  PartHeader h{};
  h.magic = kPartMagic;
  h.n_ies = p.n_ies;
  h.n_pidx = p.n_pidx;
  h.voxel_lo = p.part_voxel_lo;
  h.voxel_hi = p.part_voxel_hi;
  h.origin[0] = p.origin.x;
  h.origin[1] = p.origin.y;
  h.origin[2] = p.origin.z;
  h.voxel_size = p.voxel_size;
  for (int a = 0; a < 3; ++a) h.dims[a] = p.dims[a];
  h.dv = p.dv;
  PCR_CUDA(cudaMemcpyAsync(d, &h, sizeof(h), cudaMemcpyHostToDevice, s));
  const uint32_t* u32[6] = {p.meta.get(), p.label.get(), p.edge.get(), p.rx.get(), p.voxel.get(), p.sub.get()};
  const double4* d4[6] = {p.sc.get(), p.rp.get(), p.pp.get(), p.pn.get(), p.seg_s.get(), p.seg_e.get()};
  if (p.n_ies) {
    for (int k = 0; k < 6; ++k)
      PCR_CUDA(cudaMemcpyAsync(d + L.u32[k], u32[k], 4 * p.n_ies, cudaMemcpyDeviceToDevice, s));
    for (int k = 0; k < 6; ++k)
      PCR_CUDA(cudaMemcpyAsync(d + L.d4[k], d4[k], 32 * p.n_ies, cudaMemcpyDeviceToDevice, s));
    PCR_CUDA(cudaMemcpyAsync(d + L.range, p.range.get(), 8 * p.n_ies, cudaMemcpyDeviceToDevice, s));
  }
  if (p.n_pidx) PCR_CUDA(cudaMemcpyAsync(d + L.pidx, p.pidx.get(), 4 * p.n_pidx, cudaMemcpyDeviceToDevice, s));
  stream_wait(s);
}

void grid_assemble(Ctx& ctx, const uint8_t* parts, const uint64_t* offset, const uint64_t* bytes, uint32_t n_parts,
                   GridDev& out) {
  cudaStream_t s = ctx.stream;
  if (n_parts == 0) throw Error(1, "voxelize: no grid parts");
  std::vector<PartHeader> h(n_parts);
  for (uint32_t r = 0; r < n_parts; ++r) {
    if (bytes[r] < sizeof(PartHeader)) throw Error(1, "voxelize: grid part truncated");
    PCR_CUDA(cudaMemcpyAsync(&h[r], parts + offset[r], sizeof(PartHeader), cudaMemcpyDeviceToHost, s));
  }
  stream_wait(s);
  uint64_t n_ies = 0, n_pidx = 0;
  for (uint32_t r = 0; r < n_parts; ++r) {
    const PartHeader& x = h[r];
    if (x.magic != kPartMagic) throw Error(1, "voxelize: not a grid part");
    if (PartLayout(x.n_ies, x.n_pidx).total > bytes[r]) throw Error(1, "voxelize: grid part truncated");
    const bool same = std::memcmp(x.origin, h[0].origin, sizeof(x.origin)) == 0 && x.voxel_size == h[0].voxel_size &&
                      std::memcmp(x.dims, h[0].dims, sizeof(x.dims)) == 0 && x.dv == h[0].dv;
    if (!same) throw Error(1, "voxelize: grid parts of different grids");
    if (r && x.voxel_lo != h[r - 1].voxel_hi) throw Error(1, "voxelize: grid parts out of order");
    n_ies += x.n_ies;
    n_pidx += x.n_pidx;
  }
  const uint64_t n_cells = static_cast<uint64_t>(h[0].dims[0]) * h[0].dims[1] * h[0].dims[2];
  if (h[0].voxel_lo != 0 || h[n_parts - 1].voxel_hi != n_cells) throw Error(1, "voxelize: grid parts miss voxels");
  out.set_geometry(V3{h[0].origin[0], h[0].origin[1], h[0].origin[2]}, h[0].dims, h[0].voxel_size, h[0].dv);
  out.n_cells = n_cells;
  out.cells.alloc(n_cells ? n_cells : 1, s);
  PCR_CUDA(cudaMemsetAsync(out.cells.get(), 0, sizeof(int4) * (n_cells ? n_cells : 1), s));
  out.alloc_ies(n_ies, s);
  out.n_pidx = n_pidx;
  out.pidx.alloc(n_pidx ? n_pidx : 1, s);
  uint32_t* u32[6] = {out.meta.get(), out.label.get(), out.edge.get(), out.rx.get(), out.voxel.get(), out.sub.get()};
  double4* d4[6] = {out.sc.get(), out.rp.get(), out.pp.get(), out.pn.get(), out.seg_s.get(), out.seg_e.get()};
  uint64_t ie0 = 0, p0 = 0;
  for (uint32_t r = 0; r < n_parts; ++r) {
    const PartHeader& x = h[r];
    const PartLayout L(x.n_ies, x.n_pidx);
    const uint8_t* b = parts + offset[r];
    if (x.n_ies) {
      for (int k = 0; k < 6; ++k)
        PCR_CUDA(cudaMemcpyAsync(u32[k] + ie0, b + L.u32[k], 4 * x.n_ies, cudaMemcpyDeviceToDevice, s));
      for (int k = 0; k < 6; ++k)
        PCR_CUDA(cudaMemcpyAsync(d4[k] + ie0, b + L.d4[k], 32 * x.n_ies, cudaMemcpyDeviceToDevice, s));
      PCR_CUDA(cudaMemcpyAsync(out.range.get() + ie0, b + L.range, 8 * x.n_ies, cudaMemcpyDeviceToDevice, s));
      if (p0) {
        count_launch();
        shift_range_kernel<<<grid_blocks(x.n_ies), 256, 0, s>>>(out.range.get() + ie0, out.meta.get() + ie0, x.n_ies,
                                                                static_cast<uint32_t>(p0));
        PCR_LAUNCH_CHECK();
      }
    }
    if (x.n_pidx)
      PCR_CUDA(cudaMemcpyAsync(out.pidx.get() + p0, b + L.pidx, 4 * x.n_pidx, cudaMemcpyDeviceToDevice, s));
    ie0 += x.n_ies;
    p0 += x.n_pidx;
  }
  if (n_ies) {
    count_launch();
    cells_from_voxels_kernel<<<grid_blocks(n_ies), 256, 0, s>>>(out.voxel.get(), static_cast<uint32_t>(n_ies),
                                                                out.cells.get());
    PCR_LAUNCH_CHECK();
  }
  compute_march_distances_device(ctx, out);
  stream_wait(s);
}

}  // namespace pcr
