// host_alloc.hpp — allocation/free of the C-ABI result structs (include/pcray_b200.h).
#pragma once

#include <cstdlib>
#include <cstring>

#include "../../include/pcray_b200.h"

namespace pcr {

template <typename T>
T* halloc(size_t n) {
  void* p = std::calloc(n ? n : 1, sizeof(T));
  if (!p) throw std::bad_alloc();
  return static_cast<T*>(p);
}

inline pcr_paths* alloc_paths(uint64_t n, uint32_t stride) {
  if (stride == 0) stride = 1;
  pcr_paths* p = halloc<pcr_paths>(1);
  p->n = n;
  p->stride = stride;
  const size_t m = static_cast<size_t>(n) * stride;
  p->tx_id = halloc<uint32_t>(n);
  p->rx_id = halloc<uint32_t>(n);
  p->tx_position = halloc<double>(3 * n);
  p->rx_position = halloc<double>(3 * n);
  p->length = halloc<double>(n);
  p->delay = halloc<double>(n);
  p->converged = halloc<uint8_t>(n);
  p->gradient_norm = halloc<double>(n);
  p->n_inter = halloc<uint32_t>(n);
  p->kind = halloc<uint8_t>(m);
  p->position = halloc<double>(3 * m);
  p->label = halloc<uint32_t>(m);
  p->normal = halloc<double>(3 * m);
  p->ie_index = halloc<uint32_t>(m);
  p->edge_index = halloc<uint32_t>(m);
  return p;
}

inline void free_paths_arrays(pcr_paths* p) {
  void* a[] = {p->tx_id, p->rx_id, p->tx_position, p->rx_position, p->length, p->delay, p->converged,
               p->gradient_norm, p->n_inter, p->kind, p->position, p->label, p->normal, p->ie_index,
               p->edge_index};
  for (void* x : a) std::free(x);
}

inline pcr_grid_host* alloc_grid_host(uint64_t nc, uint64_t ni, uint64_t np) {
  pcr_grid_host* h = halloc<pcr_grid_host>(1);
  h->n_cells = nc;
  h->n_ies = ni;
  h->n_point_indices = np;
  h->cell_ie_begin = halloc<uint32_t>(nc);
  h->cell_ie_end = halloc<uint32_t>(nc);
  h->cell_march = halloc<int32_t>(nc);
  h->ie_kind = halloc<uint8_t>(ni);
  h->ie_label = halloc<uint32_t>(ni);
  h->ie_reception_point = halloc<double>(3 * ni);
  h->ie_sphere_center = halloc<double>(3 * ni);
  h->ie_sphere_radius = halloc<double>(ni);
  h->ie_point_begin = halloc<uint32_t>(ni);
  h->ie_point_end = halloc<uint32_t>(ni);
  h->ie_seg_start = halloc<double>(3 * ni);
  h->ie_seg_end = halloc<double>(3 * ni);
  h->ie_edge_index = halloc<uint32_t>(ni);
  h->ie_rx_id = halloc<uint32_t>(ni);
  h->ie_planar = halloc<uint8_t>(ni);
  h->ie_plane_point = halloc<double>(3 * ni);
  h->ie_plane_normal = halloc<double>(3 * ni);
  h->ie_voxel = halloc<uint32_t>(ni);
  h->ie_subvoxel = halloc<uint32_t>(ni);
  h->point_indices = halloc<uint32_t>(np);
  return h;
}

inline void free_grid_host(pcr_grid_host* h) {
  if (!h) return;
  void* a[] = {h->cell_ie_begin, h->cell_ie_end,      h->cell_march,       h->ie_kind,         h->ie_label,
               h->ie_reception_point, h->ie_sphere_center, h->ie_sphere_radius, h->ie_point_begin, h->ie_point_end,
               h->ie_seg_start,  h->ie_seg_end,       h->ie_edge_index,    h->ie_rx_id,        h->ie_planar,
               h->ie_plane_point, h->ie_plane_normal, h->ie_voxel,         h->ie_subvoxel,     h->point_indices};
  for (void* x : a) std::free(x);
  std::free(h);
}

}  // namespace pcr
