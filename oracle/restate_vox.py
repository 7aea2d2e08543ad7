"""CPU restatement of stage 1 (voxelization) — TEST INFRASTRUCTURE ONLY.

numpy + small Python loops restating build_grid (proj/src/voxel_grid.cpp:82-227),
compute_march_distances (:229-268) and reception_point_of (:61-80) operation by
operation, for small inputs. It is checked bit for bit against the compiled
reference (oracle/_ref) in tests/test_cpu.py, and so pins the reference's integer
and FP64 semantics independently of the CUDA path. Never imported by the product.
"""
from __future__ import annotations

import math

import numpy as np

MARCH_NO_IES = 2147483647


def _dot(a, b):
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]


def _locate(p, origin, se, dims, dv):
    """locate_subvoxel + local_linear (voxel_grid.cpp:19-34)"""
    vox, loc = [0, 0, 0], [0, 0, 0]
    for a in range(3):
        g = int(math.floor((p[a] - origin[a]) / se))
        g = min(max(g, 0), dims[a] * dv - 1)
        vox[a] = g // dv
        loc[a] = g - vox[a] * dv
    voxel = vox[0] + dims[0] * (vox[1] + dims[1] * vox[2])
    sub = loc[0] + dv * (loc[1] + dv * loc[2])
    return voxel, sub


def build_grid(scene, voxel_size=0.5, division_factor=2, max_cells=1 << 27):
    if not voxel_size > 0.0:
        raise RuntimeError("voxel_size must be > 0")
    if division_factor < 1:
        raise RuntimeError("division_factor must be >= 1")
    s = scene.normalized()
    # scene_bounds (scene.cpp:93-106)
    mn = [np.finfo(np.float64).max] * 3
    mx = [np.finfo(np.float64).min] * 3
    pts = [s.position] + [s.edges[:, 0:3], s.edges[:, 3:6], s.tx, s.rx]
    for arr in pts:
        if len(arr):
            for a in range(3):
                mn[a] = min(mn[a], float(arr[:, a].min()))
                mx[a] = max(mx[a], float(arr[:, a].max()))
    if not all(mn[a] <= mx[a] for a in range(3)):
        raise RuntimeError("empty scene")
    origin = [mn[a] - voxel_size for a in range(3)]
    hi = [mx[a] + voxel_size for a in range(3)]
    dims, prod = [0, 0, 0], 1.0
    for a in range(3):
        span = (hi[a] - origin[a]) / voxel_size
        dims[a] = max(1, int(math.ceil(span - 1e-9)))
        prod *= dims[a]
    if prod > float(max_cells):
        raise RuntimeError("grid too large")
    n_cells = int(prod)
    dv = division_factor
    se = voxel_size / dv
    radius = 0.5 * math.sqrt(3.0) * se

    # bins sorted by (voxel, subvoxel, label, point) (voxel_grid.cpp:108-124)
    n = len(s.label)
    vox = np.zeros(n, np.int64)
    sub = np.zeros(n, np.int64)
    for i in range(n):
        vox[i], sub[i] = _locate(s.position[i], origin, se, dims, dv)
    order = np.lexsort((np.arange(n), s.label.astype(np.int64), sub, vox))
    ies = []
    point_indices = []
    i = 0
    while i < n:
        j = i
        while j < n and vox[order[j]] == vox[order[i]] and sub[order[j]] == sub[order[i]] and \
                s.label[order[j]] == s.label[order[i]]:
            j += 1
        first = order[i]
        n0, p0 = s.normal[first], s.position[first]
        planar = True
        for k in range(i, j):
            q = order[k]
            if _dot(s.normal[q], n0) < 1.0 - 1e-12 or abs(_dot(s.position[q] - p0, n0)) > 1e-9:
                planar = False
                break
        begin = len(point_indices)
        point_indices.extend(int(q) for q in order[i:j])
        ies.append(dict(kind=0, label=int(s.label[first]), voxel=int(vox[first]), sub=int(sub[first]),
                        point_begin=begin, point_end=len(point_indices), planar=planar,
                        plane_point=p0.copy(), plane_normal=n0.copy(), seg_start=np.zeros(3),
                        seg_end=np.zeros(3), edge=0, rx=0))
        i = j

    # edge pieces (voxel_grid.cpp:160-195)
    for e in range(len(s.edge_label)):
        st, en = s.edges[e, 0:3], s.edges[e, 3:6]
        dvec = en - st
        ln = math.sqrt(_dot(dvec, dvec))
        if not ln > 0.0:
            continue
        dr = dvec / ln
        cuts = [0.0, ln]
        for a in range(3):
            if abs(dr[a]) < 1e-15:
                continue
            lo_, hi_ = min(st[a], en[a]), max(st[a], en[a])
            k_lo = int(math.ceil((lo_ - origin[a]) / se))
            k_hi = int(math.floor((hi_ - origin[a]) / se))
            for k in range(k_lo, k_hi + 1):
                t = ((origin[a] + k * se) - st[a]) / dr[a]
                if 1e-12 < t < ln - 1e-12:
                    cuts.append(t)
        cuts.sort()
        for c in range(len(cuts) - 1):
            if cuts[c + 1] - cuts[c] < 1e-12:
                continue
            pa = st + cuts[c] * dr
            pb = st + cuts[c + 1] * dr
            vv, ss = _locate(0.5 * (pa + pb), origin, se, dims, dv)
            ies.append(dict(kind=1, label=int(s.edge_label[e]), voxel=vv, sub=ss, point_begin=0, point_end=0,
                            planar=False, plane_point=np.zeros(3), plane_normal=np.array([0.0, 0.0, 1.0]),
                            seg_start=pa, seg_end=pb, edge=e, rx=0))
    # receivers (voxel_grid.cpp:198-208)
    for r in range(len(s.rx_id)):
        vv, ss = _locate(s.rx[r], origin, se, dims, dv)
        ies.append(dict(kind=2, label=int(s.rx_id[r]), voxel=vv, sub=ss, point_begin=0, point_end=0, planar=False,
                        plane_point=np.zeros(3), plane_normal=np.array([0.0, 0.0, 1.0]), seg_start=np.zeros(3),
                        seg_end=np.zeros(3), edge=0, rx=int(s.rx_id[r])))
    # canonical order (voxel_grid.cpp:50-57, 210)
    ies.sort(key=lambda d: (d["voxel"], d["sub"], d["kind"], d["label"], d["edge"], d["rx"],
                            tuple(float(x) for x in d["seg_start"])))
    # spheres and reception points (voxel_grid.cpp:212-216, 36-48, 61-80)
    for d in ies:
        v = [d["voxel"] % dims[0], (d["voxel"] // dims[0]) % dims[1], d["voxel"] // (dims[0] * dims[1])]
        l = [d["sub"] % dv, (d["sub"] // dv) % dv, d["sub"] // (dv * dv)]
        d["sphere_center"] = np.array([(origin[a] + v[a] * voxel_size) + (l[a] + 0.5) * se for a in range(3)])
        if d["kind"] == 0:
            acc = np.zeros(3)
            for q in point_indices[d["point_begin"]:d["point_end"]]:
                acc = acc + s.position[q]
            d["reception_point"] = acc / float(d["point_end"] - d["point_begin"])
        elif d["kind"] == 1:
            d["reception_point"] = 0.5 * (d["seg_start"] + d["seg_end"])
        else:
            k = [r for r in range(len(s.rx_id)) if s.rx_id[r] == d["rx"]][0]
            d["reception_point"] = s.rx[k].copy()
    begin = np.zeros(n_cells, np.uint32)
    end = np.zeros(n_cells, np.uint32)
    for i, d in enumerate(ies):
        c = d["voxel"]
        if begin[c] == end[c]:
            begin[c] = i
        end[c] = i + 1
    g = {
        "origin": np.array(origin), "dims": np.array(dims, np.int32), "voxel_size": voxel_size,
        "division_factor": dv, "cell_ie_begin": begin, "cell_ie_end": end,
        "ie_kind": np.array([d["kind"] for d in ies], np.uint8).reshape(-1),
        "ie_label": np.array([d["label"] for d in ies], np.uint32).reshape(-1),
        "ie_reception_point": np.array([d["reception_point"] for d in ies]).reshape(-1, 3),
        "ie_sphere_center": np.array([d["sphere_center"] for d in ies]).reshape(-1, 3),
        "ie_sphere_radius": np.full(len(ies), radius),
        "ie_point_begin": np.array([d["point_begin"] for d in ies], np.uint32).reshape(-1),
        "ie_point_end": np.array([d["point_end"] for d in ies], np.uint32).reshape(-1),
        "ie_seg_start": np.array([d["seg_start"] for d in ies]).reshape(-1, 3),
        "ie_seg_end": np.array([d["seg_end"] for d in ies]).reshape(-1, 3),
        "ie_edge_index": np.array([d["edge"] for d in ies], np.uint32).reshape(-1),
        "ie_rx_id": np.array([d["rx"] for d in ies], np.uint32).reshape(-1),
        "ie_planar": np.array([d["planar"] for d in ies], np.uint8).reshape(-1),
        "ie_plane_point": np.array([d["plane_point"] for d in ies]).reshape(-1, 3),
        "ie_plane_normal": np.array([d["plane_normal"] for d in ies]).reshape(-1, 3),
        "ie_voxel": np.array([d["voxel"] for d in ies], np.uint32).reshape(-1),
        "ie_subvoxel": np.array([d["sub"] for d in ies], np.uint32).reshape(-1),
        "point_indices": np.array(point_indices, np.uint32),
    }
    g["cell_march"] = march_distances(dims, begin != end)
    return g


def march_distances(dims, occupied):
    """compute_march_distances (voxel_grid.cpp:229-268): BFS over the 26-neighbourhood."""
    dx, dy, dz = dims
    dist = np.full(dx * dy * dz, MARCH_NO_IES, np.int32)
    frontier = list(np.nonzero(occupied)[0])
    for c in frontier:
        dist[c] = 0
    d = 0
    while frontier:
        d += 1
        nxt = []
        for idx in frontier:
            x, y, z = idx % dx, (idx // dx) % dy, idx // (dx * dy)
            for oz in (-1, 0, 1):
                for oy in (-1, 0, 1):
                    for ox in (-1, 0, 1):
                        nx, ny, nz = x + ox, y + oy, z + oz
                        if nx < 0 or ny < 0 or nz < 0 or nx >= dx or ny >= dy or nz >= dz:
                            continue
                        n = nx + dx * (ny + dy * nz)
                        if dist[n] != MARCH_NO_IES:
                            continue
                        dist[n] = d
                        nxt.append(n)
        frontier = nxt
    return dist
