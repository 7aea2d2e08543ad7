"""Sharded voxelization (SURVEY §8e, C5 sweep at G GPUs): each shard builds the IEs of
a contiguous voxel range (about N / G points), the parts are gathered and assembled
into the grid. The assembled grid must equal the unsharded build_grid bit for bit —
every cell, IE field and point_indices entry — for any shard count.

The shards run one after another on the box's one GPU (shard.build_grid_sharded_local,
the same library calls the multi-process path makes), and once as two processes that
exchange the parts through torch.distributed (gloo; the GPU path uses NCCL)."""
import os
import socket

import numpy as np
import pytest

from conftest import assert_grid_equal
from fixtures import voxel_grid_scenes
from paper_2402_13747_b200 import abi, pcray, scenes, shard

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_shards", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("name", ["C1", "C2"])
def test_sharded_grid_equals_unsharded(gpu, name, n_shards):
    scene, _ = scenes.build_scene(name)
    ds = pcray.DeviceScene(scene)
    want = pcray.build_grid(ds).to_dict()
    got = shard.build_grid_sharded_local(ds, None, n_shards).to_dict()
    assert_grid_equal(got, want)


@pytest.mark.parametrize("vs,dv", [(0.5, 2), (1.0, 4), (0.25, 1), (0.7, 3)])
def test_sharded_grid_c5(gpu, vs, dv):
    """C5 geometry (street canyon) at 3M points, several (voxel, D_v), 4 and 7 shards."""
    base = scenes.config("C3")
    scene = scenes.scene_from_planar(base.planar, scenes.scaled_density(base, 3_000_000), base.seed)
    ds = pcray.DeviceScene(scene)
    params = abi.voxel_params(vs, dv)
    want = pcray.build_grid(ds, params).to_dict()
    for n in [4, 7]:
        assert_grid_equal(shard.build_grid_sharded_local(ds, params, n).to_dict(), want)


@pytest.mark.parametrize("name", ["edge_clip", "dup_rx_ids", "oblique_edge", "partition", "nonplanar_patch",
                                  "single_point"])
def test_sharded_grid_small_scenes(gpu, name):
    """Edge pieces and receivers land in their voxel's shard; shards may be empty."""
    scene = voxel_grid_scenes()[name]
    ds = pcray.DeviceScene(scene)
    want = pcray.build_grid(ds).to_dict()
    for n in [2, 4, 16]:
        assert_grid_equal(shard.build_grid_sharded_local(ds, None, n).to_dict(), want)


def test_grid_assemble_rejects_bad_parts(gpu):
    import torch

    scene, _ = scenes.build_scene("C1")
    ds = pcray.DeviceScene(scene)
    parts, sizes = [], []
    for r in range(2):
        nb = pcray.grid_part_build(ds, r, 2)
        t = torch.empty(nb, dtype=torch.uint8, device="cuda")
        pcray.grid_part_copy(ds.ctx, t.data_ptr())
        parts.append(t)
        sizes.append(nb)
    torch.cuda.synchronize()
    allp = torch.cat(parts)
    with pytest.raises(pcray.PcrError, match="out of order|miss voxels"):  # shards swapped
        both = torch.cat([parts[1], parts[0]])
        torch.cuda.synchronize()
        pcray.grid_assemble(ds.ctx, both.data_ptr(), [0, sizes[1]], [sizes[1], sizes[0]])
    with pytest.raises(pcray.PcrError, match="miss voxels"):  # a shard missing
        pcray.grid_assemble(ds.ctx, allp.data_ptr(), [0], [sizes[0]])
    with pytest.raises(pcray.PcrError, match="truncated"):
        pcray.grid_assemble(ds.ctx, allp.data_ptr(), [0, sizes[0]], [sizes[0], 64])
    with pytest.raises(pcray.PcrError, match="shard index out of range"):
        pcray.grid_part_build(ds, 2, 2)


def _rank(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    # gloo keeps the exchange on the host: both ranks share the one GPU but never wait
    # on each other's kernels
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        scene, _ = scenes.build_scene("C2")
        ds = pcray.DeviceScene(scene, pcray.Context(0))
        g = shard.build_grid_sharded(ds).to_dict()
        q.put((rank, {k: (v.tobytes() if isinstance(v, np.ndarray) else v) for k, v in g.items()}))
    finally:
        dist.destroy_process_group()


def test_sharded_grid_two_processes(gpu):
    import multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    scene, _ = scenes.build_scene("C2")
    want = pcray.build_grid(pcray.DeviceScene(scene)).to_dict()
    for r in range(2):
        for k, v in want.items():
            if isinstance(v, np.ndarray):
                assert got[r][k] == v.tobytes(), (r, k)
