"""Sharded pipeline: every shard split of run_pipeline_on_scene must give
the unsharded RunSummary exactly — same counts (incl. the work counters summed over
shards) and the same exact paths bit for bit, whatever the exchange order. The shards
run one after another in one process on one GPU (shard.run_pipeline_sharded_local),
which is the same library code path each rank runs under torchrun."""
import numpy as np
import pytest

from fixtures import box_room, make_scene
from paper_2402_13747_b200 import abi, pcray, scenes, shard

pytestmark = pytest.mark.gpu

COUNTS = ["point_count", "edge_count", "ie_count", "coarse_paths", "refined_paths", "exact_paths",
          "transmission_rays", "cone_traces", "visibility_tests", "refine_iterations", "refine_trials",
          "refine_marches", "walk_cells", "walk_ies", "hash"]


def assert_same_summary(got, ref):
    for k in COUNTS:
        assert got[k] == ref[k], f"{k}: {got[k]} != {ref[k]}"
    assert list(got["rejected"]) == list(ref["rejected"])
    assert list(got["grid_dims"]) == list(ref["grid_dims"])
    assert [n for n, _ in got["timings"]] == [n for n, _ in ref["timings"]]
    gp, rp = got["paths"], ref["paths"]
    assert set(gp) == set(rp)
    for k in rp:
        a, b = np.ascontiguousarray(gp[k]), np.ascontiguousarray(rp[k])
        assert a.shape == b.shape, k
        if a.dtype == np.float64:
            a, b = a.view(np.uint64), b.view(np.uint64)
        assert np.array_equal(a, b), f"paths[{k}] differs"


def screen_scene():
    p = scenes.PlanarScene()
    p.add_rect((-2, 0, 0), (4, 0, 0), (0, 0, 1), 0)
    p.add_rect((-2, 0, 0), (0, 0, 1), (4, 0, 0), 1)
    p.edges.append(((-2, 0, 1), (2, 0, 1), (0, -1, 0), (0, 1, 0), 2))
    p.tx.append([0.3, -1.5, 0.4])
    p.rx.append([-0.2, 1.8, 0.55])
    return scenes.scene_from_planar(p, 5000.0, 11)


@pytest.mark.parametrize("n_shards,order", [(1, None), (2, None), (2, [1, 0]), (3, [2, 0, 1]), (5, None)])
def test_sharded_box(gpu, n_shards, order):
    sc = make_scene(box_room((2, 2, 2), 0.06), tx=[(0.6, 0.7, 0.9), (1.4, 1.1, 0.5)],
                    rx=[(1.3, 1.2, 1.1), (0.4, 1.5, 1.6)])
    cfg = abi.default_run_config(max_interactions=2, kappa=3)
    ref = pcray.run_pipeline_on_scene(sc, cfg)
    got = shard.run_pipeline_sharded_local(sc, cfg, n_shards, order)
    assert ref["coarse_paths"] > 0
    assert_same_summary(got, ref)


def test_sharded_screen_diffraction(gpu):
    sc = screen_scene()
    cfg = abi.default_run_config(max_interactions=2)
    ref = pcray.run_pipeline_on_scene(sc, cfg)
    got = shard.run_pipeline_sharded_local(sc, cfg, 3, [1, 2, 0])
    assert_same_summary(got, ref)


def test_sharded_c1(gpu):
    scene, c = scenes.build_scene("C1")
    cfg = abi.default_run_config(**c.run)
    ref = pcray.run_pipeline_on_scene(scene, cfg)
    got = shard.run_pipeline_sharded_local(scene, cfg, 4, [3, 1, 0, 2])
    assert_same_summary(got, ref)


@pytest.mark.parametrize("kappa", [1, 100])
def test_sharded_c2_reduced_depth(gpu, kappa):
    """C2 (64 RX, diffraction edges) at depth 2: kappa = 1 makes the cross-shard merge
    decide nearly every group."""
    scene, _ = scenes.build_scene("C2")
    cfg = abi.default_run_config(max_interactions=2, max_diffractions=1, kappa=kappa)
    ref = pcray.run_pipeline_on_scene(scene, cfg)
    got = shard.run_pipeline_sharded_local(scene, cfg, 3, [2, 1, 0])
    assert_same_summary(got, ref)


def test_shard_errors(gpu):
    ctx = pcray.Context(0)
    with pytest.raises(pcray.PcrError, match="shard"):
        pcray.shard_outcomes(ctx, 0)
    sc = pcray.DeviceScene(make_scene(box_room((2, 2, 2), 0.1), tx=[(0.6, 0.7, 0.9)], rx=[(1.3, 1.2, 1.1)]), ctx)
    with pytest.raises(pcray.PcrError, match="shard: index out of range"):
        pcray.shard_trace(sc, abi.default_run_config(max_interactions=1), 2, 2)


def _rank(rank, world, port, q):
    import os

    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    # gloo keeps the exchange on the host: the ranks share one GPU but never wait on
    # each other's kernels (each shard's kernels run to completion before a collective)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        scene, c = scenes.build_scene("C1")
        ds = pcray.DeviceScene(scene, pcray.Context(0))
        s = shard.run_pipeline_sharded(ds, abi.default_run_config(**c.run))
        q.put((rank, None if s is None else {k: s[k] for k in COUNTS + ["paths"]}))
    finally:
        dist.destroy_process_group()


def test_run_pipeline_sharded_distributed(gpu):
    """shard.run_pipeline_sharded itself under torch.distributed (world 2)."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[1] is None
    scene, c = scenes.build_scene("C1")
    ref = pcray.run_pipeline_on_scene(scene, abi.default_run_config(**c.run))
    got = res[0]
    for k in COUNTS:
        assert got[k] == ref[k], k
    for k, v in ref["paths"].items():
        a, b = np.ascontiguousarray(got["paths"][k]), np.ascontiguousarray(v)
        if a.dtype == np.float64:
            a, b = a.view(np.uint64), b.view(np.uint64)
        assert np.array_equal(a, b), k
