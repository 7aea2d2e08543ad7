"""Host side of the sharded pipeline, no GPU: the cyclic split, the byte
exchange over torch.distributed (gloo, world size 2 and 3), the counter sum, and the
first-kappa superset argument the per-shard pre-cap relies on (T9)."""
import os
import random
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2402_13747_b200 import shard


def test_cyclic_split_partitions():
    for n in [0, 1, 7, 100]:
        for world in [1, 2, 3, 8]:
            owned = [list(shard.shard_indices(n, r, world)) for r in range(world)]
            flat = sorted(i for o in owned for i in o)
            assert flat == list(range(n))
            for r, o in enumerate(owned):
                assert all(shard.shard_of(i, world) == r for i in o)


def first_kappa(items, kappa):
    """items: (key, group) in any order -> the first kappa keys per group in key order."""
    seen, keep = {}, []
    for key, grp in sorted(items):
        if seen.get(grp, 0) < kappa:
            keep.append((key, grp))
        seen[grp] = seen.get(grp, 0) + 1
    return keep


@pytest.mark.parametrize("seed", range(20))
def test_precap_superset_is_exact(seed):
    """Global first-kappa over the union of per-shard first-kappa lists equals the global
    first-kappa of everything (the merge in kappa_merge_rows)."""
    rng = random.Random(seed)
    n, world, kappa = rng.randint(0, 400), rng.randint(1, 6), rng.randint(1, 5)
    keys = rng.sample(range(10 ** 6), n)
    items = [(k, rng.randint(0, 12)) for k in keys]
    task = {k: rng.randint(0, 50) for k in keys}
    shards = [[it for it in items if shard.shard_of(task[it[0]], world) == r] for r in range(world)]
    merged = [it for s in shards for it in first_kappa(s, kappa)]
    rng.shuffle(merged)
    assert first_kappa(merged, kappa) == first_kappa(items, kappa)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sizes = [5, 0, 13][:world]
        buf = torch.full((sizes[rank],), rank + 1, dtype=torch.uint8)
        got = shard.all_gather_bytes(buf)
        empty = shard.all_gather_bytes(torch.empty(0, dtype=torch.uint8))
        st = shard.sum_stats(np.arange(7, dtype=np.uint64) * (rank + 1))
        g0 = shard.gather_bytes(buf, 0)
        q.put((rank, got.tolist(), empty.numel(), st.tolist(), None if g0 is None else g0.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sizes = [5, 0, 13][:world]
    want = [r + 1 for r in range(world) for _ in range(sizes[r])]
    tot = sum(range(1, world + 1))
    for rank, got, empty, st, g0 in res:
        assert got == want, rank
        assert empty == 0
        assert st == [i * tot for i in range(7)]
        assert g0 == (want if rank == 0 else None)
