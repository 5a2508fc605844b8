"""Host logic of the multi-GPU layer on CPU (no GPU): the exchange plan of
the single-process sample sort (ns_sample_sort_plan) and the shard-by-array
plan of the base-case / segmented batches (ns_shard_batch_plan), the latter
also driven by world_size 2 and 3 over gloo, each rank sorting its shard
with the oracle (the per-rank device step's CPU stand-in)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def test_sample_sort_plan_matches_definition(ns):
    from paper_2503_05934_b200 import multigpu
    rng = np.random.default_rng(1)
    for g in (1, 2, 3, 8):
        counts = rng.integers(0, 1000, size=(g, g))
        bounds = np.zeros((g, g + 1), np.int64)
        bounds[:, 1:] = np.cumsum(counts, axis=1)
        ro, rt = multigpu.sample_sort_plan(bounds)
        for dst in range(g):
            assert ro[dst, 0] == 0
            assert np.array_equal(np.diff(ro[dst]), counts[:, dst])
            assert rt[dst] == counts[:, dst].sum()
        assert rt.sum() == counts.sum()
    bad = np.array([[0, 5, 3], [0, 1, 2]], np.int64)  # row 0 decreases
    with pytest.raises(ValueError):
        multigpu.sample_sort_plan(bad)


@pytest.mark.parametrize("num_arrays,nshards", [(0, 3), (1, 4), (10, 3), (1000, 2), (4097, 8),
                                                (65536, 7)])
def test_shard_batch_plan_balances_keys(ns, num_arrays, nshards):
    from paper_2503_05934_b200 import multigpu
    offs, keys = ns.generate_batch(num_arrays, 11)
    ab = multigpu.shard_batch_plan(offs, nshards)
    assert ab[0] == 0 and ab[-1] == num_arrays and np.all(np.diff(ab) >= 0)
    total = int(offs[-1])
    for k in range(nshards):
        kk = int(offs[ab[k + 1]] - offs[ab[k]])
        # arrays stay whole: a shard misses its ideal share by < one array (<= 8 keys)
        assert abs(kk - total / nshards) <= 8 + 1e-9 or num_arrays < nshards
    shards = multigpu.shard_batch(offs, keys, nshards)
    assert sum(len(k) for _, k in shards) == len(keys)
    for o, k in shards:
        assert o[0] == 0 and o[-1] == len(k)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch_worker(rank, world, port, num_arrays, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    import paper_2503_05934_b200 as ns
    from paper_2503_05934_b200 import multigpu
    offs, keys = ns.generate_batch(num_arrays, 3)
    o, k = multigpu.shard_batch(offs, keys, world)[rank]  # this rank's arrays, rebased
    mine = O.sort_small_batch(np.ascontiguousarray(k), np.ascontiguousarray(o))
    parts = [None] * world
    dist.all_gather_object(parts, mine.tolist())
    # segmented batch: whole segments per rank
    seg_len, nseg = 100, 37
    full = O.generate_i32("random", seg_len * nseg, 4)
    s0, s1 = rank * nseg // world, (rank + 1) * nseg // world
    seg = O.segmented_quick_sort(full[s0 * seg_len:s1 * seg_len].copy(), seg_len)
    sparts = [None] * world
    dist.all_gather_object(sparts, seg.tolist())
    if rank == 0:
        q.put((parts, sparts))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shard_by_array_multi_process(ns, oracle, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, 5000, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts, sparts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    offs, keys = ns.generate_batch(5000, 3)
    got = np.array([x for part in parts for x in part], np.int32)
    assert np.array_equal(got, oracle.sort_small_batch(keys, offs))
    full = oracle.generate_i32("random", 3700, 4)
    sgot = np.array([x for part in sparts for x in part], np.int32)
    assert np.array_equal(sgot, oracle.segmented_quick_sort(full, 100))
