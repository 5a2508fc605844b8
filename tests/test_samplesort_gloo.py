"""Multi-process sample sort (BASELINE config 5) on CPU: world_size 2 (and 3)
over gloo, exercising the exchange logic of paper_2503_05934_b200/samplesort.py
with the per-rank steps injected from the oracle (test-only ops; the product
uses DeviceOps, the sm_100a library)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class OracleOps:
    """CPU stand-ins for DeviceOps with identical contracts."""

    def __init__(self):
        from oracle import oracle as O
        self.O = O

    def local_sort(self, keys):
        keys.copy_(torch.from_numpy(self.O.merge_sort(keys.numpy(), "6To8")))

    def samples(self, sorted_keys, s):
        n = sorted_keys.numel()
        if n == 0:
            return torch.full((s,), 2**31 - 1, dtype=torch.int32)
        idx = [(k + 1) * n // (s + 1) for k in range(s)]
        return sorted_keys[idx].clone()

    def splitters(self, all_samples, g):
        srt = torch.from_numpy(self.O.merge_sort(all_samples.numpy(), "6To8"))
        s = srt.numel()
        return srt[[(k + 1) * s // g for k in range(g - 1)]].clone()

    def bounds(self, sorted_keys, spl, g):
        a = sorted_keys.numpy()
        b = [0] + [int(np.searchsorted(a, int(x), side="left")) for x in spl.tolist()] + [len(a)]
        return torch.tensor(b, dtype=torch.int64)

    # pull exchange: "peer memory" is simulated by gathering every shard (the
    # metadata path — bounds all-gather, run assembly, pairing, barrier — is the
    # product's own code in samplesort.sample_sort)
    def open_peer_runs(self, shard, bounds_all, group=None):
        me, g = dist.get_rank(group), dist.get_world_size(group)
        shards = [None] * g
        dist.all_gather_object(shards, shard.numpy(), group=group)
        return [(shards[p][bounds_all[p][me]:bounds_all[p][me + 1]], bounds_all[p][me + 1] - bounds_all[p][me])
                for p in range(g)]

    def merge_pull(self, runs, device):
        pairs = [(runs[i], runs[i + 1] if i + 1 < len(runs) else (np.empty(0, np.int32), 0))
                 for i in range(0, len(runs), 2)]
        parts = []
        for (a, _), (b, _) in pairs:
            cat = np.concatenate([a, b]).astype(np.int32)
            if len(a) and len(b):
                self.O.lib().oracle_merge_i32(cat, 0, len(a) - 1, len(cat) - 1)
            parts.append(cat)
        out = torch.from_numpy(np.concatenate(parts).astype(np.int32)) if parts else torch.empty(0, dtype=torch.int32)
        if len(pairs) > 1:
            offs = [0]
            for p_ in parts:
                offs.append(offs[-1] + len(p_))
            self.merge_runs(out, offs)
        return out

    def close_peers(self):
        pass

    def merge_runs(self, keys, offs):
        out = keys.numpy().copy()
        runs = [out[offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]
        for r in runs:
            assert np.all(r[:-1] <= r[1:])
        merged = runs[0] if runs else out[:0]
        for r in runs[1:]:
            cat = np.concatenate([merged, r]).astype(np.int32)
            self.O.lib().oracle_merge_i32(cat, 0, len(merged) - 1, len(cat) - 1) if len(merged) and len(r) else None
            merged = cat
        keys.copy_(torch.from_numpy(np.ascontiguousarray(merged, np.int32)))


class FailingPeerOps(OracleOps):
    """Rank 1 cannot map its peers: every rank must see P2PUnavailable (and
    can then fall back to the NCCL exchange consistently)."""

    def open_peer_runs(self, shard, bounds_all, group=None):
        # like DeviceOps: the handle exchange (a collective) happens first,
        # mapping the peers (local, may fail) after it
        runs = super().open_peer_runs(shard, bounds_all, group)
        if dist.get_rank(group) == 1:
            raise RuntimeError("no peer access")
        return runs


def _fallback_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2503_05934_b200 import samplesort
    full = O.generate_i32("random", 9000, 5)
    m = 9000 // world
    shard = torch.from_numpy(full[rank * m:(rank + 1) * m].copy())
    raised = False
    try:
        samplesort.sample_sort(shard.clone(), ops=FailingPeerOps(), exchange="p2p")
    except samplesort.P2PUnavailable:
        raised = True
    out = samplesort.sample_sort(shard.clone(), ops=OracleOps(), exchange="nccl")
    parts = [None] * world
    dist.all_gather_object(parts, (raised, out.numpy().tolist()))
    if rank == 0:
        q.put(parts)
    dist.barrier()
    dist.destroy_process_group()


def test_p2p_failure_is_consistent_across_ranks(oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fallback_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(raised for raised, _ in parts)
    result = np.array([x for _, part in parts for x in part], np.int32)
    assert np.array_equal(result, np.sort(oracle.generate_i32("random", 9000, 5)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, dist_kind, q, exchange="nccl"):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2503_05934_b200 import samplesort
    full = O.generate_i32(dist_kind, n, 42)
    m = n // world
    lo = rank * m
    hi = n if rank == world - 1 else lo + m
    shard = torch.from_numpy(full[lo:hi].copy())
    out = samplesort.sample_sort(shard, ops=OracleOps(), exchange=exchange)
    parts = [None] * world
    dist.all_gather_object(parts, out.numpy().tolist())
    if rank == 0:
        q.put(parts)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,dist_kind,exchange", [
    (2, 20000, "random", "nccl"), (2, 5000, "sorted", "nccl"), (3, 30001, "random", "nccl"),
    (2, 3, "random", "nccl"), (2, 20000, "random", "p2p"), (3, 30001, "nearly_sorted", "p2p"),
    (4, 40000, "random", "p2p")])
def test_sample_sort_multi_process(oracle, world, n, dist_kind, exchange):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, dist_kind, q, exchange))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    result = np.array([x for part in parts for x in part], np.int32)
    full = oracle.generate_i32(dist_kind, n, 42)
    # globally sorted, a permutation of the input, equal to the oracle's sort
    assert np.array_equal(result, oracle.merge_sort(full, "6To8"))
    # every rank's slice is sorted and the ranks are in order
    for a, b in zip(parts, parts[1:]):
        if a and b:
            assert a[-1] <= b[0]
