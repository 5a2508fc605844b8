"""GPU tests of the multi-GPU C ABI behind one host thread
(ns_sample_sort_multi_i32, ns_sort_small_batch_multi_i32,
ns_segmented_sort_multi_i32) on the one B200 of the test box: the NCCL
exchange over the devices present (one), the peer-memory exchange with up to
4 virtual ranks on device 0, and the shard-by-array batches — against numpy
and the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _shards(a, g, cuda):
    import torch
    n = len(a)
    return [torch.from_numpy(a[n * d // g:n * (d + 1) // g].copy()).to(cuda) for d in range(g)]


@pytest.mark.parametrize("g", [1, 2, 3, 4])
@pytest.mark.parametrize("kind", ["random", "sorted", "dups", "tiny"])
def test_sample_sort_multi_p2p_virtual_ranks(ns, cuda, oracle, g, kind):
    from paper_2503_05934_b200 import multigpu
    if kind == "random":
        a = oracle.generate_i32("random", 3_000_017, 8)
    elif kind == "sorted":
        a = oracle.generate_i32("sorted", 1_000_000, 8)
    elif kind == "dups":
        a = (oracle.generate_i32("random", 2_000_000, 8) % 5).astype(np.int32)
    else:
        a = np.array([5, 3, 9], np.int32)[: max(1, g - 1)]  # some shards empty
    outs = multigpu.sample_sort_multi(_shards(a, g, cuda), exchange="p2p")
    got = np.concatenate([o.cpu().numpy() for o in outs])
    assert np.array_equal(got, np.sort(a))


def test_sample_sort_multi_nccl(ns, cuda, oracle):
    import torch
    from paper_2503_05934_b200 import multigpu
    if not multigpu.nccl_available():
        pytest.skip("libnccl.so.2 not loadable")
    devs = list(range(torch.cuda.device_count()))
    a = oracle.generate_i32("random", 4_000_037, 2)
    with multigpu.NcclComms(devs) as comms:
        shards = [torch.from_numpy(x).to(f"cuda:{d}")
                  for d, x in zip(devs, np.array_split(a, len(devs)))]
        outs = multigpu.sample_sort_multi(shards, exchange="nccl", comms=comms)
    got = np.concatenate([o.cpu().numpy() for o in outs])
    assert np.array_equal(got, np.sort(a))


@pytest.mark.parametrize("g", [1, 3])
def test_sort_small_batch_multi_shards(ns, cuda, oracle, g):
    import torch
    from paper_2503_05934_b200 import multigpu
    offs, keys = ns.generate_batch(100_000, 6)
    parts = multigpu.shard_batch(offs, keys, g)
    kt = [torch.from_numpy(np.ascontiguousarray(k)).to(cuda) for _, k in parts]
    ot = [torch.from_numpy(np.ascontiguousarray(o).view(np.int32)).to(cuda) for o, _ in parts]
    assert multigpu.sort_small_batch_multi(kt, ot) == [0] * g
    got = np.concatenate([k.cpu().numpy() for k in kt])
    assert np.array_equal(got, oracle.sort_small_batch(keys, offs))


def test_segmented_sort_multi_shards(ns, cuda, oracle):
    import torch
    from paper_2503_05934_b200 import multigpu
    seg, nseg = 20000, 9
    a = oracle.generate_i32("random", seg * nseg, 1)
    kt = [torch.from_numpy(a[s0 * seg:s1 * seg].copy()).to(cuda)
          for s0, s1 in ((0, 4), (4, 9))]
    multigpu.segmented_sort_multi(kt, seg)
    got = np.concatenate([k.cpu().numpy() for k in kt])
    assert np.array_equal(got, np.sort(a.reshape(nseg, seg), axis=1).reshape(-1))
