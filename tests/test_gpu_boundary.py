"""GPU tests of boundary behaviour added in round 2: the asynchronous batch
call (status word, nothing touched on a bad length anywhere in the batch),
the Python API's per-stream scratch under concurrent streams and host
threads, and the host-array entry points' zero-copy small path at every
single-CTA tile size (including the exact tile sizes whose final store is a
bulk copy into mapped host memory)."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_batch_async_status_and_untouched_on_bad_length(ns, cuda, oracle):
    import torch
    from paper_2503_05934_b200 import _lib
    offs, keys = ns.generate_batch(5000, 9)  # 5 CTAs of 1024 arrays
    k = torch.from_numpy(keys).to(cuda)
    o = torch.from_numpy(offs.view(np.int32)).to(cuda)
    st = torch.full((1,), 7, dtype=torch.int32, device=cuda)
    ns.sort_small_batch(k, o, status=st)
    assert int(st.item()) == 0
    assert np.array_equal(k.cpu().numpy(), oracle.sort_small_batch(keys, offs))
    # a 9-key array in the SECOND CTA's range: no CTA may touch its keys
    bad = offs.astype(np.int64).copy()
    bad[1501:] += 9 - (bad[1501] - bad[1500])  # array 1500 now has 9 keys
    kb = np.concatenate([keys, np.arange(int(bad[-1]) - len(keys), dtype=np.int32)])
    k2 = torch.from_numpy(kb).to(cuda)
    o2 = torch.from_numpy(bad.astype(np.uint32).view(np.int32)).to(cuda)
    before = k2.clone()
    ns.sort_small_batch(k2, o2, status=st)
    assert int(st.item()) == _lib.NS_ERR_INVALID
    assert torch.equal(k2, before)
    with pytest.raises(ValueError):
        ns.sort_small_batch(k2, o2)
    assert torch.equal(k2, before)


def test_batch_async_is_graph_capturable(ns, cuda, oracle):
    import torch
    offs, keys = ns.generate_batch(20000, 2)
    src = torch.from_numpy(keys).to(cuda)
    o = torch.from_numpy(offs.view(np.int32)).to(cuda)
    w = src.clone()
    st = torch.ones(1, dtype=torch.int32, device=cuda)
    ns.sort_small_batch(w, o, status=st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        w.copy_(src)
        ns.sort_small_batch(w, o, status=st)
    w.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    assert np.array_equal(w.cpu().numpy(), oracle.sort_small_batch(keys, offs))


def test_python_api_two_streams_and_threads(ns, cuda, oracle):
    """Sorts issued on two torch streams at once, and from two host threads
    on one stream, each through the Python API with its cached scratch."""
    import torch
    a = oracle.generate_i32("random", 3_000_000, 1)
    b = oracle.generate_i32("random", 2_000_003, 2)
    ta, tb = torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    cfg = ns.find_config("6To8")
    for _ in range(3):
        wa, wb = ta.clone(), tb.clone()
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            ns.optimized_merge_sort(wa, cfg)
            ns.optimized_quick_sort(wa, cfg)
        with torch.cuda.stream(s2):
            ns.optimized_quick_sort(wb, cfg)
            ns.optimized_merge_sort(wb, cfg)
        torch.cuda.synchronize()
        assert np.array_equal(wa.cpu().numpy(), np.sort(a))
        assert np.array_equal(wb.cpu().numpy(), np.sort(b))
    outs = {}

    def work(name, arr):
        t = torch.from_numpy(arr).to(cuda)
        for _ in range(5):
            ns.optimized_merge_sort(t, cfg)
        torch.cuda.current_stream().synchronize()
        outs[name] = t.cpu().numpy()

    th = [threading.Thread(target=work, args=(i, x)) for i, x in enumerate((a, b, a[::-1].copy()))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert np.array_equal(outs[0], np.sort(a)) and np.array_equal(outs[1], np.sort(b))
    assert np.array_equal(outs[2], np.sort(a))


@pytest.mark.parametrize("n", [2, 31, 512, 513, 2048, 4096, 8192, 10_000, 16383, 16384])
@pytest.mark.parametrize("algo", ["merge", "quick"])
def test_host_small_path_zero_copy(ns, oracle, n, algo):
    a = oracle.generate_i32("random", n, n)
    h = a.copy()
    (ns.optimized_merge_sort if algo == "merge" else ns.optimized_quick_sort)(
        h, ns.find_config("3To5"))
    assert np.array_equal(h, np.sort(a))
    h64 = oracle.generate_i64("random", n, 3)
    w = h64.copy()
    ns.optimized_merge_sort(w, ns.find_config("6To8"))
    assert np.array_equal(w, np.sort(h64))


@pytest.mark.parametrize("n", [1, 5000, 16384, 300_001, 3_000_000, 9_000_001])
def test_sort_host_async_two_streams(ns, cuda, oracle, n):
    """ns_*_sort_host_async_i32: several sorts in flight on two streams, pinned
    and pageable buffers, out-of-place and in place, both algorithms."""
    import torch
    a = oracle.generate_i32("random", n, 77)
    want = np.sort(a)
    src = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy()
    np.copyto(src, a)
    outs = [torch.empty(n, dtype=torch.int32, pin_memory=True).numpy() for _ in range(3)]
    sts = [torch.cuda.Stream(), torch.cuda.Stream()]
    algos = [ns.Algorithm.merge_sort, ns.Algorithm.quick_sort, ns.Algorithm.merge_sort]
    cfgs = [ns.find_config("6To8"), ns.find_config("3To5"), ns.find_config("PowerOf2")]
    for k in range(3):
        ns.sort_host_async(src, outs[k], cfgs[k], algos[k], stream=sts[k % 2])
    torch.cuda.synchronize()
    for o in outs:
        assert np.array_equal(o, want)
    assert np.array_equal(src, a)  # the input is only read
    inplace = a.copy()  # pageable, in place
    ns.sort_host_async(inplace, inplace, cfgs[0], stream=sts[0])
    sts[0].synchronize()
    assert np.array_equal(inplace, want)
    ns.release_scratch()
