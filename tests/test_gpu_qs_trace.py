"""GPU parity of the traced quick sort (qs_trace.cu): the reference's own
recursion — median_of_three + hoare_partition at every node of
quick_sort_rec (hybrid.hpp:105-150) — executed on the device.  Checked
against the CPU oracle (pinned to the reference's counters by
tests/test_oracle.py::test_dispatch_counters_match_reference): the same
arrangement after every single partition, the same split, and the same
DispatchStats (network hits by width, partitions, max depth) for whole sorts
of every config, distribution and size class (one-CTA segments, grid-wide
levels, both)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev(a, cuda):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(cuda)


def _oracle_partition(oracle, a, lo, hi, p):
    u = a.copy()
    fn = oracle.lib().oracle_hoare_partition_i64 if a.dtype == np.int64 else \
        oracle.lib().oracle_hoare_partition_i32
    j = fn(u, lo, hi, int(p))
    return u, j


def test_hoare_partition_small_exhaustive(ns, cuda, oracle):
    """Every (low, high, pivot cell) of small arrays with many duplicates
    (the contract test of test_hybrid.cpp:225-269, here against the
    reference's exact cells)."""
    rng = np.random.default_rng(5)
    for _ in range(12):
        n = int(rng.integers(2, 9))
        base = rng.integers(0, 4, n).astype(np.int32)
        for lo in range(n):
            for hi in range(lo + 1, n):
                for p in range(lo, hi + 1):
                    want, wj = _oracle_partition(oracle, base, lo, hi, base[p])
                    t = _dev(base, cuda)
                    j = ns.hoare_partition(t, lo, hi, int(base[p]))
                    assert j == wj, (base, lo, hi, p)
                    assert np.array_equal(t.cpu().numpy(), want), (base, lo, hi, p)


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_hoare_partition_large_ranges(ns, cuda, oracle, dtype):
    """Ranges of 2 .. 3M keys (one chunk, many chunks), random / few distinct
    values / sorted / reversed, pivots from the range: identical cells and
    split; the keys outside [low, high] untouched."""
    rng = np.random.default_rng(11)
    cases = [(2, 1 << 20), (33, 3), (4097, 1 << 30), (8193, 5), (100_003, 1 << 31),
             (1 << 20, 17), (3_000_001, 1 << 31)]
    for n, vr in cases:
        for dist in ("random", "sorted", "reversed"):
            a = rng.integers(-vr, vr, n).astype(dtype)
            if dist == "sorted":
                a.sort()
            elif dist == "reversed":
                a = np.sort(a)[::-1].copy()
            lo = int(rng.integers(0, max(1, n // 7)))
            hi = n - 1 - int(rng.integers(0, max(1, n // 9)))
            if hi <= lo:
                lo, hi = 0, n - 1
            p = a[int(rng.integers(lo, hi + 1))]
            want, wj = _oracle_partition(oracle, a, lo, hi, p)
            t = _dev(a, cuda)
            j = ns.hoare_partition(t, lo, hi, int(p))
            assert j == wj, (n, vr, dist)
            assert np.array_equal(t.cpu().numpy(), want), (n, vr, dist)


def test_hoare_partition_pivot_outside_keys_rejected(ns, cuda):
    a = np.arange(100, dtype=np.int32)
    t = _dev(a, cuda)
    with pytest.raises(ValueError):
        ns.hoare_partition(t, 0, 99, 1000)
    with pytest.raises(ValueError):
        ns.hoare_partition(t, 0, 99, -5)
    assert np.array_equal(t.cpu().numpy(), a)
    with pytest.raises(ValueError):
        ns.hoare_partition(t, 5, 5, 5)  # low < high required


def test_median_of_three_device_and_host(ns, cuda, oracle):
    """median_of_three (hybrid.hpp:105-114) in place, test_hybrid.cpp:204-223."""
    L = oracle.lib()
    rng = np.random.default_rng(2)
    for _ in range(40):
        n = int(rng.integers(1, 12))
        a = rng.integers(0, 5, n).astype(np.int32)
        lo = int(rng.integers(0, n))
        hi = int(rng.integers(lo, n))
        want = a.copy()
        wp = L.oracle_median_of_three_i32(want, lo, hi)
        t = _dev(a, cuda)
        assert ns.median_of_three(t, lo, hi) == wp
        assert np.array_equal(t.cpu().numpy(), want)
        h = a.copy()
        assert ns.median_of_three(h, lo, hi) == wp
        assert np.array_equal(h, want)
        h64 = a.astype(np.int64)
        assert ns.median_of_three(h64, lo, hi) == wp


def _stats_equal(st, ost):
    return (list(st.network_hits) == list(ost.network_hits) and st.merges == ost.merges
            and st.partitions == ost.partitions and st.max_depth == ost.max_depth)


@pytest.mark.parametrize("cfg", ["Classic", "PowerOf2", "Even", "Odd", "3", "3To4", "3To5",
                                 "3To8", "6To8", "VarSort3", "VarSort4", "VarSort5"])
def test_traced_stats_every_config(ns, cuda, oracle, cfg):
    """run_variant(quick sort, a, stats) for all 12 Table-3 configs at the
    one-CTA sizes and across the grid-wide threshold (8192 keys)."""
    for n in (1, 2, 3, 7, 9, 13, 100, 1000, 8192, 8193, 25_000, 100_000):
        a = oracle.generate_i32("random", n, 11 + n)
        want, ost = oracle.quick_sort(a, cfg, stats=True)
        t = _dev(a, cuda)
        st = ns.DispatchStats()
        ns.run_variant(ns.SortVariant(ns.Algorithm.quick_sort, ns.find_config(cfg)), t, st)
        assert np.array_equal(t.cpu().numpy(), want), (cfg, n)
        assert _stats_equal(st, ost), (cfg, n, st, ost)


@pytest.mark.parametrize("dist", ["random", "sorted", "nearly_sorted"])
def test_traced_stats_c4_sizes(ns, cuda, oracle, dist):
    """3To5 at the C4 sizes (10K, 1M, 16M; SURVEY A.2 quotes depth 23-46),
    device tensors."""
    for n in (10_000, 1_000_000, 1 << 24):
        a = oracle.generate_i32(dist, n, 42)
        want, ost = oracle.quick_sort(a, "3To5", stats=True)
        t = _dev(a, cuda)
        st = ns.quick_sort_traced(t, 0, n - 1, ns.find_config("3To5"))
        assert _stats_equal(st, ost), (dist, n, st, ost)
        assert np.array_equal(t.cpu().numpy(), want), (dist, n)


def test_traced_adversarial_shapes(ns, cuda, oracle):
    """All equal keys, two values, organ pipe, sawtooth, reversed: shapes
    that make Hoare's scans stop on every key or make the tree deep."""
    n = 200_000
    i = np.arange(n)
    shapes = {
        "equal": np.full(n, 7, np.int32),
        "two": (i % 2).astype(np.int32),
        "organ": np.minimum(i, n - i).astype(np.int32),
        "saw": (i % 1000).astype(np.int32),
        "reversed": (n - i).astype(np.int32),
    }
    for name, a in shapes.items():
        for cfg in ("Classic", "3To5", "6To8"):
            want, ost = oracle.quick_sort(a, cfg, stats=True)
            t = _dev(a, cuda)
            st = ns.quick_sort_traced(t, 0, n - 1, ns.find_config(cfg))
            assert _stats_equal(st, ost), (name, cfg, st, ost)
            assert np.array_equal(t.cpu().numpy(), want), (name, cfg)


def test_traced_int64_and_ranges(ns, cuda, oracle):
    """int64 keys (the reference's own benchmark type) and a sub-range
    [low, high]: the counters of optimized_quick_sort(a, low, high, cfg,
    stats) and the keys outside untouched."""
    R = oracle.ref() if oracle.ref_available() else None
    for n in (5, 4000, 70_000, 600_000):
        a = oracle.generate_i64("random", n, 3 + n)
        want, ost = oracle.quick_sort(a, "3To8", stats=True)
        t = _dev(a, cuda)
        st = ns.quick_sort_traced(t, 0, n - 1, ns.find_config("3To8"))
        assert _stats_equal(st, ost) and np.array_equal(t.cpu().numpy(), want), n
        if R is not None:
            rs = np.zeros(12, np.uint64)
            ref_out = a.copy()
            mask, vs = next((m, v) for nm, m, v in oracle.REGISTRY if nm == "3To8")
            R.ref_quick_sort_i64(ref_out, n, mask, vs, rs.ctypes.data)
            assert st.partitions == rs[10] and st.max_depth == rs[11]
    a = oracle.generate_i32("random", 50_000, 9)
    lo, hi = 1234, 40_000
    sub, ost = oracle.quick_sort(a[lo:hi + 1].copy(), "6To8", stats=True)
    t = _dev(a, cuda)
    st = ns.DispatchStats()
    ns.optimized_quick_sort(t, lo, hi, ns.find_config("6To8"), st)
    got = t.cpu().numpy()
    assert _stats_equal(st, ost)
    assert np.array_equal(got[lo:hi + 1], sub)
    assert np.array_equal(got[:lo], a[:lo]) and np.array_equal(got[hi + 1:], a[hi + 1:])


def test_traced_host_arrays(ns, cuda, oracle):
    """The host-span forms (the reference's call shape): traced sort,
    partition and run_variant on numpy arrays; counters accumulate across
    calls like the reference's Stats object."""
    a = oracle.generate_i32("nearly_sorted", 300_000, 4)
    want, ost = oracle.quick_sort(a, "3To5", stats=True)
    h = a.copy()
    st = ns.DispatchStats()
    ns.run_variant(ns.SortVariant(ns.Algorithm.quick_sort, ns.find_config("3To5")), h, st)
    assert np.array_equal(h, want) and _stats_equal(st, ost)
    h2 = a.copy()
    ns.run_variant(ns.SortVariant(ns.Algorithm.quick_sort, ns.find_config("3To5")), h2, st)
    assert st.partitions == 2 * ost.partitions
    assert st.network_hits == [2 * x for x in ost.network_hits]
    b = oracle.generate_i64("random", 20_000, 8)
    u, wj = _oracle_partition(oracle, b, 10, 19_000, b[500])
    hb = b.copy()
    assert ns.hoare_partition(hb, 10, 19_000, int(b[500])) == wj
    assert np.array_equal(hb, u)
    st0 = ns.DispatchStats()
    ns.run_variant(ns.SortVariant(ns.Algorithm.quick_sort, ns.find_config("3To5")),
                   np.zeros(0, np.int32), st0)
    assert st0.partitions == 0 and st0.max_depth == 0


def test_traced_c_abi_temp_and_args(ns, cuda):
    import torch
    L = ns.lib()
    t = torch.arange(20_000, dtype=torch.int32, device=cuda)
    out = (C.c_uint64 * 12)()
    tb = L.ns_quick_sort_traced_temp_bytes(20_000)
    small = torch.empty(16, dtype=torch.uint8, device=cuda)
    rc = L.ns_quick_sort_traced_i32(t.data_ptr(), 20_000, 0, 5, C.cast(out, C.c_void_p),
                                    small.data_ptr(), 16, None)
    assert rc == 4  # NS_ERR_TEMP
    tmp = torch.empty(tb, dtype=torch.uint8, device=cuda)
    assert L.ns_quick_sort_traced_i32(None, 10, 0, 5, C.cast(out, C.c_void_p), tmp.data_ptr(),
                                      tb, None) == 1
    assert L.ns_quick_sort_traced_i32(t.data_ptr(), 20_000, 0, 5, None, tmp.data_ptr(), tb,
                                      None) == 1
    assert L.ns_quick_sort_traced_i32(t.data_ptr(), 20_000, 0, 5, C.cast(out, C.c_void_p),
                                      tmp.data_ptr(), tb, None) == 0
    torch.cuda.synchronize()
    assert torch.equal(t, torch.arange(20_000, dtype=torch.int32, device=cuda))
    assert out[10] > 0 and out[11] > 0
