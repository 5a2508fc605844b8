"""CPU tests of the oracle (test infrastructure) — pinned against the
reference's own golden vectors and against the reference compiled from
/root/reference (oracle/_ref) where that library exists."""
import hashlib
import itertools
import math

import numpy as np
import pytest

U64 = 2**64


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---- input generation: the reference's KATs (test_datagen.cpp) -------------

def test_splitmix64_published_vectors(oracle):
    """test_datagen.cpp:25-35."""
    import ctypes as C
    L = oracle.lib()
    for seed, want in ((0, [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]),
                       (42, [0xBDD732262FEB6E95, 0x28EFE333B266F103, 0x47526757130F9F52])):
        st = C.c_uint64(seed)
        got = [L.oracle_splitmix64_next(C.byref(st)) for _ in range(3)]
        assert got == want


def test_frozen_nearly_sorted_outputs(oracle):
    """test_datagen.cpp:79-91 (frozen specs) and 54-56, 64-69."""
    assert oracle.generate_i64("nearly_sorted", 10, 3, 0.001).tolist() == [0, 3, 2, 1, 4, 5, 6, 7, 8, 9]
    assert oracle.generate_i64("nearly_sorted", 10, 7, 0.25).tolist() == [0, 1, 2, 6, 7, 5, 3, 4, 8, 9]
    assert oracle.generate_i64("sorted", 5, 42).tolist() == [0, 1, 2, 3, 4]
    assert oracle.generate_i64("nearly_sorted", 100, 42, 0.0).tolist() == list(range(100))
    for seed in (1, 2, 3, 42):
        v = oracle.generate_i64("nearly_sorted", 100, seed, 0.01)
        assert not np.all(v[:-1] <= v[1:])


def test_swap_rule_restatement(oracle):
    """test_datagen.cpp:93-106: floor(p*n) swaps (min 1) of (next()%n, next()%n)."""
    import ctypes as C
    n, p = 200, 0.03
    expect = list(range(n))
    swaps = max(int(p * n), 1)
    st = C.c_uint64(77)
    L = oracle.lib()
    for _ in range(swaps):
        i = L.oracle_splitmix64_next(C.byref(st)) % n
        j = L.oracle_splitmix64_next(C.byref(st)) % n
        expect[i], expect[j] = expect[j], expect[i]
    assert oracle.generate_i64("nearly_sorted", n, 77, p).tolist() == expect


def test_perturbation_range_and_tiny_sizes(oracle):
    with pytest.raises(ValueError):
        oracle.generate_i64("nearly_sorted", 10, 1, -0.1)
    with pytest.raises(ValueError):
        oracle.generate_i32("nearly_sorted", 10, 1, 1.5)
    for d in ("random", "sorted", "nearly_sorted"):
        assert len(oracle.generate_i32(d, 0, 11, 0.5)) == 0
        assert len(oracle.generate_i32(d, 1, 11, 0.5)) == 1


def test_int32_stream_is_the_reference_stream_narrowed(oracle):
    """random int32 = top 31 bits of the reference's word."""
    w = oracle.generate_i64("random", 5000, 42).view(np.uint64)
    assert np.array_equal(oracle.generate_i32("random", 5000, 42), (w >> np.uint64(33)).astype(np.int32))
    for d in ("sorted", "nearly_sorted"):
        assert np.array_equal(oracle.generate_i32(d, 5000, 9), oracle.generate_i64(d, 5000, 9))


@pytest.mark.skipif("not __import__('oracle.oracle').oracle.ref_available()")
def test_generator_matches_reference_build(oracle):
    R = oracle.ref()
    for kind in range(3):
        for n, seed in ((0, 1), (1, 2), (1000, 42), (100000, 7)):
            want = np.empty(n, np.int64)
            assert R.ref_generate_i64(kind, n, seed, 0.01, want) == 0
            got = oracle.generate_i64(["random", "sorted", "nearly_sorted"][kind], n, seed)
            assert np.array_equal(got, want)


# ---- networks (test_networks.cpp / acceptance criteria 1-2) ----------------

def test_networks_zero_one_permutations_counts(oracle):
    counts = {2: 1, 3: 3, 4: 5, 5: 9, 6: 12, 7: 16, 8: 19}
    for w in range(2, 9):
        net = oracle.network(w)
        assert len(net) == counts[w]
        assert all(lo < hi < w for lo, hi in net)
        for bits in range(1 << w):
            v = [(bits >> i) & 1 for i in range(w)]
            for lo, hi in net:
                if v[hi] < v[lo]:
                    v[lo], v[hi] = v[hi], v[lo]
            assert v == sorted(v)
        for perm in itertools.permutations(range(1, w + 1)):
            a = np.array(perm, np.int32)
            oracle.lib().oracle_sort_small_i32(a, w)
            assert a.tolist() == list(range(1, w + 1))
    for bad in (-1, 0, 1, 9):
        with pytest.raises(ValueError):
            oracle.network(bad)


@pytest.mark.skipif("not __import__('oracle.oracle').oracle.ref_available()")
def test_network_sizes_match_reference(oracle):
    buf = np.zeros(64, np.uint8)
    for w in range(2, 9):
        assert oracle.ref().ref_network(w, buf, 32) == len(oracle.network(w))
    assert oracle.ref().ref_network(9, buf, 32) == -1


def test_duplicates_and_idempotence(oracle):
    for w in range(2, 9):
        v = np.array([(w - i) % 3 for i in range(w)], np.int32)
        oracle.lib().oracle_sort_small_i32(v, w)
        assert v.tolist() == sorted(v.tolist())
        oracle.lib().oracle_sort_small_i32(v, w)
        assert v.tolist() == sorted(v.tolist())


# ---- hybrid sorts ----------------------------------------------------------

def test_sorts_match_numpy(oracle):
    """acceptance.cpp:101-132 restated on the oracle (subset of seeds)."""
    for n in list(range(0, 65)) + [1000, 10000]:
        for d in ("random", "sorted", "nearly_sorted"):
            for seed in (0, 1, 42):
                a = oracle.generate_i32(d, n, seed)
                want = np.sort(a)
                for name, _, _ in oracle.REGISTRY:
                    assert np.array_equal(oracle.merge_sort(a, name), want)
                    assert np.array_equal(oracle.quick_sort(a, name), want)


def test_ternary_exhaustive_len5(oracle):
    """test_hybrid.cpp:283-304."""
    for length in range(0, 6):
        for code in itertools.product(range(3), repeat=length):
            a = np.array(code, np.int32)
            want = np.sort(a)
            for name, _, _ in oracle.REGISTRY:
                assert np.array_equal(oracle.merge_sort(a, name), want)
                assert np.array_equal(oracle.quick_sort(a, name), want)


def test_dispatch_counters(oracle):
    """test_hybrid.cpp:169-202 / acceptance.cpp:168-197."""
    a = oracle.generate_i32("random", 13, 5)
    out, st = oracle.merge_sort(a, "6To8", stats=True)
    assert sum(st.network_hits) == 2 and st.network_hits[7] == 1 and st.network_hits[6] == 1
    assert st.merges == 1
    _, st = oracle.merge_sort(oracle.generate_i32("random", 8, 6), "PowerOf2", stats=True)
    assert sum(st.network_hits) == 1 and st.network_hits[8] == 1 and st.merges == 0
    _, st = oracle.merge_sort(oracle.generate_i32("random", 10, 7), "6To8", stats=True)
    assert sum(st.network_hits) == 0
    _, st = oracle.quick_sort(oracle.generate_i32("random", 7, 8), "Odd", stats=True)
    assert sum(st.network_hits) == 1 and st.network_hits[7] == 1 and st.partitions == 0


@pytest.mark.skipif("not __import__('oracle.oracle').oracle.ref_available()")
def test_dispatch_counters_match_reference(oracle):
    R = oracle.ref()
    for name, mask, vs in oracle.REGISTRY:
        for n in (0, 1, 2, 7, 13, 100, 1000, 25000):
            a = oracle.generate_i32("random", n, 11 + n)
            for algo in ("merge", "quick"):
                out, st = (oracle.merge_sort if algo == "merge" else oracle.quick_sort)(a, name, stats=True)
                ref_out = a.copy()
                rs = np.zeros(12, np.uint64)
                (R.ref_merge_sort_i32 if algo == "merge" else R.ref_quick_sort_i32)(
                    ref_out, n, mask, vs, rs.ctypes.data)
                assert np.array_equal(out, ref_out)
                if n == 0:
                    continue  # run_variant's stats overload skips empty input
                assert list(st.network_hits) == rs[:9].tolist(), (name, algo, n)
                assert st.merges == rs[9] and st.partitions == rs[10]
                assert st.max_depth == rs[11]


def test_median_and_partition_contract(oracle):
    """test_hybrid.cpp:204-269."""
    L = oracle.lib()
    for v, want in (([3, 9, 5], 5), ([1, 1, 1], 1)):
        assert L.oracle_median_of_three_i32(np.array(v, np.int32), 0, 2) == want
    assert L.oracle_median_of_three_i32(np.array([9, 4], np.int32), 0, 1) == 9
    assert L.oracle_median_of_three_i32(np.array([6], np.int32), 0, 0) == 6
    rng = np.random.default_rng(21)
    for _ in range(60):
        n = int(rng.integers(2, 11))
        base = rng.integers(0, 8, n).astype(np.int32)
        for lo in range(n):
            for hi in range(lo + 1, n):
                for p in range(lo, hi + 1):
                    u = base.copy()
                    j = L.oracle_hoare_partition_i32(u, lo, hi, int(base[p]))
                    assert lo <= j < hi
                    assert np.all(u[lo:j + 1] <= base[p]) and np.all(u[j + 1:hi + 1] >= base[p])
                    assert np.array_equal(np.sort(u[lo:hi + 1]), np.sort(base[lo:hi + 1]))
                    assert np.array_equal(u[:lo], base[:lo]) and np.array_equal(u[hi + 1:], base[hi + 1:])


def _hoare_closed_form(a, lo, hi, p):
    """The rank form of hoare_partition that qs_trace.cu computes in
    parallel: swap the pairs (L_k, R_k) while L_k < R_k (L ascending
    positions of keys >= p, R descending positions of keys <= p, both on the
    input), return max(R_{S+1}, L_S) with the j == high fix-up."""
    seg = a[lo:hi + 1]
    L = lo + np.flatnonzero(seg >= p)
    R = (lo + np.flatnonzero(seg <= p))[::-1]
    m = min(len(L), len(R))
    ok = L[:m] < R[:m]
    S = int(np.argmin(ok)) if not ok.all() else m
    a[L[:S]], a[R[:S]] = a[R[:S]].copy(), a[L[:S]].copy()
    j = max(int(R[S]) if S < len(R) else -1, int(L[S - 1]) if S else -1)
    return j if j < hi else hi - 1


def test_hoare_closed_form(oracle):
    """The closed form the GPU partition uses gives the reference loop's
    cells and split (hybrid.hpp:121-133) on every tested input."""
    L = oracle.lib()
    rng = np.random.default_rng(8)
    for _ in range(3000):
        n = int(rng.integers(2, 60))
        a = rng.integers(0, int(rng.choice([2, 3, 5, 1000])), n).astype(np.int32)
        lo = int(rng.integers(0, n - 1))
        hi = int(rng.integers(lo + 1, n))
        p = int(a[rng.integers(lo, hi + 1)])
        u, v = a.copy(), a.copy()
        j = L.oracle_hoare_partition_i32(u, lo, hi, p)
        assert _hoare_closed_form(v, lo, hi, p) == j
        assert np.array_equal(u, v)


def test_quick_sort_depth_bound_sorted(oracle):
    """test_hybrid.cpp:271-281."""
    for name in ("Classic", "3To5"):
        _, st = oracle.quick_sort(np.arange(10000, dtype=np.int32), name, stats=True)
        assert st.max_depth <= 4 * math.log2(10000) + 16


# ---- golden fixtures (outputs of the reference itself) ---------------------

def test_golden_small_cases_inline(oracle, golden):
    for c in golden["cases"]:
        if "input" not in c:
            continue
        a = np.array(c["input"], np.int32)
        assert np.array_equal(oracle.generate_i32(c["dist"], c["n"], c["seed"]), a)
        fn = oracle.merge_sort if c["algo"] == "merge" else oracle.quick_sort
        assert fn(a, c["config"]).tolist() == c["output"]


def test_golden_digests_up_to_1m(oracle, golden):
    for c in golden["cases"]:
        if c["n"] > 1_000_000:
            continue
        a = oracle.generate_i32(c["dist"], c["n"], c["seed"])
        assert sha(a) == c["input_sha256"]
        fn = oracle.merge_sort if c["algo"] == "merge" else oracle.quick_sort
        assert sha(fn(a, c["config"])) == c["output_sha256"], (c["algo"], c["config"], c["n"])


def test_golden_small_batch(oracle, golden):
    sb = golden["small_batch"]
    offs, keys = oracle.generate_batch_i32(sb["num_arrays"], sb["seed"])
    assert offs.tolist() == sb["offsets"] and keys.tolist() == sb["input"]
    assert oracle.sort_small_batch(keys, offs).tolist() == sb["output"]
    lens = np.diff(offs)
    assert lens.min() >= 3 and lens.max() <= 8


def test_golden_kat(golden):
    assert golden["kat"]["splitmix64"]["0"][0] == hex(0xE220A8397B1DCDAF)
    assert golden["kat"]["splitmix64"]["42"][0] == hex(0xBDD732262FEB6E95)


def test_multiset_digest_is_order_independent(oracle):
    a = oracle.generate_i32("random", 10000, 3)
    assert oracle.multiset_digest(a) == oracle.multiset_digest(np.sort(a))
    b = a.copy()
    b[0] ^= 1
    assert oracle.multiset_digest(a) != oracle.multiset_digest(b)


# ---- int64 keys: the reference's own benchmark type -

def test_golden_i64_reference_outputs(oracle, golden):
    """The oracle's int64 instantiation reproduces the reference's int64 sorts
    of the reference's own generate() stream (full 64-bit values)."""
    for c in golden["cases_i64"]:
        if c["n"] > 1_000_000:
            continue
        a = oracle.generate_i64(c["dist"], c["n"], c["seed"])
        assert sha(a) == c["input_sha256"], c
        if "input" in c:
            assert [str(x) for x in a.tolist()] == c["input"]
        fn = oracle.merge_sort if c["algo"] == "merge" else oracle.quick_sort
        out = fn(a, c["config"])
        assert out.dtype == np.int64
        assert sha(out) == c["output_sha256"], (c["algo"], c["config"], c["dist"], c["n"])
        if "output" in c:
            assert [str(x) for x in out.tolist()] == c["output"]


@pytest.mark.skipif("not __import__('oracle.oracle').oracle.ref_available()")
def test_dispatch_counters_match_reference_i64(oracle):
    R = oracle.ref()
    for name, mask, vs in oracle.REGISTRY:
        for n in (1, 2, 7, 13, 1000, 25000):
            a = oracle.generate_i64("random", n, 17 + n)
            for algo in ("merge", "quick"):
                out, st = (oracle.merge_sort if algo == "merge" else oracle.quick_sort)(
                    a, name, stats=True)
                ref_out = a.copy()
                rs = np.zeros(12, np.uint64)
                (R.ref_merge_sort_i64 if algo == "merge" else R.ref_quick_sort_i64)(
                    ref_out, n, mask, vs, rs.ctypes.data)
                assert np.array_equal(out, ref_out)
                assert list(st.network_hits) == rs[:9].tolist(), (name, algo, n)
                assert st.merges == rs[9] and st.partitions == rs[10]
                assert st.max_depth == rs[11]


def test_i64_extremes_and_digest(oracle):
    ext = np.array([2**63 - 1, -2**63, 0, -1, 1, 2**63 - 1, -2**63, 2**31, -2**31 - 1], np.int64)
    for fn in (oracle.merge_sort, oracle.quick_sort):
        assert np.array_equal(fn(ext, "6To8"), np.sort(ext))
    a = oracle.generate_i64("random", 5000, 9)
    assert oracle.multiset_digest(a) == oracle.multiset_digest(np.sort(a))
    # int64 keys that agree in their low 32 bits still digest differently
    b = a.copy()
    b[0] ^= 1 << 40
    assert oracle.multiset_digest(a) != oracle.multiset_digest(b)


def test_stable_pairs_restatement(oracle):
    """Classical merge is stable (test_hybrid.cpp:119-150 restated: equal keys
    keep their tags' input order); the pairs oracle equals a stable argsort."""
    rng = np.random.default_rng(8)
    for n in (0, 1, 2, 3, 17, 1000, 65537):
        k = rng.integers(-3, 3, n).astype(np.int32)
        tags = np.arange(n, dtype=np.uint32)
        sk, sv = oracle.stable_sort_pairs(k, tags)
        p = np.argsort(k, kind="stable")
        assert np.array_equal(sk, k[p]) and np.array_equal(sv, tags[p])
        for key in np.unique(k):
            t = sv[sk == key]
            assert np.all(t[:-1] < t[1:])  # input order kept among equals
