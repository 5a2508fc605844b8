"""GPU parity for int64 keys: the reference's own
benchmark type.  Inputs are the reference's generate() stream (full 64-bit
values, datagen.cpp:18-50); outputs are checked bit-exactly against the
reference's int64 sorts frozen in tests/golden/golden.json["cases_i64"] and
against the oracle's int64 instantiation."""
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SIZES = [0, 1, 2, 3, 5, 8, 9, 31, 33, 100, 255, 257, 1000, 4095, 4096, 4097, 8191, 8192, 8193,
         16383, 16384, 16385, 20000, 65537, 100000, 262145, 1000000]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def to_dev(a, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.int64)).to(dev)


def run(ns, algo, t, cfg_name):
    fn = ns.optimized_merge_sort if algo == "merge" else ns.optimized_quick_sort
    fn(t, ns.find_config(cfg_name))
    return t.cpu().numpy()


def test_golden_i64_reference_outputs(ns, cuda, oracle, golden):
    for c in golden["cases_i64"]:
        a = oracle.generate_i64(c["dist"], c["n"], c["seed"])
        assert sha(a) == c["input_sha256"], c
        got = run(ns, c["algo"], to_dev(a, cuda), c["config"])
        assert got.dtype == np.int64
        assert sha(got) == c["output_sha256"], (c["algo"], c["config"], c["dist"], c["n"])


@pytest.mark.parametrize("algo", ["merge", "quick"])
@pytest.mark.parametrize("dist", ["random", "sorted", "nearly_sorted"])
def test_i64_sizes_match_oracle(ns, cuda, oracle, algo, dist):
    cfg = "6To8" if algo == "merge" else "3To5"
    for n in SIZES:
        a = oracle.generate_i64(dist, n, 77 + n)
        want = (oracle.merge_sort if algo == "merge" else oracle.quick_sort)(a, cfg)
        assert np.array_equal(run(ns, algo, to_dev(a, cuda), cfg), want), (algo, dist, n)


@pytest.mark.parametrize("cfg_name", ["Classic", "PowerOf2", "Even", "Odd", "3", "3To4", "3To5",
                                      "3To8", "6To8", "VarSort3", "VarSort4", "VarSort5"])
def test_i64_every_config(ns, cuda, oracle, cfg_name):
    for n in (2, 7, 33, 1000, 9000, 40000):
        a = oracle.generate_i64("random", n, 900 + n)
        for algo in ("merge", "quick"):
            assert np.array_equal(run(ns, algo, to_dev(a, cuda), cfg_name), np.sort(a)), \
                (algo, cfg_name, n)


def test_i64_extremes_duplicates_and_sentinel_collisions(ns, cuda):
    """INT64_MAX is the kernels' +inf sentinel / tile pad: real keys equal to
    it, INT64_MIN, and heavy duplicates must all survive."""
    rng = np.random.default_rng(5)
    lo, hi = np.iinfo(np.int64).min, np.iinfo(np.int64).max
    cases = [
        np.full(30000, hi, np.int64),
        np.full(30000, lo, np.int64),
        rng.choice(np.array([lo, hi, 0, -1, 1], np.int64), 200000),
        rng.integers(-3, 3, 300001).astype(np.int64),
        np.concatenate([np.full(50000, hi, np.int64), rng.integers(lo, hi, 70000, dtype=np.int64)]),
        (np.arange(123457, dtype=np.int64) << 32)[::-1].copy(),  # differ only in the high word
    ]
    for a in cases:
        for algo in ("merge", "quick"):
            assert np.array_equal(run(ns, algo, to_dev(a, cuda), "6To8"), np.sort(a)), \
                (algo, a.size)


def test_i64_range_sort_and_host_arrays(ns, cuda, oracle):
    a = oracle.generate_i64("random", 50000, 3)
    t = to_dev(a, cuda)
    ns.optimized_merge_sort(t, 1000, 40999, ns.find_config("6To8"))
    got = t.cpu().numpy()
    assert np.array_equal(got[:1000], a[:1000]) and np.array_equal(got[41000:], a[41000:])
    assert np.array_equal(got[1000:41000], np.sort(a[1000:41000]))
    # host numpy arrays (the reference's span call shape); 5M keys takes the
    # chunked upload path of the host entry point
    for n in (1000, 300000, 5_000_000):
        h = oracle.generate_i64("random", n, 123 + n)
        want = np.sort(h)
        m, q = h.copy(), h.copy()
        ns.optimized_merge_sort(m, ns.find_config("6To8"))
        ns.optimized_quick_sort(q, ns.find_config("3To5"))
        assert np.array_equal(m, want) and np.array_equal(q, want), n


def test_i64_checking_helpers_match_oracle(ns, cuda, oracle):
    a = oracle.generate_i64("random", 1 << 20, 8)
    t = to_dev(a, cuda)
    assert ns.multiset_digest(t) == oracle.multiset_digest(a)
    assert ns.count_inversions(t) > 0
    ns.optimized_merge_sort(t, ns.find_config("6To8"))
    assert ns.count_inversions(t) == 0
    assert ns.multiset_digest(t) == oracle.multiset_digest(a)


@pytest.mark.slow
@pytest.mark.parametrize("algo,n", [("merge", 1 << 28), ("quick", 1 << 27)])
def test_i64_full_size_properties(ns, cuda, algo, n):
    """2 GiB / 1 GiB of int64 keys (no oracle at this size): the result is
    sorted and is a permutation of the input (multiset digest)."""
    import torch
    g = torch.Generator(device=cuda)
    g.manual_seed(2024)
    t = torch.randint(np.iinfo(np.int64).min, np.iinfo(np.int64).max, (n,), dtype=torch.int64,
                      device=cuda, generator=g)
    before = ns.multiset_digest(t)
    (ns.optimized_merge_sort if algo == "merge" else ns.optimized_quick_sort)(
        t, ns.find_config("6To8" if algo == "merge" else "3To5"))
    assert ns.count_inversions(t) == 0
    assert ns.multiset_digest(t) == before
    del t
    ns.release_scratch()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("seg_len", [2, 7, 100, 513, 4096, 9000, 16384, 20000, 70001])
def test_i64_segmented(ns, cuda, oracle, seg_len):
    import torch
    nseg = max(1, (1 << 18) // seg_len)
    a = oracle.generate_i64("random", nseg * seg_len, 31 + seg_len)
    for algo in (ns.Algorithm.merge_sort, ns.Algorithm.quick_sort):
        t = to_dev(a, cuda)
        ns.segmented_sort(t, seg_len, ns.find_config("3To5"), algo)
        assert np.array_equal(t.cpu().numpy().reshape(nseg, seg_len),
                              np.sort(a.reshape(nseg, seg_len), axis=1)), (seg_len, algo)
