"""GPU parity: the sm_100a kernels, called through the C ABI, against the CPU
oracle (oracle/netsort_oracle.c) and the reference's own outputs frozen in
tests/golden/golden.json.  Bit-exact for every case (int32 keys)."""
import hashlib
import itertools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SIZES = [0, 1, 2, 3, 4, 5, 7, 8, 9, 13, 16, 17, 31, 32, 33, 63, 64, 100, 255, 256, 257, 501,
         1000, 1023, 4096, 8191, 8192, 8193, 10000, 16383, 16384, 16385, 20000, 25000, 32768,
         65537, 100000, 262144, 1000000]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def to_dev(a, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.int32)).to(dev)


def from_dev(t):
    return t.cpu().numpy()


@pytest.mark.parametrize("algo", ["merge", "quick"])
@pytest.mark.parametrize("dist", ["random", "sorted", "nearly_sorted"])
def test_sizes_match_oracle(ns, cuda, oracle, algo, dist):
    cfg_name = "6To8" if algo == "merge" else "3To5"
    cfg = ns.find_config(cfg_name)
    for n in SIZES:
        a = oracle.generate_i32(dist, n, seed=42 + n)
        want = oracle.merge_sort(a, cfg_name) if algo == "merge" else oracle.quick_sort(a, cfg_name)
        t = to_dev(a, cuda)
        (ns.optimized_merge_sort if algo == "merge" else ns.optimized_quick_sort)(t, cfg)
        got = from_dev(t)
        assert np.array_equal(got, want), f"{algo} {dist} n={n}"


@pytest.mark.parametrize("cfg_name", ["Classic", "PowerOf2", "Even", "Odd", "3", "3To4", "3To5",
                                      "3To8", "6To8", "VarSort3", "VarSort4", "VarSort5"])
def test_every_config_both_algorithms(ns, cuda, oracle, cfg_name):
    cfg = ns.find_config(cfg_name)
    for n in (0, 1, 2, 3, 4, 7, 16, 33, 64, 501, 1000, 9000, 40000):
        a = oracle.generate_i32("random", n, seed=3000 + n)
        want = np.sort(a)
        for fn in (ns.optimized_merge_sort, ns.optimized_quick_sort):
            t = to_dev(a, cuda)
            fn(t, cfg)
            assert np.array_equal(from_dev(t), want), f"{fn.__name__} {cfg_name} n={n}"


def test_golden_reference_outputs(ns, cuda, oracle, golden):
    """Every frozen reference output (SHA-256) is reproduced bit-exactly."""
    for c in golden["cases"]:
        a = oracle.generate_i32(c["dist"], c["n"], c["seed"])
        assert sha(a) == c["input_sha256"], c
        t = to_dev(a, cuda)
        cfg = ns.find_config(c["config"])
        (ns.optimized_merge_sort if c["algo"] == "merge" else ns.optimized_quick_sort)(t, cfg)
        assert sha(from_dev(t)) == c["output_sha256"], (c["algo"], c["config"], c["dist"], c["n"])


def test_ternary_exhaustive(ns, cuda):
    """All {0,1,2} arrays of length <= 8 through both algorithms (acceptance.cpp:135-164),
    batched as segments so the whole sweep is a handful of launches."""
    import torch
    for length in range(2, 9):
        codes = np.array(list(itertools.product(range(3), repeat=length)), np.int32)
        flat = codes.reshape(-1)
        for algo in (ns.Algorithm.merge_sort, ns.Algorithm.quick_sort):
            for cfg_name in ("Classic", "3To5", "6To8", "Odd", "VarSort3"):
                t = to_dev(flat, cuda)
                ns.segmented_sort(t, length, ns.find_config(cfg_name), algo)
                got = from_dev(t).reshape(-1, length)
                assert np.array_equal(got, np.sort(codes, axis=1)), (length, cfg_name, algo)
    torch.cuda.synchronize()


def test_networks_exhaustive_on_device(ns, cuda):
    """Zero-one principle and every permutation, widths 2..8, through the
    base-case batch kernel (each array hits its own width's network)."""
    import torch
    for w in range(2, 9):
        perms = np.array(list(itertools.permutations(range(1, w + 1))), np.int32)
        bits = np.array([[(b >> i) & 1 for i in range(w)] for b in range(1 << w)], np.int32)
        arr = np.concatenate([perms, bits])
        offs = np.arange(0, arr.size + 1, w, dtype=np.int32)
        keys = to_dev(arr.reshape(-1), cuda)
        ns.sort_small_batch(keys, torch.from_numpy(offs).to(cuda))
        got = from_dev(keys).reshape(-1, w)
        assert np.array_equal(got, np.sort(arr, axis=1)), w


def test_sort_small_batch_matches_reference(ns, cuda, oracle, golden):
    import torch
    sb = golden["small_batch"]
    keys = to_dev(np.array(sb["input"], np.int32), cuda)
    offs = torch.tensor(sb["offsets"], dtype=torch.int32, device=cuda)
    ns.sort_small_batch(keys, offs)
    assert from_dev(keys).tolist() == sb["output"]
    # 2^20 ragged arrays against the oracle
    o, k = oracle.generate_batch_i32(1 << 20, 11)
    want = oracle.sort_small_batch(k, o)
    t = to_dev(k, cuda)
    ns.sort_small_batch(t, torch.from_numpy(o.view(np.int32)).to(cuda))
    assert np.array_equal(from_dev(t), want)


def test_sort_small_batch_edge_cases(ns, cuda):
    import torch
    # lengths 0 and 1 are no-ops; an empty batch is fine
    keys = to_dev(np.array([5, 3, 9, 2, 1], np.int32), cuda)
    offs = torch.tensor([0, 0, 1, 1, 3, 5], dtype=torch.int32, device=cuda)
    ns.sort_small_batch(keys, offs)
    assert from_dev(keys).tolist() == [5, 3, 9, 1, 2]
    ns.sort_small_batch(keys, torch.tensor([0], dtype=torch.int32, device=cuda))
    # a length above 8 is rejected (networks.hpp:99-103 throws there)
    bad = torch.tensor([0, 9], dtype=torch.int32, device=cuda)
    k9 = to_dev(np.arange(9, 0, -1, dtype=np.int32), cuda)
    with pytest.raises(ValueError):
        ns.sort_small_batch(k9, bad)
    assert from_dev(k9).tolist() == list(range(9, 0, -1))


def test_sort_small_batch_unaligned_views_keep_neighbours(ns, cuda, oracle):
    """Key arrays starting 0..3 keys past a 16-byte boundary, totals that are
    not multiples of 4, and CTAs whose arrays end in empty ones: the batch
    kernel stages each CTA's 16-byte cover with one bulk copy but must write
    back exactly its own keys — the guard keys around the view stay put."""
    import torch
    for shift in range(4):
        for narr, seed in ((1, 1), (7, 2), (1023, 3), (1025, 4), (5000, 5), (70001, 6)):
            o, k = oracle.generate_batch_i32(narr, seed)
            if narr > 2:  # a run of empty arrays at the end of the first CTA
                lens = np.diff(o.astype(np.int64))
                lens[min(1020, narr - 1):min(1024, narr)] = 0
                o = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
                k = k[:int(o[-1])]
            want = oracle.sort_small_batch(k, o)
            buf = np.full(len(k) + shift + 7, -12345, np.int32)
            buf[shift:shift + len(k)] = k
            t = to_dev(buf, cuda)
            view = t[shift:shift + len(k)]
            ns.sort_small_batch(view, torch.from_numpy(o.view(np.int32)).to(cuda))
            got = from_dev(t)
            assert np.array_equal(got[shift:shift + len(k)], want), (shift, narr)
            assert (got[:shift] == -12345).all() and (got[shift + len(k):] == -12345).all()


def test_segmented_matches_reference_prefix(ns, cuda, oracle, golden):
    g = golden["segmented"]
    nseg, seg = g["num_segments_checked"], g["seg_len"]
    a = oracle.generate_i32("random", nseg * seg, g["seed"])
    assert sha(a) == g["input_prefix_sha256"]
    t = to_dev(a, cuda)
    ns.segmented_sort(t, seg, ns.find_config(g["config"]), ns.Algorithm.quick_sort)
    assert sha(from_dev(t)) == g["output_prefix_sha256"]


def test_segmented_odd_lengths(ns, cuda, oracle):
    # every tile shape of the segmented path: <32,16> .. <128,16>, then
    # 32 keys per thread <128,32> (2049..4096), <256,32> (..8192), <512,32>
    # (..16384), and whole-array sorts above
    for seg in (1, 2, 3, 5, 100, 2049, 3000, 4096, 4097, 6000, 8192, 12345, 16384, 20000):
        nseg = max(1, 200000 // seg)
        a = oracle.generate_i32("random", nseg * seg, seed=seg)
        want = np.sort(a.reshape(nseg, seg), axis=1).reshape(-1)
        for algo in (ns.Algorithm.merge_sort, ns.Algorithm.quick_sort):
            t = to_dev(a, cuda)
            ns.segmented_sort(t, seg, ns.find_config("3To5"), algo)
            assert np.array_equal(from_dev(t), want), (seg, algo)
    # every leaf shape (LEAF 1 / 2 / 8) through the 32-keys-per-thread tiles
    for cfg in ("Classic", "VarSort3", "6To8"):
        for seg in (3000, 6000, 16384):
            nseg = max(1, 100000 // seg)
            a = oracle.generate_i32("random", nseg * seg, seed=seg + 1)
            want = np.sort(a.reshape(nseg, seg), axis=1).reshape(-1)
            t = to_dev(a, cuda)
            ns.segmented_sort(t, seg, ns.find_config(cfg), ns.Algorithm.merge_sort)
            assert np.array_equal(from_dev(t), want), (seg, cfg)


@pytest.mark.parametrize("key_bytes", [4, 8])
def test_segmented_small_segments_share_warps(ns, cuda, oracle, key_bytes):
    """Segments of up to 512 keys: 2^LV lanes of a warp per segment, several
    segments per warp (small_segments_kernel).  Every lane-group size and its
    boundaries, segment counts that leave warps and CTAs partly empty, every
    leaf shape, duplicates and the extreme key values (the pad value itself)."""
    import torch
    dt = np.int32 if key_bytes == 4 else np.int64
    info = np.iinfo(dt)
    rng = np.random.default_rng(7)
    for seg in (1, 2, 7, 8, 15, 16, 17, 31, 32, 33, 63, 64, 65, 100, 128, 129, 200, 256, 257,
                300, 511, 512):
        for nseg in (1, 3, 37, 255, 257, 1000):
            a = rng.integers(info.min, info.max, size=nseg * seg, dtype=dt, endpoint=True)
            a[:: max(1, seg // 2)] = info.max   # real keys equal to the pad value
            a[1:: 5] = info.min
            if seg > 3:
                m = min(len(a[2:: 3]), len(a[3:: 3]))
                a[2:: 3][:m] = a[3:: 3][:m]  # duplicates
            want = np.sort(a.reshape(nseg, seg), axis=1).reshape(-1)
            for cfg in ("6To8", "Classic") if nseg == 37 else ("3To5",):
                for algo in (ns.Algorithm.merge_sort, ns.Algorithm.quick_sort):
                    t = torch.from_numpy(a.copy()).to(cuda)
                    ns.segmented_sort(t, seg, ns.find_config(cfg), algo)
                    assert np.array_equal(t.cpu().numpy(), want), (seg, nseg, cfg, algo)


@pytest.mark.parametrize("nseg,seg", [(7, 16385), (5, 40000), (3, 100_001), (2, (1 << 21) + 3),
                                      (64, 32768), (40, 50_000)])
def test_segmented_merge_sort_long_segments_batched(ns, cuda, oracle, nseg, seg):
    """Segments longer than one tile, merge sort: every segment sorted at once
    (segment-aligned tiles, passes whose run pairs never cross a segment);
    sorted, duplicate-heavy and random segments."""
    for kind in ("random", "dups", "sorted"):
        if kind == "random":
            a = oracle.generate_i32("random", nseg * seg, seed=seg + nseg)
        elif kind == "dups":
            a = (oracle.generate_i32("random", nseg * seg, seed=seg) % 11).astype(np.int32)
        else:
            a = np.tile(np.arange(seg, dtype=np.int32)[::-1], nseg)  # each segment descending
        want = np.sort(a.reshape(nseg, seg), axis=1).reshape(-1)
        t = to_dev(a, cuda)
        ns.segmented_sort(t, seg, ns.find_config("6To8"), ns.Algorithm.merge_sort)
        assert np.array_equal(from_dev(t), want), (nseg, seg, kind)


def test_range_sorts_leave_outside_untouched(ns, cuda, oracle):
    """test_hybrid.cpp:320-342, on the device path and the host path."""
    base = oracle.generate_i32("random", 40000, 17)
    lo, hi = 10007, 29999
    for name in ("Classic", "3To8", "VarSort4", "6To8", "3To5"):
        cfg = ns.find_config(name)
        for fn in (ns.optimized_merge_sort, ns.optimized_quick_sort):
            t = to_dev(base, cuda)
            fn(t, lo, hi, cfg)
            got = from_dev(t)
            assert np.array_equal(got[:lo], base[:lo]) and np.array_equal(got[hi + 1:], base[hi + 1:])
            assert np.array_equal(got[lo:hi + 1], np.sort(base[lo:hi + 1]))
            h = base.copy()
            fn(h, lo, hi, cfg)
            assert np.array_equal(h, got)
            # inverted range is a no-op (hybrid.hpp:160, 201)
            h2 = base.copy()
            fn(h2, 5, 4, cfg)
            assert np.array_equal(h2, base)


def test_host_entry_points(ns, cuda, oracle):
    for n in (0, 1, 7, 10000, 1000000):
        a = oracle.generate_i32("random", n, 5)
        want = np.sort(a)
        for fn, cfg in ((ns.optimized_merge_sort, "6To8"), (ns.optimized_quick_sort, "3To5"),
                        (ns.classical_merge_sort, None), (ns.classical_quick_sort, None)):
            h = a.copy()
            fn(h, ns.find_config(cfg)) if cfg else fn(h)
            assert np.array_equal(h, want), (fn.__name__, n)


def test_duplicates_and_extremes(ns, cuda):
    rng = np.random.default_rng(0)
    cases = [
        np.full(100000, 7, np.int32),
        np.full(50000, np.iinfo(np.int32).max, np.int32),
        np.full(50000, np.iinfo(np.int32).min, np.int32),
        rng.integers(0, 3, 300000).astype(np.int32),
        rng.integers(np.iinfo(np.int32).min, np.iinfo(np.int32).max, 300000, dtype=np.int32),
        np.concatenate([np.full(200000, 5, np.int32), rng.integers(0, 10, 100000).astype(np.int32)]),
        np.arange(300000, 0, -1, dtype=np.int32),
        np.tile(np.arange(1000, dtype=np.int32), 300),
    ]
    for a in cases:
        for fn, cfg in ((ns.optimized_merge_sort, "6To8"), (ns.optimized_quick_sort, "3To5")):
            t = to_dev(a, cuda)
            fn(t, ns.find_config(cfg))
            assert np.array_equal(from_dev(t), np.sort(a)), (fn.__name__, a[:5])


def test_sentinel_valued_keys_through_every_path(ns, cuda):
    """The merge loops run over +inf-sentinel-padded runs (K or K+4 key-maximum
    sentinels after every run, no cursor clamps): real keys equal to the
    sentinel must come out right through every path that uses them — the
    one-CTA and two-tile small sorts, the tiled merge sort, the segmented
    tiles (16 and 32 keys per thread), the quick-sort buckets, merge() and
    the int64 twins."""
    import torch
    rng = np.random.default_rng(11)
    imax, imin = np.iinfo(np.int32).max, np.iinfo(np.int32).min

    def heavy(n, dtype=np.int32):
        info = np.iinfo(dtype)
        a = rng.integers(-1000, 1000, n).astype(dtype)
        a[rng.random(n) < 0.4] = info.max
        a[rng.random(n) < 0.05] = info.min
        return a

    for n in (5000, 8192, 10000, 16384, 20000, 100003, (1 << 21) + 5):
        a = heavy(n)
        for fn, cfg in ((ns.optimized_merge_sort, "6To8"), (ns.optimized_quick_sort, "3To5")):
            t = to_dev(a, cuda)
            fn(t, ns.find_config(cfg))
            assert np.array_equal(from_dev(t), np.sort(a)), (fn.__name__, n)
    for seg in (3000, 6000, 12000, 16384):
        nseg = 40
        a = heavy(nseg * seg)
        want = np.sort(a.reshape(nseg, seg), axis=1).reshape(-1)
        for algo in (ns.Algorithm.merge_sort, ns.Algorithm.quick_sort):
            t = to_dev(a, cuda)
            ns.segmented_sort(t, seg, ns.find_config("3To5"), algo)
            assert np.array_equal(from_dev(t), want), (seg, algo)
    # merge(): two sorted runs whose tails are all INT_MAX
    left = np.sort(heavy(70001))
    right = np.sort(heavy(50003))
    a = np.concatenate([left, right])
    t = to_dev(a, cuda)
    ns.merge(t, 0, len(left) - 1, len(a) - 1)
    assert np.array_equal(from_dev(t), np.sort(a))
    # int64 keys equal to INT64_MAX through the tiled and segmented paths
    for n in (20000, (1 << 20) + 3):
        a = heavy(n, np.int64)
        t = torch.from_numpy(a).to(cuda)
        ns.optimized_merge_sort(t, ns.find_config("6To8"))
        assert np.array_equal(t.cpu().numpy(), np.sort(a)), n
    a = heavy(30 * 16384, np.int64)
    t = torch.from_numpy(a).to(cuda)
    ns.segmented_sort(t, 16384, ns.find_config("3To5"), ns.Algorithm.merge_sort)
    assert np.array_equal(t.cpu().numpy(), np.sort(a.reshape(30, 16384), axis=1).reshape(-1))
    assert imax > imin


def test_checking_helpers(ns, cuda, oracle):
    a = oracle.generate_i32("random", 123457, 9)
    t = to_dev(a, cuda)
    assert ns.multiset_digest(t) == oracle.multiset_digest(a)
    assert ns.count_inversions(t) == int(np.sum(a[:-1] > a[1:]))
    ns.optimized_merge_sort(t, ns.find_config("6To8"))
    assert ns.count_inversions(t) == 0
    assert ns.multiset_digest(t) == oracle.multiset_digest(a)


@pytest.mark.slow
@pytest.mark.parametrize("algo", ["merge", "quick"])
def test_full_size_properties(ns, cuda, oracle, algo):
    """At BASELINE's largest single-array size: sorted + same multiset."""
    import torch
    n = 1 << 30 if algo == "merge" else 16_777_216
    g = torch.Generator(device=cuda)
    g.manual_seed(1234)
    t = torch.randint(0, 2**31 - 1, (n,), dtype=torch.int32, device=cuda, generator=g)
    d0 = ns.multiset_digest(t)
    (ns.optimized_merge_sort if algo == "merge" else ns.optimized_quick_sort)(
        t, ns.find_config("6To8" if algo == "merge" else "3To5"))
    assert ns.count_inversions(t) == 0
    assert ns.multiset_digest(t) == d0
    del t
    ns.release_scratch()
    torch.cuda.empty_cache()


def test_merge_pairs_from_separate_buffers(ns, cuda, oracle):
    """ns_merge_pairs_i32 with every run in its own allocation and at odd
    offsets — the same kernel that, in the p2p sample sort, reads the runs
    from peer GPUs over NVLink (on one GPU the "peers" are local buffers;
    nothing waits on another kernel)."""
    import torch
    from paper_2503_05934_b200 import samplesort
    rng = np.random.default_rng(9)
    ops = samplesort.DeviceOps()
    for lens in ([5000, 7000], [0, 300000, 1, 77777, 123456, 0, 9, 50000],
                 [100000] * 8, [3, 0, 0], [250000, 250001, 249999]):
        bufs, runs, allk = [], [], []
        for i, ln in enumerate(lens):
            v = np.sort(rng.integers(-2**31, 2**31 - 1, ln, dtype=np.int64).astype(np.int32))
            if i % 3 == 0:
                v[: ln // 2] = 7  # duplicates across runs
                v = np.sort(v)
            pad = i % 4  # misaligned start inside its allocation
            t = torch.zeros(ln + pad + 1, dtype=torch.int32, device=cuda)
            t[pad:pad + ln] = torch.from_numpy(v).to(cuda)
            bufs.append(t)
            runs.append((t.data_ptr() + 4 * pad, ln))
            allk.append(v)
        out = ops.merge_pull(runs, cuda)
        want = np.sort(np.concatenate(allk))
        assert np.array_equal(out.cpu().numpy(), want), lens


def test_ipc_handle_export(ns, cuda):
    import ctypes as C
    import torch
    t = torch.empty(1 << 20, dtype=torch.int32, device=cuda)
    h = (C.c_uint8 * 64)()
    off = C.c_uint64()
    assert ns.lib().ns_ipc_get_handle(t.data_ptr() + 4096, C.cast(h, C.c_void_p), C.byref(off)) == 0
    assert off.value % 4 == 0 and off.value >= 4096 and any(bytes(h))


@pytest.mark.parametrize("world,n,dist_kind", [(2, 3_000_000, "random"), (3, 1_000_003, "sorted"),
                                               (4, 2_000_000, "nearly_sorted")])
def test_p2p_sample_sort_processes_one_gpu(ns, cuda, world, n, dist_kind):
    """The p2p exchange end to end: `world` processes on one GPU, each rank's
    pull-merge kernel reading the other ranks' shards through CUDA IPC
    mappings (host-side gloo for the metadata; no kernel waits on another)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "tests", "multiproc_p2p_gpu.py"),
                          str(world), str(n), dist_kind], cwd=root, capture_output=True,
                         text=True, timeout=600)
    assert "P2P_OK" in out.stdout, (out.stdout[-1500:], out.stderr[-3000:])


@pytest.mark.slow
def test_full_batch_matches_reference_digest(ns, cuda, oracle, golden):
    """BASELINE config 2 at full size: 2^24 ragged arrays, digest of the
    reference's own output (tests/golden/golden.json)."""
    import torch
    b = golden["batch"]
    offs, keys = oracle.generate_batch_i32(b["num_arrays"], b["seed"])
    assert sha(offs) == b["offsets_sha256"] and sha(keys) == b["input_sha256"]
    k = to_dev(keys, cuda)
    ns.sort_small_batch(k, torch.from_numpy(offs.view(np.int32)).to(cuda))
    assert sha(from_dev(k)) == b["output_sha256"]


@pytest.mark.slow
def test_full_segmented_batch(ns, cuda, oracle, golden):
    """BASELINE config 4's segmented batch at full size (65,536 x 16,384):
    the reference digest of the first 1,024 segments plus sortedness of every
    segment and the multiset of the whole batch."""
    import torch
    g = golden["segmented"]
    seg, nseg = g["seg_len"], g["full_num_segments"]
    n = seg * nseg
    t = torch.empty(n, dtype=torch.int32, device=cuda)
    from paper_2503_05934_b200._lib import check
    check(ns.lib().ns_generate_i32(t.data_ptr(), n, 0, g["seed"],
                                   torch.cuda.current_stream().cuda_stream), "gen")
    d0 = ns.multiset_digest(t)
    ns.segmented_sort(t, seg, ns.find_config(g["config"]), ns.Algorithm.quick_sort)
    prefix = from_dev(t[: g["num_segments_checked"] * seg])
    assert sha(prefix) == g["output_prefix_sha256"]
    v = t.view(nseg, seg)
    assert bool((v[:, 1:] >= v[:, :-1]).all())
    assert ns.multiset_digest(t) == d0


@pytest.mark.slow
def test_p2p_sample_sort_large(ns, cuda):
    """Config 5's exchange at scale: 2^27 keys over 2 processes (p2p pull-merge)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "tests", "multiproc_p2p_gpu.py"),
                          "2", str(1 << 27), "random"], cwd=root, capture_output=True,
                         text=True, timeout=900)
    assert "P2P_OK" in out.stdout, (out.stdout[-1500:], out.stderr[-3000:])


def test_merge_standalone_matches_oracle(ns, cuda, oracle):
    """merge (hybrid.hpp:186-193): stable merge of a[left..mid], a[mid+1..right],
    int32 and int64, device tensors and host arrays, against oracle_merge."""
    rng = np.random.default_rng(12)
    for n, left, mid, right in [(10, 0, 4, 9), (1000, 0, 0, 999), (1000, 0, 998, 999),
                                (50000, 100, 30000, 49000), (1 << 20, 0, 700000, (1 << 20) - 1),
                                (300001, 5, 5, 300000)]:
        for dt in (np.int32, np.int64):
            a = rng.integers(-1000, 1000, n).astype(dt)
            a[left:mid + 1].sort()
            a[mid + 1:right + 1].sort()
            want = a.copy()
            want[left:right + 1] = np.sort(a[left:right + 1], kind="stable")
            if dt == np.int32:
                w32 = a.copy()
                oracle.lib().oracle_merge_i32(w32, left, mid, right)
                assert np.array_equal(w32, want)
            import torch
            t = torch.from_numpy(a.copy()).to(cuda)
            ns.merge(t, left, mid, right)
            assert np.array_equal(t.cpu().numpy(), want), (n, left, mid, right, dt)
            h = a.copy()
            ns.merge(h, left, mid, right)
            assert np.array_equal(h, want), (n, dt, "host")
    with pytest.raises(ValueError):
        ns.merge(np.zeros(4, np.int32), 2, 1, 3)


def test_run_variant_with_stats(ns, cuda, oracle):
    import torch
    st = ns.DispatchStats()
    a = oracle.generate_i32("random", 100000, 3)
    t = torch.from_numpy(a).to(cuda)
    ns.run_variant(ns.SortVariant(ns.Algorithm.merge_sort, ns.find_config("6To8")), t, st)
    want, ost = oracle.merge_sort(a, "6To8", stats=True)
    assert np.array_equal(t.cpu().numpy(), want)
    assert st.network_hits == list(ost.network_hits) and st.merges == ost.merges
    assert st.max_depth == ost.max_depth
    # quick sort: the traced reference recursion (qs_trace.cu), counters added
    q = ns.DispatchStats()
    t = torch.from_numpy(a).to(cuda)
    ns.run_variant(ns.SortVariant(ns.Algorithm.quick_sort, ns.find_config("3To5")), t, q)
    want, qst = oracle.quick_sort(a, "3To5", stats=True)
    assert np.array_equal(t.cpu().numpy(), want)
    assert q.network_hits == list(qst.network_hits) and q.partitions == qst.partitions
    assert q.max_depth == qst.max_depth and q.merges == 0


def test_merge_runs_many_runs_both_key_types(ns, cuda):
    """ns_merge_runs_* (the g-way merge of the sample sort and of the chunked
    host path): ragged runs, 1..64 of them, int32 and int64."""
    import ctypes as C
    import torch
    L = ns.lib()
    rng = np.random.default_rng(4)
    for dt, tt, sfx in ((np.int32, torch.int32, "i32"), (np.int64, torch.int64, "i64")):
        for nruns in (2, 3, 7, 16, 33, 64):
            lens = rng.integers(0, 40000, nruns)
            lens[rng.integers(0, nruns)] = 0
            runs = [np.sort(rng.integers(-2**31, 2**31, l).astype(dt)) for l in lens]
            flat = np.concatenate(runs)
            offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
            t = torch.from_numpy(flat.copy()).to(cuda)
            tb = getattr(L, "ns_merge_runs_temp_bytes" + ("" if sfx == "i32" else "_i64"))(
                flat.size, nruns)
            tmp = torch.empty(max(tb, 1), dtype=torch.uint8, device=cuda)
            o = (C.c_int64 * (nruns + 1))(*offs.tolist())
            rc = getattr(L, f"ns_merge_runs_{sfx}")(t.data_ptr(), C.cast(o, C.c_void_p), nruns,
                                                    tmp.data_ptr(), tb,
                                                    torch.cuda.current_stream().cuda_stream)
            assert rc == 0
            assert np.array_equal(t.cpu().numpy(), np.sort(flat)), (sfx, nruns)


@pytest.mark.parametrize("n", [0, 1, 2, 7, 1000, 16384, 16385, 100000, 1 << 20, 3_000_001])
def test_sort_pairs_and_argsort_stable(ns, cuda, oracle, n):
    """Stable key-value sort / argsort against the
    classical stable merge sort oracle, many duplicate keys."""
    import torch
    rng = np.random.default_rng(n)
    keys = rng.integers(-50, 50, n).astype(np.int32)
    if n > 10:
        keys[: n // 10] = np.iinfo(np.int32).max   # real keys equal to the sentinel
        keys[n // 10: n // 5] = np.iinfo(np.int32).min
    vals = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    wk, wv = oracle.stable_sort_pairs(keys, vals)
    tk = torch.from_numpy(keys.copy()).to(cuda)
    tv = torch.from_numpy(vals.view(np.int32).copy()).to(cuda)
    ns.sort_pairs(tk, tv)
    assert np.array_equal(tk.cpu().numpy(), wk)
    assert np.array_equal(tv.cpu().numpy().view(np.uint32), wv)
    tk2 = torch.from_numpy(keys.copy()).to(cuda)
    perm = ns.argsort(tk2)
    assert np.array_equal(tk2.cpu().numpy(), keys)  # unchanged
    assert np.array_equal(perm.cpu().numpy(), np.argsort(keys, kind="stable"))


@pytest.mark.slow
def test_merge_sort_beyond_2_31_keys(ns, cuda):
    """n = 2^31 + 4099 int32 keys (8.6 GB): indexing past 32 bits in every
    kernel of the merge sort; sorted and a permutation of the input."""
    import torch
    n = (1 << 31) + 4099
    t = torch.empty(n, dtype=torch.int32, device=cuda)
    L = ns.lib()
    from paper_2503_05934_b200._lib import check
    check(L.ns_generate_i32(t.data_ptr(), n, 0, 99, torch.cuda.current_stream().cuda_stream), "gen")
    before = ns.multiset_digest(t)
    ns.optimized_merge_sort(t, ns.find_config("6To8"))
    assert ns.count_inversions(t) == 0
    assert ns.multiset_digest(t) == before
    del t
    ns.release_scratch()
    torch.cuda.empty_cache()


@pytest.mark.slow
@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
def test_bench_multi_rank_code_path_on_one_gpu(exchange):
    """bench.py's N>1 path (sample sort, max-over-ranks timing, nvlink object)
    with 2 ranks sharing cuda:0 over gloo (BENCH_TEST_ONE_GPU=1): a code-path
    check, never a bench number."""
    import json
    import os
    import socket
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, BENCH_TEST_ONE_GPU="1")
    r = subprocess.run(["python", "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
                        "2", "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1",
                        "--warmup", "1", "--keys", str(1 << 24), "--exchange", exchange],
                       capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["verified"] is True
    assert line["nvlink"]["bytes_per_rank_max"] > 0
    assert line["exchange"]["mode"] == exchange
    sb = line["sharded_batches"]  # the batch configs split by array over the ranks
    assert sb["batch"]["verified"] is True and sb["segmented"]["verified"] is True


@pytest.mark.slow
def test_bench_single_gpu_line_contract():
    """bench.py at N=1 on a small array: one JSON line with the keys the
    driver reads (value, timing, roofline, byte model, e2e with its copy
    bytes, launches, clocks, every BASELINE config cell verified against the
    reference's digests) and a verified sort."""
    import json
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run(["python", os.path.join(root, "bench.py"), "--steps", "2", "--warmup", "3",
                        "--keys", str(1 << 24), "--no-cpu-baseline", "--no-size-sweep"],
                       capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "byte_model", "e2e", "gpu_launches", "clocks", "configs"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 2 and line["warmup"] == 3
    assert line["verified"] is True and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["roofline"]["bound"] == "hbm" and 0 < line["roofline"]["frac"] < 2
    assert line["e2e"]["h2d_bytes_per_step"] == 4 << 24 == line["e2e"]["d2h_bytes_per_step"]
    cells = line["configs"]
    assert len(cells) == 18, sorted(cells)
    for name, rec in cells.items():
        assert rec["verified"] is True, name
        assert rec["device_ms"] > 0 and rec["hbm_frac"] > 0, name
    assert "workload" in line["config"]


@pytest.mark.slow
@pytest.mark.parametrize("kind", ["all_equal", "three_values", "reverse", "sawtooth", "int_max_heavy"])
def test_adversarial_inputs_large(ns, cuda, kind):
    """2^26 keys of adversarial shapes through both algorithms: ties everywhere
    (merge-path ties, constant quick-sort buckets), reverse order, periodic
    runs, and heavy use of INT_MAX (the kernels' sentinel/pad value)."""
    import torch
    n = 1 << 26
    g = torch.Generator(device=cuda)
    g.manual_seed(7)
    if kind == "all_equal":
        base = torch.full((n,), 12345, dtype=torch.int32, device=cuda)
    elif kind == "three_values":
        base = torch.randint(0, 3, (n,), dtype=torch.int32, device=cuda, generator=g)
    elif kind == "reverse":
        base = torch.arange(n, 0, -1, dtype=torch.int32, device=cuda)
    elif kind == "sawtooth":
        base = (torch.arange(n, dtype=torch.int32, device=cuda) % 4099) * 3
    else:
        base = torch.randint(0, 2**31 - 1, (n,), dtype=torch.int32, device=cuda, generator=g)
        base[torch.rand(n, device=cuda, generator=g) < 0.3] = 2**31 - 1
    want_digest = ns.multiset_digest(base)
    for fn, cfg in ((ns.optimized_merge_sort, "6To8"), (ns.optimized_quick_sort, "3To5")):
        t = base.clone()
        fn(t, ns.find_config(cfg))
        assert ns.count_inversions(t) == 0, (kind, fn.__name__)
        assert ns.multiset_digest(t) == want_digest, (kind, fn.__name__)
    del base, t
    ns.release_scratch()
    torch.cuda.empty_cache()


def test_c_abi_status_codes_on_device(ns, cuda):
    """The C ABI never throws; bad arguments / short scratch return statuses
    and leave the keys untouched (include/netsort_b200.h conventions)."""
    import ctypes as C
    import torch
    from paper_2503_05934_b200 import _lib
    L = ns.lib()
    s = torch.cuda.current_stream().cuda_stream
    n = 100_000
    a = torch.randint(0, 1000, (n,), dtype=torch.int32, device=cuda)
    before = a.clone()
    need = L.ns_merge_sort_temp_bytes(n)
    assert need > 0
    small = torch.empty(need // 2, dtype=torch.uint8, device=cuda)
    # scratch too small -> NS_ERR_TEMP, nothing launched on the keys
    assert L.ns_merge_sort_i32(a.data_ptr(), n, 1 << 8, 0, small.data_ptr(), need // 2, s) == \
        _lib.NS_ERR_TEMP
    assert L.ns_merge_sort_i32(a.data_ptr(), n, 1 << 8, 0, None, 0, s) == _lib.NS_ERR_TEMP
    torch.cuda.synchronize()
    assert torch.equal(a, before)
    # null keys with n > 0 -> NS_ERR_INVALID; n == 0 is a no-op on null
    assert L.ns_merge_sort_i32(None, n, 1 << 8, 0, None, 0, s) == _lib.NS_ERR_INVALID
    assert L.ns_quick_sort_i32(None, 10, 1 << 3, 0, None, 0, s) == _lib.NS_ERR_INVALID
    assert L.ns_quick_sort_i64(None, 1, 1 << 3, 0, None, 0, s) == _lib.NS_ERR_INVALID
    assert L.ns_merge_sort_i32(None, 0, 1 << 8, 0, None, 0, s) == _lib.NS_OK
    assert L.ns_quick_sort_i64(None, 0, 1 << 3, 0, None, 0, s) == _lib.NS_OK
    qneed = L.ns_quick_sort_temp_bytes(n)
    assert L.ns_quick_sort_i32(a.data_ptr(), n, 1 << 3, 0, small.data_ptr(), 16, s) == \
        _lib.NS_ERR_TEMP
    # merge runs: bad run count / decreasing offsets
    offs = (C.c_int64 * 3)(0, 60_000, 50_000)
    tb = L.ns_merge_runs_temp_bytes(n, 2)
    big = torch.empty(max(tb, qneed, 1), dtype=torch.uint8, device=cuda)
    assert L.ns_merge_runs_i32(a.data_ptr(), C.cast(offs, C.c_void_p), 2, big.data_ptr(), tb,
                               s) == _lib.NS_ERR_INVALID
    assert L.ns_merge_runs_i32(a.data_ptr(), C.cast(offs, C.c_void_p), 0, big.data_ptr(), tb,
                               s) == _lib.NS_ERR_INVALID
    # batch with an array longer than 8 -> NS_ERR_INVALID, keys untouched
    keys = torch.arange(20, 0, -1, dtype=torch.int32, device=cuda)
    koffs = torch.tensor([0, 4, 16, 20], dtype=torch.int32, device=cuda)
    kb = keys.clone()
    assert L.ns_sort_small_batch_i32(keys.data_ptr(), koffs.data_ptr(), 3, s) == _lib.NS_ERR_INVALID
    assert torch.equal(keys, kb)
    # key-value: n >= 2^32 rejected without touching memory
    assert L.ns_sort_pairs_i32(a.data_ptr(), None, 1 << 33, big.data_ptr(), tb, s) == \
        _lib.NS_ERR_INVALID
    # the status strings are never NULL
    for st in range(-1, 6):
        assert L.ns_status_string(st)
    torch.cuda.synchronize()
    assert torch.equal(a, before)


def test_two_streams_concurrently(ns, cuda, oracle):
    """Stream-ordered and reentrant on disjoint buffers: two sorts on two
    streams, each with its own scratch, overlap without interference."""
    import torch
    from paper_2503_05934_b200._lib import check
    L = ns.lib()
    n = 1 << 22
    a = oracle.generate_i32("random", n, 1)
    b = oracle.generate_i32("nearly_sorted", n, 2)
    ta, tb_ = torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda)
    need = L.ns_merge_sort_temp_bytes(n)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    xa = torch.empty(need, dtype=torch.uint8, device=cuda)
    xb = torch.empty(need, dtype=torch.uint8, device=cuda)
    torch.cuda.synchronize()
    for _ in range(3):
        ta.copy_(torch.from_numpy(a))
        tb_.copy_(torch.from_numpy(b))
        torch.cuda.synchronize()
        check(L.ns_merge_sort_i32(ta.data_ptr(), n, 1 << 8, 0, xa.data_ptr(), need, sa.cuda_stream), "a")
        check(L.ns_merge_sort_i32(tb_.data_ptr(), n, 1 << 8, 0, xb.data_ptr(), need,
                                  sb.cuda_stream), "b")
        torch.cuda.synchronize()
        assert np.array_equal(ta.cpu().numpy(), np.sort(a))
        assert np.array_equal(tb_.cpu().numpy(), np.sort(b))


def test_batch_from_two_host_threads(ns, cuda, oracle):
    """The batch call validates lengths through a device flag read back at
    the end of the call: calls from two host threads (one with a bad length,
    one good, each on its own stream) must not see each other's flag."""
    import threading
    import torch
    o, k = oracle.generate_batch_i32(1 << 16, 5)
    want = oracle.sort_small_batch(k, o)
    bad_o = o.copy()
    bad_o[1:] += 9  # the first array has 9 + len keys: invalid (> 8)
    kb = np.concatenate([k, np.zeros(9, np.int32)])
    errors = {}

    def run(tag, keys, offs, reps):
        torch.cuda.set_device(cuda)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            tk = torch.from_numpy(keys).to(cuda)
            to = torch.from_numpy(offs.view(np.int32)).to(cuda)
            res = []
            for _ in range(reps):
                w = tk.clone()
                try:
                    ns.sort_small_batch(w, to)
                    res.append(("ok", w.cpu().numpy()))
                except ValueError:
                    res.append(("bad", None))
            errors[tag] = res

    ta = threading.Thread(target=run, args=("good", k, o, 20))
    tb = threading.Thread(target=run, args=("bad", kb, bad_o, 20))
    ta.start(); tb.start(); ta.join(); tb.join()
    assert all(r == "ok" and np.array_equal(v, want) for r, v in errors["good"])
    assert all(r == "bad" for r, _ in errors["bad"])


_PARTITION_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2503_05934_b200 as ns
from oracle import oracle as O
for n in (16385, 20000, 65537, 100003, 1000001, 3 * 8192 * 37 + 5):
    for dist in ("random", "sorted", "nearly_sorted"):
        a = O.generate_i32(dist, n, n)
        t = torch.from_numpy(a).cuda()
        ns.optimized_merge_sort(t, ns.find_config("6To8"))
        assert np.array_equal(t.cpu().numpy(), np.sort(a)), (n, dist)
        a64 = O.generate_i64(dist, n, n)
        t = torch.from_numpy(a64).cuda()
        ns.optimized_merge_sort(t, ns.find_config("6To8"))
        assert np.array_equal(t.cpu().numpy(), np.sort(a64)), (n, dist, "i64")
print("ok")
"""


@pytest.mark.parametrize("env", [{"NSB_FUSED_MAX": "0"},
                                 {"NSB_FUSED_MAX": "0", "NSB_SAMPLES": "0"}])
def test_partition_kernels_at_small_sizes(env):
    """The separate partition kernels (block-sample bracketed v3, plain v2)
    normally run only for passes of > 4096 tiles (~32 M keys); forcing them
    at odd small sizes checks partial last blocks and pairs against numpy."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run(["python", "-c", _PARTITION_SCRIPT, root], capture_output=True, text=True,
                       timeout=600, env=dict(os.environ, **env), cwd=root)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]


@pytest.mark.slow
def test_merge_sort_odd_size_above_fused_threshold(ns, cuda):
    """n = 2^25 + 12345: passes with separate partitions and block samples,
    ragged last pairs and a partial last sample block."""
    import torch
    from paper_2503_05934_b200._lib import check
    n = (1 << 25) + 12345
    t = torch.empty(n, dtype=torch.int32, device=cuda)
    check(ns.lib().ns_generate_i32(t.data_ptr(), n, 0, 5, torch.cuda.current_stream().cuda_stream),
          "gen")
    before = ns.multiset_digest(t)
    ns.optimized_merge_sort(t, ns.find_config("6To8"))
    assert ns.count_inversions(t) == 0 and ns.multiset_digest(t) == before
