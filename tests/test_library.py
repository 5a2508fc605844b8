"""CPU tests of the product library boundary: the C-ABI .so loads, exports
every symbol include/netsort_b200.h declares, and its host-side logic
(configuration registry, base_case_applies, network tables) matches the
reference.  No compute call runs here except the no-fallback check."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "netsort_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ns_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    fns = declared_functions()
    for must in ("ns_merge_sort_i32", "ns_quick_sort_i32", "ns_sort_small_batch_i32",
                 "ns_segmented_sort_i32", "ns_find_config", "ns_base_case_applies",
                 "ns_merge_sort_host_i32", "ns_quick_sort_host_i32", "ns_bucket_bounds_i32",
                 "ns_merge_runs_i32"):
        assert must in fns


def test_library_exports_every_declared_symbol(ns):
    from paper_2503_05934_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (ns_[a-z0-9_]+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    # the Python binding declares exactly the header's functions
    assert sorted(_lib.SIGNATURES) == declared_functions()


def test_library_is_sm100a_only(ns):
    from paper_2503_05934_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_registry_matches_reference(ns, oracle):
    reg = ns.config_registry()
    assert [(c.name, c.width_mask, c.varsort_max) for c in reg] == oracle.REGISTRY
    assert reg[0].is_classic() and len(ns.bundled_variants()) == 24
    assert ns.find_config("9To12") is None and ns.find_config("classic") is None
    if oracle.ref_available():
        R = oracle.ref()
        assert R.ref_config_count() == len(reg)
        for i, c in enumerate(reg):
            assert R.ref_config_name(i).decode() == c.name
            m, v = C.c_uint32(), C.c_int()
            assert R.ref_find_config(c.name.encode(), C.byref(m), C.byref(v)) == 0
            assert (m.value, v.value) == (c.width_mask, c.varsort_max)


def test_base_case_applies_table(ns, oracle):
    """test_hybrid.cpp:48-100 restated against the library."""
    f = ns.find_config
    assert ns.base_case_applies(7, f("6To8")) and not ns.base_case_applies(5, f("6To8"))
    assert ns.base_case_applies(2, f("VarSort5")) and ns.base_case_applies(5, f("VarSort5"))
    assert not ns.base_case_applies(6, f("VarSort5"))
    assert ns.base_case_applies(8, f("PowerOf2")) and not ns.base_case_applies(2, f("3"))
    for c in ns.config_registry():
        for size in range(-1, 12):
            want = bool(oracle.lib().oracle_base_case_applies(size, c.width_mask, c.varsort_max))
            assert ns.base_case_applies(size, c) == want


def test_network_tables_zero_one(ns):
    counts = {2: 1, 3: 3, 4: 5, 5: 9, 6: 12, 7: 16, 8: 19}
    for w in range(2, 9):
        net = ns.network(w)
        assert len(net) == counts[w]
        for bits in range(1 << w):
            v = [(bits >> i) & 1 for i in range(w)]
            for lo, hi in net:
                assert lo < hi < w
                if v[hi] < v[lo]:
                    v[lo], v[hi] = v[hi], v[lo]
            assert v == sorted(v)
    for bad in (-1, 0, 1, 9):
        with pytest.raises(ValueError):
            ns.network(bad)


def test_thread_sort_networks_host_compiled(tmp_path):
    """The per-thread base case of the tile sort (networks.cuh: LEAF-wide
    networks, then Batcher odd-even merges up to K) compiled for the host and
    checked by the zero-one principle (tests/cpp/thread_sort_check.cpp)."""
    exe = tmp_path / "thread_sort_check"
    subprocess.run(["g++", "-std=c++20", "-O2", "-D__host__=", "-D__device__=",
                    "-D__forceinline__=inline", "-Wno-unknown-pragmas",
                    "-I" + os.path.join(ROOT, "paper_2503_05934_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "thread_sort_check.cpp"), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and "thread_sort ok" in out.stdout, out.stdout + out.stderr


def test_leaf_width_follows_reference_recursion_on_8(ns, oracle):
    """The per-thread base case equals the reference recursion's leaves on an
    8-key window: largest of 8/4/2 the config sends to a network, else 1."""
    for c in ns.config_registry():
        a = oracle.generate_i32("random", 8, 1)
        _, st = oracle.merge_sort(a, c.name, stats=True)
        hits = [w for w in range(9) if st.network_hits[w]]
        want = hits[0] if hits else 1
        assert ns.leaf_width(c) == want, c.name


def test_config_constructors(ns):
    with pytest.raises(ValueError):
        ns.make_fixed_config("bad", [2])
    with pytest.raises(ValueError):
        ns.make_fixed_config("bad", [9])
    with pytest.raises(ValueError):
        ns.make_varsort_config("bad", 6)
    assert ns.make_fixed_config("x", [3, 4, 5]).width_mask == ns.find_config("3To5").width_mask


def test_status_strings(ns):
    L = ns.lib()
    assert L.ns_status_string(0) == b"ok"
    assert L.ns_status_string(1) == b"invalid argument"
    assert L.ns_status_string(99) == b"unknown status"
    assert L.ns_version() >= 100


def test_no_cpu_fallback(ns):
    """Without a GPU the compute entry points fail loudly instead of sorting
    on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("host has a GPU")
    a = np.arange(100, 0, -1, dtype=np.int32)
    with pytest.raises(ns.NetsortError):
        ns.optimized_merge_sort(a, ns.find_config("6To8"))
    assert a[0] == 100  # untouched


def test_temp_bytes_queries(ns):
    L = ns.lib()
    assert L.ns_merge_sort_temp_bytes(100) == 0          # one CTA, on chip
    assert L.ns_merge_sort_temp_bytes(1 << 20) >= 4 << 20
    assert L.ns_quick_sort_temp_bytes(1 << 20) >= 4 << 20
    assert L.ns_merge_runs_temp_bytes(1000, 1) == 0


def test_merge_sort_dispatch_stats_match_reference(oracle):
    """DispatchStats (hybrid.hpp:18-34) of the reference's merge sort, from the
    library's host-side recursion-shape count, equal the counters the
    reference records (oracle/_ref) and the oracle's own — every config."""
    import paper_2503_05934_b200 as ns
    for name, mask, vs in oracle.REGISTRY:
        cfg = ns.find_config(name)
        for n in (1, 2, 3, 7, 8, 9, 13, 100, 1000, 25000, 100000, 123457):
            st = ns.merge_sort_dispatch_stats(n, cfg)
            _, ost = oracle.merge_sort(oracle.generate_i32("random", n, 5), name, stats=True)
            assert st.network_hits == list(ost.network_hits), (name, n)
            assert st.merges == ost.merges and st.max_depth == ost.max_depth
            assert st.partitions == 0
            if oracle.ref_available():
                rs = np.zeros(12, np.uint64)
                a = oracle.generate_i32("random", n, 5)
                oracle.ref().ref_merge_sort_i32(a, n, mask, vs, rs.ctypes.data)
                assert st.network_hits == rs[:9].tolist() and st.merges == rs[9]
                assert st.max_depth == rs[11]
    # 6To8 fires no network at n = 10,000; w8 x 2^21 at 2^24
    assert ns.merge_sort_dispatch_stats(10_000, ns.find_config("6To8")).total_network_hits() == 0
    big = ns.merge_sort_dispatch_stats(1 << 24, ns.find_config("6To8"))
    assert big.network_hits[8] == 2_097_152 and big.max_depth == 22
    assert ns.merge_sort_dispatch_stats(0, ns.find_config("6To8")).max_depth == 0


def test_host_generator_matches_oracle_and_golden(ns, oracle, golden):
    """ns.generate / ns.generate_batch (the library's host generator, row
    a19) reproduce the oracle's streams and the golden input digests (the
    reference's datagen.cpp:18-50 narrowed to int32; int64 unnarrowed)."""
    import hashlib
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    for dist in ("random", "sorted", "nearly_sorted"):
        for n in (0, 1, 2, 3, 1000, 65537):
            assert np.array_equal(ns.generate(dist, n, 42), oracle.generate_i32(dist, n, 42))
            assert np.array_equal(ns.generate(dist, n, 7, dtype=np.int64),
                                  oracle.generate_i64(dist, n, 7))
    seen = 0
    for c in golden["cases"]:
        if c["n"] <= 1_000_000 and c["seed"] == 42:
            assert sha(ns.generate(c["dist"], c["n"], c["seed"])) == c["input_sha256"], c
            seen += 1
    assert seen >= 14
    offs, keys = ns.generate_batch(40, 7)
    assert offs.tolist() == golden["small_batch"]["offsets"]
    o2, k2 = oracle.generate_batch_i32(40, 7)
    assert np.array_equal(keys, k2)
    with pytest.raises(ValueError):
        ns.generate("nearly_sorted", 10, 1, p=1.5)
