"""Bounds-checked build over every kernel family — the stand-in for the
sanitizer CI of SURVEY.md §5 (memcheck / racecheck / synccheck in place of
the reference's debug asserts, networks.hpp:36, 134, 153 and hybrid.hpp:107,
124, 161, 189, 202).  compute-sanitizer is closed on this GPU pool (runs under
it have left GPUs needing a reset), so:

  - libnetsort_b200_checked.so is the same sources built with NSB_CHECKED=1:
    every data-dependent index of the hot kernels is checked on the device
    (merge cursors against their slice + sentinel pad in the tile sort, the
    merge pass and the pointer-pair merge; staged slice extents and
    merge-path splits; bucket ids, scatter positions and work-list capacities
    of the quick sort; the batch kernel's staged arrays) and a failed check
    traps;
  - tests/cpp/checked_cases.cpp drives it through the C ABI at small sizes
    (one-CTA and tiled merge sorts, int32 / int64, quick sort at one and two
    partition levels with sorted and duplicate-heavy input, the base-case
    batch valid and invalid, segmented sorts, key-value sort, argsort, run
    merges, the pointer-pair merge, the host-span path) with guard zones
    around every device buffer, poisoned scratch and a std::sort check;
  - the run-time knobs force the rarer paths at those sizes: the separate
    partition kernels (NSB_FUSED_MAX=0), the search without block samples
    (NSB_SAMPLES=0), the thread-per-tile partition (NSB_PART_WARP_MAX=0) and
    launches without programmatic dependent launch (NSB_PDL=0).
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "checked_cases.cpp")
BIN = os.path.join(ROOT, "build", "checked_cases")


def build_binary():
    from paper_2503_05934_b200 import _lib
    if not os.path.exists(_lib.CHECKED_LIB_PATH):
        _lib.build(checked=True)
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    libdir = os.path.dirname(_lib.CHECKED_LIB_PATH)
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    "-I", "/usr/local/cuda/include", SRC, "-o", BIN, "-L", libdir,
                    "-l:libnetsort_b200_checked.so", f"-Wl,-rpath,{libdir}",
                    "-L/usr/local/cuda/lib64", "-lcudart"], check=True)
    return BIN


def test_checked_driver_builds_and_links_the_checked_library():
    b = build_binary()
    out = subprocess.run(["ldd", b], capture_output=True, text=True)
    assert "libnetsort_b200_checked.so" in out.stdout


def test_checked_build_has_the_checks_and_default_build_does_not():
    from paper_2503_05934_b200 import _lib
    build_binary()
    strings = lambda p: subprocess.run(["strings", p], capture_output=True, text=True).stdout  # noqa: E731
    assert "NSB_DCHECK failed" in strings(_lib.CHECKED_LIB_PATH)
    assert "NSB_DCHECK failed" not in strings(_lib.LIB_PATH)


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{}, {"NSB_FUSED_MAX": "0"},
                                 {"NSB_FUSED_MAX": "0", "NSB_SAMPLES": "0"},
                                 {"NSB_FUSED_MAX": "0", "NSB_PART_WARP_MAX": "0"},
                                 {"NSB_PDL": "0"}],
                         ids=["default", "partition-kernels", "no-block-samples",
                              "thread-partition", "no-pdl"])
def test_checked_build_all_kernels(env):
    b = build_binary()
    e = dict(os.environ)
    e.update(env)
    out = subprocess.run([b], capture_output=True, text=True, timeout=900, env=e)
    text = out.stdout + out.stderr
    assert "NSB_DCHECK failed" not in text, text[-4000:]
    assert out.returncode == 0, text[-4000:]
    assert "PASSED" in out.stdout, text[-4000:]


@pytest.mark.gpu
def test_checked_build_traps_on_a_failed_check():
    """Negative control: the checked library's self-test kernel fails an
    NSB_DCHECK on purpose; the launch must trap and the message must name the
    condition (so a green run above means the checks ran and held)."""
    import sys
    from paper_2503_05934_b200 import _lib
    build_binary()
    code = ("import ctypes, sys; L = ctypes.CDLL(sys.argv[1]); "
            "r = L.ns_checked_selftest(); print('status', r); sys.stdout.flush()")
    out = subprocess.run([sys.executable, "-c", code, _lib.CHECKED_LIB_PATH],
                         capture_output=True, text=True, timeout=120)
    text = out.stdout + out.stderr
    assert "NSB_DCHECK failed" in text and "i < bound" in text, text[-3000:]
    assert "status 2" in text, text[-3000:]  # NS_ERR_CUDA


def test_selftest_symbol_only_in_checked_build():
    from paper_2503_05934_b200 import _lib
    build_binary()
    nm = lambda p: subprocess.run(["nm", "-D", p], capture_output=True, text=True).stdout  # noqa: E731
    assert "ns_checked_selftest" in nm(_lib.CHECKED_LIB_PATH)
    assert "ns_checked_selftest" not in nm(_lib.LIB_PATH)
