"""the reference's own benchmark harness (measure_loop,
run_benchmark, compute_speedup, emit_csv — compiled unmodified by
oracle/Makefile) timing the B200 library through its sort_fn injection point
(oracle/harness_adapter.cpp -> oracle/_ref/harness_gpu)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HARNESS = os.path.join(ROOT, "oracle", "_ref", "harness_gpu")
CSV_HEADER = "algorithm,config,distribution,size,iterations,mean_ns,total_ns,speedup"


def _have_reference():
    return os.path.isdir("/root/reference/proj/include/netsort")


@pytest.mark.skipif(not _have_reference(), reason="reference tree absent (GPU box)")
def test_harness_links_against_the_library(oracle, ns):
    oracle.build(harness=True)
    assert os.path.exists(HARNESS)
    out = subprocess.run(["ldd", HARNESS], capture_output=True, text=True).stdout
    assert "libnetsort_b200.so" in out and "not found" not in out


@pytest.mark.gpu
def test_harness_runs_gpu_variants_in_reference_csv(tmp_path):
    if not os.path.exists(HARNESS):
        pytest.fail("oracle/_ref/harness_gpu not built (run __graft_entry__.build())")
    csv = tmp_path / "cells.csv"
    r = subprocess.run([HARNESS, "--sizes", "1000,20000", "--gpu-ms", "5", "--cpu-ms", "5",
                        "--csv", str(csv)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = csv.read_text().splitlines()
    assert lines[0] == CSV_HEADER
    # 2 sizes x 3 distributions x (2 CPU Classic + 24 GPU variants)
    assert len(lines) - 1 == 2 * 3 * 26
    gpu_rows = [l for l in lines[1:] if l.split(",")[1].startswith("B200:")]
    assert len(gpu_rows) == 2 * 3 * 24
    assert "speedup vs Classic" in r.stdout
