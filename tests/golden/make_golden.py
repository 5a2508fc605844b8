"""Generate tests/golden/golden.json from the REFERENCE ITSELF.

Runs in the build container only (needs /root/reference to build
oracle/_ref/libnetsort_ref.so).  For every BASELINE.json configuration (and a
sweep of small cases over all 12 network configs) it records the SHA-256 of
the int32 input and of the reference's sorted output, so the GPU box — which
has no /root/reference — can check bit-exact parity without re-running the
reference.  Inputs come from the oracle generator (int32 narrowing of the
reference's SplitMix64 stream); the generator itself is
pinned to the reference's int64 stream in tests/test_oracle.py.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_sort(algo: str, a: np.ndarray, cfg: str) -> np.ndarray:
    R = O.ref()
    mask, vs = O.CONFIGS[cfg]
    out = a.copy()
    fn = R.ref_merge_sort_i32 if algo == "merge" else R.ref_quick_sort_i32
    fn(out, len(out), mask, vs, None)
    return out


def main() -> None:
    O.build()
    if not O.ref_available():
        sys.exit("oracle/_ref not built: /root/reference missing")
    cases = []
    t0 = time.time()

    def add(algo, cfg, dist, n, seed=42):
        a = O.generate_i32(dist, n, seed)
        out = ref_sort(algo, a, cfg)
        rec = {"algo": algo, "config": cfg, "dist": dist, "n": n, "seed": seed,
               "input_sha256": sha(a), "output_sha256": sha(out)}
        if n <= 64:
            rec["input"] = a.tolist()
            rec["output"] = out.tolist()
        cases.append(rec)

    # BASELINE config 1 and 3: merge sort 6To8
    add("merge", "6To8", "random", 10_000)
    for n in (25_000, 100_000, 1_000_000):
        for d in ("random", "sorted", "nearly_sorted"):
            add("merge", "6To8", d, n)
    # BASELINE config 4: quick sort 3To5
    for n in (10_000, 1_000_000, 16_777_216):
        for d in ("sorted", "random"):
            add("quick", "3To5", d, n)
    # every config x both algorithms on small and awkward sizes
    for cfg, _, _ in O.REGISTRY:
        for algo in ("merge", "quick"):
            for n in (0, 1, 2, 3, 5, 7, 8, 13, 33, 64, 501, 1000, 8193, 20000):
                add(algo, cfg, "random", n, seed=3000 + n)

    # int64: the reference's OWN generator stream
    # (generate(), datagen.cpp:18-50, full 64-bit values) sorted by the
    # reference's int64 instantiation — the type its benchmarks use.
    cases_i64 = []

    def add64(algo, cfg, dist, n, seed=42):
        a = np.empty(n, np.int64)
        O.ref().ref_generate_i64(O.KIND[dist], n, seed, 0.01, a)
        out = a.copy()
        mask, vs = O.CONFIGS[cfg]
        (O.ref().ref_merge_sort_i64 if algo == "merge" else O.ref().ref_quick_sort_i64)(
            out, n, mask, vs, None)
        rec = {"algo": algo, "config": cfg, "dist": dist, "n": n, "seed": seed,
               "input_sha256": sha(a), "output_sha256": sha(out)}
        if n <= 64:
            rec["input"] = [str(x) for x in a.tolist()]
            rec["output"] = [str(x) for x in out.tolist()]
        cases_i64.append(rec)

    for n in (10_000, 25_000, 100_000, 1_000_000, 16_777_216):
        for d in ("random", "sorted", "nearly_sorted"):
            add64("merge", "6To8", d, n)
    for n in (10_000, 1_000_000, 16_777_216):
        for d in ("sorted", "random"):
            add64("quick", "3To5", d, n)
    for cfg, _, _ in O.REGISTRY:
        for algo in ("merge", "quick"):
            for n in (0, 1, 2, 5, 8, 33, 1000, 20000):
                add64(algo, cfg, "random", n, seed=5000 + n)

    # BASELINE config 2: base-case batch, 2^24 ragged arrays
    offs, keys = O.generate_batch_i32(1 << 24, 42)
    out = keys.copy()
    O.ref().ref_sort_small_batch_i32(out, offs, len(offs) - 1)
    batch = {"num_arrays": 1 << 24, "seed": 42, "num_keys": int(len(keys)),
             "offsets_sha256": sha(offs), "input_sha256": sha(keys), "output_sha256": sha(out)}
    # a small batch spelled out, for the CPU tests
    so, sk = O.generate_batch_i32(40, 7)
    sout = sk.copy()
    O.ref().ref_sort_small_batch_i32(sout, so, len(so) - 1)
    small_batch = {"num_arrays": 40, "seed": 7, "offsets": so.tolist(), "input": sk.tolist(),
                   "output": sout.tolist()}

    # BASELINE config 4 segmented: 65,536 x 16,384; the reference takes ~95 s
    # for all of it, so the digest covers the first 1,024 segments (the GPU
    # test sorts the full batch and checks this prefix plus properties).
    nseg, seg = 1024, 16384
    a = O.generate_i32("random", nseg * seg, 42)
    out = a.copy()
    mask, vs = O.CONFIGS["3To5"]
    O.ref().ref_segmented_quick_sort_i32(out, nseg, seg, mask, vs)
    segmented = {"num_segments_checked": nseg, "full_num_segments": 65536, "seg_len": seg,
                 "seed": 42, "config": "3To5", "input_prefix_sha256": sha(a),
                 "output_prefix_sha256": sha(out)}

    # Reference KATs reproduced through oracle/_ref (test_datagen.cpp:25-35, 79-91)
    R = O.ref()
    kat = {"splitmix64": {str(s): [hex(R.ref_splitmix64_nth(s, k)) for k in range(3)]
                          for s in (0, 42)}}
    gold = {"generator": "oracle.generate_i32 (int32(next()>>33) | ramp | ramp+swaps)",
            "reference_build": "oracle/Makefile ref -> oracle/_ref/libnetsort_ref.so",
            "cases": cases, "cases_i64": cases_i64, "batch": batch, "small_batch": small_batch,
            "segmented": segmented, "kat": kat}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(gold, f, indent=1)
    print(f"wrote {path}: {len(cases)} cases in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
