# occupancy A/B over prebuilt libraries: base-case batch shape, int64 tile occupancy
cp paper_2503_05934_b200/lib/libnetsort_b200.so /tmp/lib_orig.so
for v in build/variants/*.so; do
  echo "== $v"; cp "$v" paper_2503_05934_b200/lib/libnetsort_b200.so
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "batch or network" 2>&1 | tail -1
  python tools/batch_time.py
  python tests/kind_profile.py merge 268435456 i64 | grep -E "call|tile"
  python tests/kind_profile.py quick 16777216 i64 | grep -E "call|bucket"
done
cp /tmp/lib_orig.so paper_2503_05934_b200/lib/libnetsort_b200.so
