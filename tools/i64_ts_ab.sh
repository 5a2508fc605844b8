# int64 tile sort variants (build/variants/*.so) x NSB_TILE64 (1 skewed <1024,8>, 2 padded <512,16>)
cp paper_2503_05934_b200/lib/libnetsort_b200.so /tmp/lib_orig.so
for v in build/variants/*.so; do
  cp "$v" paper_2503_05934_b200/lib/libnetsort_b200.so
  for t in 1 2; do
    echo "== $v NSB_TILE64=$t"
    NSB_TILE64=$t python -m pytest tests/test_gpu_int64.py -x -q -k "sizes or golden or extremes" 2>&1 | tail -1
    NSB_TILE64=$t python tests/kind_profile.py merge 268435456 i64 | grep -E "call|tile"
  done
done
cp /tmp/lib_orig.so paper_2503_05934_b200/lib/libnetsort_b200.so
