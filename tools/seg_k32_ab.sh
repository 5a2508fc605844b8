# NSB_SEG_K32 A/B: segmented batch and quick-sort bucket tiles as 16 vs 32 keys per thread
for v in 0 1; do
  export NSB_SEG_K32=$v; echo "== NSB_SEG_K32=$v"
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "quick or segmented or bucket" 2>&1 | tail -1
  python tools/seg_time.py
  for n in 1000000 16777216 67108864; do python tests/kind_profile.py quick $n | grep -E "call|bucket"; done
done
