# partition policy A/B: warp-per-tile partition up to NSB_PART_WARP_MAX tiles,
# in-kernel (fused) search up to NSB_FUSED_MAX tiles
NSB_PART_WARP_MAX=1000000000 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_int64.py -x -q -k "sizes or distributions or adversarial or full or i64" 2>&1 | tail -1
for w in 0 4096 16384 65536; do
  for f in 4096 512 0; do
    NSB_PART_WARP_MAX=$w NSB_FUSED_MAX=$f python tests/size_sweep.py --min=18 --max=27 | python -c "
import sys,json
print('warp_max=$w fused_max=$f', ' '.join(f\"{json.loads(l)['log2n']}:{json.loads(l)['ms']*1000:.1f}\" for l in sys.stdin))"
  done
done
