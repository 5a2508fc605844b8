# partition kernel A/B: NSB_PART=3 (thread per tile) vs 4 (warp per tile)
for v in 3 4; do
  export NSB_PART=$v; echo "== NSB_PART=$v"
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_int64.py -x -q -k "sizes or distributions or adversarial or 2p31 or full" 2>&1 | tail -1
  for n in 16777216 268435456 1073741824; do python tests/kind_profile.py merge $n | grep -E "call|partition|merge_pass"; done
  python tests/size_sweep.py --min=22 --max=30 | python -c "
import sys,json
print(' '.join(f\"{json.loads(l)['log2n']}:{json.loads(l)['ms']*1000:.1f}\" for l in sys.stdin))"
done
