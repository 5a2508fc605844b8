for t in 16384 32768; do
  echo "== NSB_TILE=$t"
  NSB_TILE=$t timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "sizes or distributions" 2>&1 | tail -1
  for n in 268435456 1073741824; do NSB_TILE=$t python tests/kind_profile.py merge $n | grep -E "call|merge_pass|tile"; done
  NSB_TILE=$t python tests/size_sweep.py --min=22 --max=30 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['log2n'], round(d['ms']*1000,1), d['sorted'])"
done
