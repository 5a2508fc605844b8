# programmatic dependent launch: default (on up to 2^19 keys) vs always on vs off
for v in 1 2 0; do
  NSB_PDL=$v python tests/size_sweep.py --min=16 --max=27 | python -c "
import sys,json
print('pdl=$v', ' '.join(f\"{json.loads(l)['log2n']}:{json.loads(l)['ms']*1000:.1f}\" for l in sys.stdin))"
done
