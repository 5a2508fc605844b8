# RECORD: k-way passes (NSB_KWAY) vs pairwise after the v5 merge loop (profiles/r01_kway_streaming_experiment.txt)
set -e
for k in 4 8; do NSB_KWAY=$k NSB_KWAY_MIN=20000 python -m pytest tests/test_gpu_parity.py -x -q -k "sizes or golden or every_config or duplicates or kway" 2>&1 | tail -1; done
for k in 0 4 8; do echo "== NSB_KWAY=$k"; NSB_KWAY=$k python tests/size_sweep.py --min=22 --max=30; done
