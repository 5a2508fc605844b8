# RECORD ONLY: the NSB_PIPE overlapped schedule was measured (profiles/r01_pipeline_overlap_experiment.txt)
# and removed: the merge pass is issue-heavy too, so the ALU-bound tile sort has nothing to overlap with.
set -e
NSB_PIPE=8 NSB_PIPE_MIN=20000 python -m pytest tests/test_gpu_parity.py tests/test_gpu_int64.py -x -q -k "sizes or golden or every_config or duplicates or extremes" 2>&1 | tail -2
for p in 0 4 8 16 32; do echo "== NSB_PIPE=$p"; NSB_PIPE=$p python tests/size_sweep.py --min=24 --max=30; done
