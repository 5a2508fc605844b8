for n in 1048576 16777216; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$n.csv python tests/prof_run.py merge $n > /dev/null 2>&1
done
