#!/bin/bash
# Launch list of one c3 step at the current build (ncu gpu__time_duration, cold-cache, serialised).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02u; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
  python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
gzip -f $O/launches_c3.csv
