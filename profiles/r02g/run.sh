#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02g; mkdir -p $O
timeout 600 python bench.py --config c3 --steps 5 --warmup 2 --no-cpu-baseline --residual explicit > $O/bench_c3_forced_explicit.json 2> $O/bench_c3_forced_explicit.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/ncu_c3.log 2>&1
