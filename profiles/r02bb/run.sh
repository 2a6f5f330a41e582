#!/bin/bash
# Final-build evidence: full GPU suite, smoke, the driver's command lines (default bench with its CPU
# leg; 20-step bench), c1-c5 bench lines, ncu launch list of a c3 run.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bb; mkdir -p $O
timeout 2400 python -m pytest tests -x -q -p no:cacheprovider -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
( time timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err ) 2> $O/bench_default.time
for c in c3 c1 c2 c4; do timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 1500 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
  python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
gzip -f $O/launches_c3.csv
