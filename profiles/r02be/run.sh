#!/bin/bash
# Last check of the committed build: full GPU suite, smoke, default bench, c2 line.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02be; mkdir -p $O
timeout 2400 python -m pytest tests -x -q -p no:cacheprovider -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
( time timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err ) 2> $O/bench_default.time
timeout 600 python bench.py --config c2 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config c1 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
