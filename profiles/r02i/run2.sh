#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02i; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_dmma.py -q -p no:cacheprovider -x > $O/pytest_dmma.log 2>&1; echo "rc=$?" >> $O/pytest_dmma.log
timeout 300 python profiles/r02c/chol_bench.py > $O/chol_bench.log 2>&1
for c in c3 c1 c2; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_${c}_2.json 2> $O/bench_${c}_2.err; done
