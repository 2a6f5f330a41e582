#!/bin/bash
# Leaf stores only the upper triangle of X (R skipped when unused): full GPU suite, chol timing, benches.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02m; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_dmma.py -x -q -p no:cacheprovider > $O/pytest_dmma.log 2>&1; echo "rc=$?" >> $O/pytest_dmma.log
BCUR_LEAF_TIMING=1 timeout 120 python profiles/r02e/leaf_timing.py > $O/leaf_timing.log 2>&1
timeout 300 python profiles/r02c/chol_bench.py > $O/chol_bench.log 2>&1
for c in c3 c4 c1 c2; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
