#!/bin/bash
# Persistent blocked Cholesky + inverse (k_chol_persistent): DMMA/Cholesky tests, timing, parity, benches.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02o; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_dmma.py -x -q -p no:cacheprovider > $O/pytest_dmma.log 2>&1; echo "rc=$?" >> $O/pytest_dmma.log
timeout 300 python profiles/r02c/chol_bench.py > $O/chol_bench.log 2>&1
BCUR_CHOL_REC=1 timeout 300 python profiles/r02c/chol_bench.py > $O/chol_bench_rec.log 2>&1
BCUR_LEAF_TIMING=1 timeout 120 python profiles/r02e/leaf_timing.py > $O/leaf_timing.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -x -q -p no:cacheprovider > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
for c in c3 c4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
