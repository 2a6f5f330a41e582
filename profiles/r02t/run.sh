#!/bin/bash
# Persistent Cholesky with two 4-warp workers per CTA (bulk), whole-CTA critical items, idle TPC partner.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02t; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_dmma.py -x -q -p no:cacheprovider > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
for c in c3 c4 c1 c2; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 300 python profiles/r02c/chol_bench.py > $O/chol_bench.log 2>&1
BCUR_LEAF_TIMING=1 timeout 300 python profiles/r02c/chol_bench.py 2>&1 | grep chol_persistent > $O/chol_timing.log
