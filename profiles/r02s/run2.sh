#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02s; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_dmma.py -x -q -p no:cacheprovider > $O/pytest_dmma.log 2>&1; echo "rc=$?" >> $O/pytest_dmma.log
timeout 300 python profiles/r02c/chol_bench.py > $O/chol_bench.log 2>&1
BCUR_LEAF_TIMING=1 timeout 300 python profiles/r02c/chol_bench.py 2>&1 | grep chol_persistent > $O/chol_timing.log
