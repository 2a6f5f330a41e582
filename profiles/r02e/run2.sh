#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02e; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_dmma.py -q -p no:cacheprovider -x > $O/pytest_dmma2.log 2>&1; echo "rc=$?" >> $O/pytest_dmma2.log
BCUR_LEAF_TIMING=1 timeout 120 python profiles/r02e/leaf_timing.py > $O/leaf_timing2.log 2>&1
timeout 300 python profiles/r02c/chol_bench.py > $O/chol_bench2.log 2>&1
