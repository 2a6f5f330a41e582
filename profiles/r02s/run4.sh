#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02s; mkdir -p $O
BCUR_LEAF_TIMING=1 timeout 300 python profiles/r02c/chol_bench.py 2>&1 | grep chol_persistent > $O/chol_timing3.log
BCUR_CHOL_HALF=1 BCUR_LEAF_TIMING=1 timeout 300 python profiles/r02c/chol_bench.py 2>&1 | grep chol_persistent > $O/chol_timing3h.log
timeout 300 python profiles/r02c/chol_bench.py > $O/chol_bench3.log 2>&1
BCUR_CHOL_HALF=1 timeout 300 python profiles/r02c/chol_bench.py > $O/chol_bench3h.log 2>&1
