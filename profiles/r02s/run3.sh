#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02s; mkdir -p $O
BCUR_LEAF_TIMING=1 timeout 300 python profiles/r02c/chol_bench.py 2>&1 | grep chol_persistent > $O/chol_timing2.log
