#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02s; mkdir -p $O
BCUR_LEAF_TIMING=2 timeout 300 python profiles/r02c/chol_bench.py > $O/chol_timing7.log 2>&1
