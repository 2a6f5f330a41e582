#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02p; mkdir -p $O
BCUR_LEAF_TIMING=1 timeout 300 python profiles/r02c/chol_bench.py > $O/chol_bench_timing3.log 2>&1
timeout 300 python profiles/r02c/chol_bench.py > $O/chol_bench3.log 2>&1
