#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02e; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 microbench/dmma_rate.cu -o /tmp/dmma_rate && /tmp/dmma_rate > $O/dmma_rate.log 2>&1
BCUR_LEAF_TIMING=1 timeout 120 python profiles/r02e/leaf_timing.py > $O/leaf_timing.log 2>&1
