#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02e; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 microbench/ifetch.cu -o /tmp/ifetch && /tmp/ifetch > $O/ifetch.log 2>&1
