#!/bin/bash
# Persistent Cholesky phase clocks + ncu of the persistent kernel (DMMA pipe use) at w = 4096.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02p; mkdir -p $O
BCUR_LEAF_TIMING=1 timeout 300 python profiles/r02c/chol_bench.py > $O/chol_bench_timing2.log 2>&1
timeout 300 python profiles/r02c/chol_bench.py > $O/chol_bench2.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_chol_persistent -s 18 -c 1 -o $O/chol_pers python profiles/r02c/chol_bench.py > $O/ncu.log 2>&1
ncu -i $O/chol_pers.ncu-rep --page raw --csv > $O/chol_pers_raw.csv 2>&1
rm -f $O/chol_pers.ncu-rep
