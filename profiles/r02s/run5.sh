#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02s; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_chol_persistent -s 18 -c 1 -o $O/chol_pers2 python profiles/r02c/chol_bench.py > $O/ncu2.log 2>&1
ncu -i $O/chol_pers2.ncu-rep --page source --csv --print-source sass > $O/chol_pers2_sass.csv 2>&1
ncu -i $O/chol_pers2.ncu-rep --page raw --csv > $O/chol_pers2_raw.csv 2>&1
gzip -f $O/chol_pers2_sass.csv
rm -f $O/chol_pers2.ncu-rep
