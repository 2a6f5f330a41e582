#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02c; mkdir -p $O
timeout 300 python profiles/r02c/chol_bench.py > $O/chol_bench.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "pythagoras or two_rank or planted or steep" > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/chol_launches.csv python profiles/r02c/chol_bench.py > $O/ncu_chol.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chol_inv_leaf -c 1 -o $O/leaf python profiles/r02c/chol_bench.py > $O/ncu_leaf.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dgemm -s 40 -c 1 -o $O/dgemm python profiles/r02c/chol_bench.py > $O/ncu_dgemm.log 2>&1
