#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02d; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_dmma.py -q -p no:cacheprovider -x > $O/pytest_dmma.log 2>&1; echo "rc=$?" >> $O/pytest_dmma.log
timeout 300 python profiles/r02c/chol_bench.py > $O/chol_bench.log 2>&1
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/chol_launches.csv python profiles/r02c/chol_bench.py > $O/ncu_chol.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chol_inv_leaf -s 10 -c 1 -o $O/leaf python profiles/r02c/chol_bench.py > $O/ncu_leaf.log 2>&1
