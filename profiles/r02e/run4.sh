#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02e; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_dmma.py -q -p no:cacheprovider -x > $O/pytest_dmma4.log 2>&1; echo "rc=$?" >> $O/pytest_dmma4.log
BCUR_LEAF_TIMING=1 timeout 120 python profiles/r02e/leaf_timing.py > $O/leaf_timing4.log 2>&1
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3_4.json 2> $O/bench_c3_4.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -q -p no:cacheprovider -x > $O/pytest_parity4.log 2>&1; echo "rc=$?" >> $O/pytest_parity4.log
