#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02h; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 microbench/dmma_rate.cu -o /tmp/dmma_rate && /tmp/dmma_rate > $O/dmma_rate2.log 2>&1
timeout 300 python -m pytest tests/test_gpu_dmma.py -q -p no:cacheprovider -x > $O/pytest_dmma2.log 2>&1; echo "rc=$?" >> $O/pytest_dmma2.log
BCUR_LEAF_TIMING=1 timeout 120 python profiles/r02e/leaf_timing.py > $O/leaf_timing2.log 2>&1
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3_2.json 2> $O/bench_c3_2.err
