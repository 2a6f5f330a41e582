#!/bin/bash
# r02a: full GPU suite (incl. full-size c3/c4/c5 parity), then the c3 bench, then the CPU legs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/r02a/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02a/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02a/bench_c3.json 2> gpurun_out/r02a/bench_c3.err
echo "bench rc=$?" >> gpurun_out/r02a/bench_c3.err
timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02a/bench_c3_reference.json 2> gpurun_out/r02a/bench_c3_reference.err
echo "ref rc=$?" >> gpurun_out/r02a/bench_c3_reference.err
