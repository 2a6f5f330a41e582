#!/bin/bash
mkdir -p gpurun_out/p2
timeout 60 scratch/tri_prof > gpurun_out/p2/tri_prof.txt 2>&1
timeout 300 python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/p2/pre.json 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_umma -c 2 -f -o gpurun_out/p2/c3_rf \
    python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/p2/c3_rf.log 2>&1
BCUR_UMMA_X3_PAIR=1 timeout 600 python bench.py --config c4 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/p2/pre4.json 2>&1 && \
BCUR_UMMA_X3_PAIR=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_umma2_x3 -c 1 -f -o gpurun_out/p2/c4_pair \
    python bench.py --config c4 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/p2/c4_pair.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_umma<\(bool\)0, \(int\)0, \(int\)2, \(bool\)1>" -c 1 -f -o gpurun_out/p2/c4_single \
    python bench.py --config c4 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/p2/c4_single.log 2>&1
echo done
