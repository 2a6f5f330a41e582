#!/bin/bash
# round-1 evidence run: GPU tests, bench lines (c1-c5, reference arm), ncu launch list + full capture (c3)
mkdir -p gpurun_out/r01b
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r01b/pytest_gpu.log 2>&1; tail -2 gpurun_out/r01b/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r01b/bench_c3.json 2> gpurun_out/r01b/bench_c3.err
for c in c1 c2 c4; do timeout 900 python bench.py --config $c > gpurun_out/r01b/bench_$c.json 2> gpurun_out/r01b/bench_$c.err; done
timeout 1200 python bench.py --config c5 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r01b/bench_c5.json 2> gpurun_out/r01b/bench_c5.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r01b/bench_c3_reference.json 2> gpurun_out/r01b/bench_c3_reference.err
timeout 300 python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r01b/pre_ncu.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01b/launches_c3.csv \
    python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r01b/launch_ncu.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_umma -c 14 -f -o gpurun_out/r01b/c3_umma_full \
    python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r01b/full_ncu.log 2>&1
echo done
