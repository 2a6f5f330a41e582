#!/bin/bash
# round-1 evidence refresh: GPU tests, bench lines (c1-c5, reference arm), ncu launch list + full capture (c3)
O=gpurun_out/r01f
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
for c in c1 c2 c4; do timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 1200 python bench.py --config c5 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_c3_reference.json 2> $O/bench_c3_reference.err
timeout 300 python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > $O/pre_ncu.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
    python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > $O/launch_ncu.log 2>&1
timeout 1800 ncu --set full --import-source on --clock-control none -k regex:"k_umma|k_block_sumsq" -c 16 -f -o $O/c3_full \
    python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > $O/full_ncu.log 2>&1
echo done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
