#!/bin/bash
# Row-Σ² pass with L2 eviction hints (A evict-first, X evict-last): DRAM bytes and step time, on / off.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ad; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_umma.py -x -q -p no:cacheprovider -k "rowsq" > $O/pytest_rowsq.log 2>&1; echo "rc=$?" >> $O/pytest_rowsq.log
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
BCUR_ROWSQ_NO_L2HINT=1 timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3_nohint.json 2> $O/bench_c3_nohint.err
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3_b.json 2> $O/bench_c3_b.err
for v in 0 1; do
  BCUR_ROWSQ_NO_L2HINT=$v timeout 900 ncu --kernel-name regex:k_umma2_rowsq -c 1 --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --csv python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/ncu_rowsq_nohint$v.csv 2> $O/ncu_rowsq_nohint$v.err
done
