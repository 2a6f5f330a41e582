#!/bin/bash
# Row-Σ² L2 hint = 1 (X evict-last only): DRAM bytes + step time; c1/c2 launch lists (latency-bound configs).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ae; mkdir -p $O
BCUR_ROWSQ_L2HINT=1 timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3_hint1.json 2> $O/bench_c3_hint1.err
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
BCUR_ROWSQ_L2HINT=1 timeout 900 ncu --kernel-name regex:k_umma2_rowsq -c 1 --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --csv python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/ncu_rowsq_hint1.csv 2> $O/ncu_rowsq_hint1.err
for c in c1 c2; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/launches_$c.csv 2> $O/launches_$c.err
  gzip -f $O/launches_$c.csv
done
