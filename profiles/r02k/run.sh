#!/bin/bash
# Sync-free power-iteration orthonormalization + fused basis epilogues: parity, benches, launch list.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02k; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_umma.py -x -q -p no:cacheprovider > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
for c in c3 c4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
  python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
gzip -f $O/launches_c3.csv
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_umma2_rowsq' -c 1 \
  -o $O/full_rowsq python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > $O/ncu_full.log 2>&1
ncu -i $O/full_rowsq.ncu-rep --page raw --csv > $O/full_rowsq_raw.csv 2>&1
ls -la $O > $O/ls.txt
