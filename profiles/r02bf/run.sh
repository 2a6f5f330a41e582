#!/bin/bash
# Final-build evidence: ncu launch list of a c3 bench run and ncu --set full of the step's tensor /
# streaming / factorization kernels, summarized on the box (profiles/summarize_ncu.py).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bf; mkdir -p $O
timeout 600 python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > $O/bench_plain.json 2> $O/bench_plain.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
  python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 1800 ncu --set full --import-source on --clock-control none \
  -k 'regex:k_umma2_rowsq|k_umma2_h3|k_chol_persistent|k_block_sumsq<float>|k_umma<|k_copy_segments|k_jacobi_packed' -c 24 \
  -o /tmp/full_c3 python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline > $O/ncu_full.log 2>&1
ls -la /tmp/full_c3.ncu-rep >> $O/ncu_full.log 2>&1
python profiles/summarize_ncu.py $O $O/launches_c3.csv /tmp/full_c3.ncu-rep c3 6 > $O/summarize.log 2>&1
ncu -i /tmp/full_c3.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/full_c3_raw.csv.gz
gzip -f $O/launches_c3.csv
