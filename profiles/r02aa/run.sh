#!/bin/bash
# Evidence at the session's mid-point: smoke, launch list of a c3 step, ncu --set full of the
# step's tensor / streaming / factorization kernels (exported to CSV on the box).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02aa; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 300 python -m pytest tests/test_gpu_umma.py -q -p no:cacheprovider > $O/pytest_umma.log 2>&1; echo "rc=$?" >> $O/pytest_umma.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
  python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
gzip -f $O/launches_c3.csv
timeout 1800 ncu --set full --import-source on --clock-control none \
  -k 'regex:k_umma2_rowsq|k_umma2_h3|k_chol_persistent|k_block_sumsq<float>|k_umma<' -c 12 \
  -o $O/full_c3 python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline > $O/ncu_full.log 2>&1
ncu -i $O/full_c3.ncu-rep --page raw --csv > $O/full_c3_raw.csv 2>&1
gzip -f $O/full_c3_raw.csv
ls -la $O/full_c3.ncu-rep >> $O/ncu_full.log 2>&1
mv $O/full_c3.ncu-rep /tmp/ 2>/dev/null
