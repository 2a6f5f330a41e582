#!/bin/bash
# Two-leaf Cholesky through the recursion (w <= 256); Jacobi source-level ncu (c2's w = 64, c3's w = 60).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02af; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dmma.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
for c in c1 c2; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 ncu --kernel-name regex:k_jacobi_packed -c 1 --set full --import-source on --clock-control none \
  -o /tmp/jac_c2 python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > $O/ncu_jac_c2.log 2>&1
ncu -i /tmp/jac_c2.ncu-rep --page source --csv > $O/jac_c2_source.csv 2>/dev/null; gzip -f $O/jac_c2_source.csv
ncu -i /tmp/jac_c2.ncu-rep --page raw --csv > $O/jac_c2_raw.csv 2>/dev/null; gzip -f $O/jac_c2_raw.csv
ncu -i /tmp/jac_c2.ncu-rep --page details --csv > $O/jac_c2_details.csv 2>/dev/null
