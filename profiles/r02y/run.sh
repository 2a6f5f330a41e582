#!/bin/bash
# Full-square Jacobi (contiguous warp runs): round clocks, parity, benches.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02y; mkdir -p $O
BCUR_JACOBI_TIMING=1 BCUR_JACOBI_DEBUG=1 timeout 300 python bench.py --config c3 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > $O/jac_c3.out 2> $O/jac_c3.err
BCUR_JACOBI_TIMING=1 BCUR_JACOBI_DEBUG=1 timeout 300 python bench.py --config c4 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > $O/jac_c4.out 2> $O/jac_c4.err
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_ref_css.py tests/test_ref_leverage.py tests/test_alg1.py -x -q -p no:cacheprovider -m gpu > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
for c in c3 c4 c2 c1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
