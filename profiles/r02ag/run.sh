#!/bin/bash
# Jacobi: rotation replay with a warp per V row pair (syncwarp between rounds), parallel eigenvalue
# ranking, the trailing no-op sweep skipped by an exact convergence check.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ag; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_alg1.py tests/test_gpu_dmma.py -x -q -p no:cacheprovider -m gpu > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
for c in c1 c2 c3; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
