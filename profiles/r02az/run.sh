#!/bin/bash
# Spin-then-block stream wait (A/B via BCUR_SYNC_SPIN_US=0), the hybrid-Cholesky ABI test, odd-shape gather tests.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02az; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_dmma.py tests/test_gpu_parity.py tests/test_alg1.py tests/test_cli.py tests/test_cpp_api.py -x -q -p no:cacheprovider -m gpu > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
for c in c1 c2 c3; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  BCUR_SYNC_SPIN_US=0 timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_${c}_nospin.json 2> $O/bench_${c}_nospin.err
done
