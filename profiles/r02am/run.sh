#!/bin/bash
# Hybrid Cholesky (one recursion level around two persistent launches, off-diagonal quarter on
# tcgen05 3xFP16) for >= 3072-wide fp32-class Grams: parity subset + c3/c4 A/B.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02am; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_umma.py tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_zfullsize.py -x -q -p no:cacheprovider -m gpu -k "not c5" > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
for c in c3 c4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  BCUR_CHOL_HYBRID=0 timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_${c}_nohyb.json 2> $O/bench_${c}_nohyb.err
done
