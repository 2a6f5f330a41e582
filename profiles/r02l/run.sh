#!/bin/bash
# CTA-pair 3×FP16 products (k_umma2_h3): parity and benches, with the single-CTA form beside it.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02l; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_umma.py -x -q -p no:cacheprovider > $O/pytest_umma.log 2>&1; echo "rc=$?" >> $O/pytest_umma.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -x -q -p no:cacheprovider > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
for c in c4 c3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  BCUR_UMMA_NO_H3_PAIR=1 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_${c}_nopair.json 2> $O/bench_${c}_nopair.err
done
