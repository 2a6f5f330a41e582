#!/bin/bash
# One-accumulator CTA-pair 3xFP16 products (k_umma2_h3m, GEMM_FAST_ACC): parity incl. full-size c3/c4, benches.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02z; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_umma.py -x -q -p no:cacheprovider > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
timeout 900 python -m pytest tests/test_gpu_zfullsize.py -x -q -p no:cacheprovider -k "c3 or c4" > $O/pytest_full.log 2>&1; echo "rc=$?" >> $O/pytest_full.log
for c in c4 c3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  BCUR_UMMA_NO_FAST_ACC=1 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_${c}_nofast.json 2> $O/bench_${c}_nofast.err
done
