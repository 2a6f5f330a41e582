#!/bin/bash
# One-barrier ping-pong Jacobi (k_jacobi_pp), one-launch block gather (copy_segments), split-K for
# few-tile DMMA products, hybrid Cholesky memset trims: parity + c1/c2/c3 bench (Jacobi A/B) + lists.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ao; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_dmma.py tests/test_gpu_parity.py tests/test_golden.py tests/test_alg1.py tests/test_gpu_umma.py tests/test_gpu_zfullsize.py -x -q -p no:cacheprovider -m gpu -k "not c5" > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
for c in c1 c2 c3; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  BCUR_JACOBI_NO_PP=1 timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_${c}_nopp.json 2> $O/bench_${c}_nopp.err
done
for c in c1 c2 c3; do timeout 600 python tools/timeline.py --config $c --steps 2 --warmup 3 --top 10 --json $O/timeline_$c.json --list $O/step_$c.txt > $O/timeline_$c.log 2>&1; done
