#!/bin/bash
# Thin-N (64 x 16 tile) DMMA products: dmma tests, c1/c2 parity + bench A/B, per-kernel step lists.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02an; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dmma.py tests/test_gpu_parity.py tests/test_golden.py tests/test_alg1.py -x -q -p no:cacheprovider -m gpu > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
for c in c1 c2; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  BCUR_DGEMM_NO_THIN=1 timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_${c}_nothin.json 2> $O/bench_${c}_nothin.err
done
for c in c1 c2 c3; do timeout 600 python tools/timeline.py --config $c --steps 2 --warmup 3 --top 10 --json $O/timeline_$c.json --list $O/step_$c.txt > $O/timeline_$c.log 2>&1; done
