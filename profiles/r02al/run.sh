#!/bin/bash
# NaN-safe Jacobi ranking (the deferred finiteness read of block_css): full GPU suite, smoke,
# c1/c2/c3/c4 bench, c1/c3 timelines.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02al; mkdir -p $O
CUDA_LAUNCH_BLOCKING=1 timeout 300 python profiles/r02al/nan_diag.py > $O/nan_diag.log 2>&1
timeout 2400 python -m pytest tests -x -q -p no:cacheprovider -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
for c in c1 c2 c3 c4; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
for c in c1 c2 c3; do timeout 600 python tools/timeline.py --config $c --steps 2 --warmup 3 --top 40 --json $O/timeline_$c.json > $O/timeline_$c.log 2>&1; done
