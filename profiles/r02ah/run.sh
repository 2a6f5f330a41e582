#!/bin/bash
# Re-entry check after the container was re-created: full GPU suite, smoke, c1/c3 bench.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ah; mkdir -p $O
timeout 1800 python -m pytest tests -x -q -p no:cacheprovider -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
for c in c1 c3; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
