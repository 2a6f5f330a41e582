#!/bin/bash
# Small reads through the pinned read area (d2h, chol_any): full GPU suite, smoke, c1-c4 bench.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ax; mkdir -p $O
timeout 2400 python -m pytest tests -x -q -p no:cacheprovider -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
for c in c2 c1 c3 c4; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 600 python tools/timeline.py --config c2 --steps 2 --warmup 3 --top 10 --json $O/timeline_c2.json --list $O/step_c2.txt > $O/timeline_c2.log 2>&1
