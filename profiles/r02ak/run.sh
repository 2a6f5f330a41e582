#!/bin/bash
# Fewer host round trips (pinned upload ring, deferred reads: block_css 4 synchronizations,
# one read per CholQR2 decision): full GPU suite, c1/c2/c3 bench, c1/c3 timelines.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ak; mkdir -p $O
timeout 1800 python -m pytest tests -x -q -p no:cacheprovider -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for c in c1 c2 c3; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
for c in c1 c3; do timeout 600 python tools/timeline.py --config $c --steps 2 --warmup 3 --top 30 --json $O/timeline_$c.json > $O/timeline_$c.log 2>&1; done
