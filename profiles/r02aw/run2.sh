#!/bin/bash
# Result downloads (pinned direct / pageable staged), block_cur out_u: tests, c4 bench, c3/c1 sanity.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02aw; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_alg1.py tests/test_cpp_api.py tests/test_cli.py tests/test_io_bcur.py tests/test_abi.py -x -q -p no:cacheprovider -m gpu > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
for c in c4 c3 c1; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 600 python tools/timeline.py --config c4 --steps 2 --warmup 2 --top 12 --json $O/timeline_c4b.json --list $O/step_c4b.txt > $O/timeline_c4b.log 2>&1
