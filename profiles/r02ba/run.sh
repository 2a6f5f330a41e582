#!/bin/bash
# Greedy: steps against a basis of all m rows skip the CGS2 / rank test, frozen saturated steps take
# one read: parity (greedy, c2 full, two-rank, golden, CLI), c2 bench + step list.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ba; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_cli.py tests/test_cpp_api.py -x -q -p no:cacheprovider -m gpu > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
timeout 600 python bench.py --config c2 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python tools/timeline.py --config c2 --steps 2 --warmup 3 --top 10 --json $O/timeline_c2.json --list $O/step_c2.txt > $O/timeline_c2.log 2>&1
