#!/bin/bash
# Greedy: the frozen tail's picks in one launch and one read: parity + c2 bench.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bc; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_cli.py tests/test_cpp_api.py -x -q -p no:cacheprovider -m gpu > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
timeout 600 python bench.py --config c2 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config c2 --steps 20 --warmup 3 > $O/bench_c2_cpu.json 2> $O/bench_c2_cpu.err
