#!/bin/bash
# The tree as committed (after the reverted experiments): smoke, the quick GPU tests, default bench.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bj; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_umma.py tests/test_gpu_dmma.py tests/test_golden.py -x -q -p no:cacheprovider -m gpu > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
timeout 900 python bench.py --no-cpu-baseline --steps 20 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
