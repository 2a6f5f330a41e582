#!/bin/bash
# BASIS epilogue loads 8 columns' aux values per round trip; the fast-accumulator product test.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ab; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_umma.py tests/test_gpu_parity.py tests/test_golden.py -x -q -p no:cacheprovider > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
for c in c3 c4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
