#!/bin/bash
# r02b: DMMA fp64 products + recursive Cholesky/inverse (no cuBLAS); rowsq diagnosis
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02b; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_dmma.py -q -p no:cacheprovider -x > $O/pytest_dmma.log 2>&1; echo "rc=$?" >> $O/pytest_dmma.log
timeout 600 python profiles/r02b/diag_rowsq.py > $O/diag_rowsq.log 2>&1
for c in c1 c2 c3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
