#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02i; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -q -p no:cacheprovider -k "cur or c4" > $O/pytest_cur.log 2>&1; echo "rc=$?" >> $O/pytest_cur.log
timeout 900 python -m pytest tests/test_gpu_zfullsize.py -q -p no:cacheprovider -k c4 > $O/pytest_c4full.log 2>&1; echo "rc=$?" >> $O/pytest_c4full.log
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
