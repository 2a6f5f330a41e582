#!/bin/bash
# Sketch correction from the basis's interleaved fp16 split (no fp32 copy): c3-shaped parity, golden, bench.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02r; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_umma.py -x -q -p no:cacheprovider > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
timeout 900 python -m pytest tests/test_gpu_zfullsize.py -x -q -p no:cacheprovider -k c3 > $O/pytest_c3full.log 2>&1; echo "rc=$?" >> $O/pytest_c3full.log
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
