#!/bin/bash
# CholQR2 second-pass correction on one fp16 MMA (GEMM_HI_ONLY): parity + c3/c4 bench + timeline.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02aj; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_umma.py tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_zfullsize.py -x -q -p no:cacheprovider -m gpu -k "not c5" > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
for c in c3 c4; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
BCUR_UMMA_NO_HI_ONLY=1 timeout 600 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c3_nohi.json 2> $O/bench_c3_nohi.err
timeout 600 python tools/timeline.py --config c3 --steps 2 --warmup 3 --top 40 --json $O/timeline_c3.json > $O/timeline_c3.log 2>&1
