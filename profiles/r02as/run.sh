#!/bin/bash
# fp32 SPLIT/BASIS epilogues of the one-accumulator pair product; double-angle Jacobi rotation:
# parity (umma, parity, golden, full-size c3/c4, dmma, alg1), c1-c4 bench, Jacobi phase clocks.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02as; mkdir -p $O
timeout 2400 python -m pytest tests/test_gpu_umma.py tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_zfullsize.py tests/test_gpu_dmma.py tests/test_alg1.py -x -q -p no:cacheprovider -m gpu -k "not c5" > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
for c in c3 c1 c2 c4; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
for c in c1 c2 c3; do BCUR_JACOBI_TIMING=1 timeout 300 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | grep jacobi_packed | sort | uniq -c > $O/jacobi_clocks_$c.log; done
