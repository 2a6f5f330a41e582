#!/bin/bash
# Full-square Jacobi layout (conflict-free update phase), draw kernel state in shared memory, rowsq
# roofline accounting over the processed tiles: full GPU suite, c1-c4 bench, Jacobi A/B + phase clocks.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02av; mkdir -p $O
timeout 2400 python -m pytest tests -x -q -p no:cacheprovider -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for c in c3 c1 c2 c4; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
for c in c1 c2; do BCUR_JACOBI_PACKED_ONLY=1 timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_${c}_packed.json 2> $O/bench_${c}_packed.err; done
for c in c1 c2 c3 c4; do BCUR_JACOBI_TIMING=1 timeout 300 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | grep jacobi_packed | sort | uniq -c > $O/jacobi_clocks_$c.log; done
