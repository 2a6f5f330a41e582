#!/bin/bash
# After the flag-race fix in k_jacobi_packed: c4 x5 (20 steps + e2e), c2/c5-shaped parity, full GPU suite.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02at; mkdir -p $O
for i in 1 2 3 4 5; do timeout 600 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $O/c4_fixed_$i.json 2> $O/c4_fixed_$i.err; echo "rc=$?" >> $O/c4_fixed_$i.err; done
timeout 2400 python -m pytest tests -x -q -p no:cacheprovider -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for c in c3 c1 c2; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
