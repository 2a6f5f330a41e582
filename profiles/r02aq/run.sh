#!/bin/bash
# Full GPU suite + smoke + c1-c5 bench after: hybrid Cholesky, thin-N DMMA tiles, split-K for
# under-half-wave products, one-launch block gather, Jacobi index math.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02aq; mkdir -p $O
timeout 2400 python -m pytest tests -x -q -p no:cacheprovider -m gpu --durations=8 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
for c in c3 c1 c2 c4; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 1500 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/bench_c5.json 2> $O/bench_c5.err
for c in c1 c2 c3; do BCUR_JACOBI_TIMING=1 timeout 300 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | grep jacobi_packed | sort | uniq -c > $O/jacobi_clocks_$c.log; done
