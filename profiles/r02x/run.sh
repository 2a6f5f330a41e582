#!/bin/bash
# Full GPU suite + benches (c1-c5) after: async uploads (double-buffered e2e), leaf column-copy
# load of symmetric diagonal blocks, triangular pair products without the wave barrier.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02x; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for c in c3 c4 c1 c2; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 1200 python bench.py --config c5 --steps 3 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 300 python profiles/r02c/chol_bench.py > $O/chol_bench.log 2>&1
