#!/bin/bash
# Full GPU suite + benches after: persistent Cholesky (batched RMW epilogue, 128x64 bulk items),
# fast final orth in the range finder, CTA-pair 3xFP16, fused basis epilogues.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02q; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for c in c3 c4 c1 c2; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 300 python profiles/r02c/chol_bench.py > $O/chol_bench.log 2>&1
