#!/bin/bash
# Round-2 evidence refresh at the session's starting HEAD: GPU suite, smoke, benches,
# launch list and one ncu --set full capture of the c3 step's tensor/streaming kernels.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02j; mkdir -p $O
nvidia-smi > $O/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
for c in c1 c2 c4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
  python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k 'regex:k_umma|k_block_sumsq|k_chol_inv_leaf|k_dgemm' -c 60 \
  -o $O/full_c3 python bench.py --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline > $O/ncu_full.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
