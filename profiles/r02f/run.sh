#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02f; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "explicit or forced or pythagoras" > $O/pytest_explicit.log 2>&1; echo "rc=$?" >> $O/pytest_explicit.log
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c3 --steps 5 --warmup 2 --no-cpu-baseline --noise 1e-6 --residual explicit > $O/bench_c3_explicit.json 2> $O/bench_c3_explicit.err
timeout 600 python bench.py --config c3 --steps 5 --warmup 2 --no-cpu-baseline --noise 1e-6 > $O/bench_c3_lownoise_auto.json 2> $O/bench_c3_lownoise_auto.err
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python profiles/r02f/san.py > $O/sanitizer_$tool.log 2>&1; echo "rc=$?" >> $O/sanitizer_$tool.log
done
