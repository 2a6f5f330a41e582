#!/bin/bash
# quick round trip: GPU tests + c3/c4 (+ c5 when $1 == all) bench lines into gpurun_out/$TAG
TAG=${TAG:-q}
mkdir -p gpurun_out/$TAG
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/$TAG/gpu.log 2>&1; tail -3 gpurun_out/$TAG/gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/$TAG/c3.json 2> gpurun_out/$TAG/c3.err; tail -1 gpurun_out/$TAG/c3.err
timeout 300 python bench.py --config c4 --steps 3 --warmup 2 --e2e-steps 1 --no-cpu-baseline > gpurun_out/$TAG/c4.json 2> gpurun_out/$TAG/c4.err; tail -1 gpurun_out/$TAG/c4.err
if [ "$1" == "all" ]; then
for c in c1 c2; do timeout 300 python bench.py --config $c --e2e-steps 1 --no-cpu-baseline > gpurun_out/$TAG/$c.json 2> gpurun_out/$TAG/$c.err; tail -1 gpurun_out/$TAG/$c.err; done
timeout 900 python bench.py --config c5 --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/$TAG/c5.json 2> gpurun_out/$TAG/c5.err; tail -1 gpurun_out/$TAG/c5.err
fi
