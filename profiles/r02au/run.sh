#!/bin/bash
# The driver's command lines on the final build: default bench (c3, CPU baseline inside), the same
# under torchrun at N = 1, the reference arm (3 timed full CPU decompositions), c1/c2 with their CPU legs.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02au; mkdir -p $O
( time timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err ) 2> $O/bench_default.time
( time timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_torchrun.json 2> $O/bench_torchrun.err ) 2> $O/bench_torchrun.time
( time timeout 1500 python bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err ) 2> $O/bench_reference.time
for c in c1 c2; do timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
