#!/bin/bash
# torchrun launch path of bench.py at N=1 (both arms), as the driver's scaling step runs it.
mkdir -p gpurun_out/r01g
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 \
  bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/r01g/torchrun_n1.json 2> gpurun_out/r01g/torchrun_n1.err
echo "mine rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29532 \
  bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/r01g/torchrun_n1_ref.json 2> gpurun_out/r01g/torchrun_n1_ref.err
echo "ref rc=$?"
python bench.py > gpurun_out/r01g/bench_default.json 2> gpurun_out/r01g/bench_default.err
echo "default rc=$?"
tail -c 600 gpurun_out/r01g/torchrun_n1.json; tail -c 400 gpurun_out/r01g/torchrun_n1_ref.json
