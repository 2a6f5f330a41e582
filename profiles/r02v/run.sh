#!/bin/bash
# Double-buffered e2e (bcur_dmat_upload_async) next to the serial form; the async-upload test.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02v; mkdir -p $O
timeout 300 python -m pytest tests/test_io_bcur.py -x -q -p no:cacheprovider -m gpu > $O/pytest_io.log 2>&1; echo "rc=$?" >> $O/pytest_io.log
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --e2e-steps 6 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --e2e-steps 6 --e2e-serial --no-cpu-baseline > $O/bench_c3_serial.json 2> $O/bench_c3_serial.err
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --e2e-steps 6 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 --e2e-steps 6 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
