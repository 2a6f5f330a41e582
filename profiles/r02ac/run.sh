#!/bin/bash
# Residual pass skips the selected blocks' tiles (their projected mass is their own norm); sketch
# correction weighted by the unskipped share of each component.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ac; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_umma.py -x -q -p no:cacheprovider > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
timeout 900 python -m pytest tests/test_gpu_zfullsize.py -x -q -p no:cacheprovider -k "c3" > $O/pytest_full.log 2>&1; echo "rc=$?" >> $O/pytest_full.log
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
BCUR_NO_KNOWN_COLS=1 timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3_noskip.json 2> $O/bench_c3_noskip.err
