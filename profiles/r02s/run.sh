#!/bin/bash
# Jacobi (packed two-sided) round clocks at l = 60 (c3), 110 (c4); persistent Cholesky phase clocks.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02s; mkdir -p $O
BCUR_JACOBI_TIMING=1 BCUR_JACOBI_DEBUG=1 timeout 300 python bench.py --config c3 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $O/jac_c3.json 2> $O/jac_c3.err
BCUR_JACOBI_TIMING=1 BCUR_JACOBI_DEBUG=1 timeout 300 python bench.py --config c4 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $O/jac_c4.json 2> $O/jac_c4.err
