#!/bin/bash
# Source-level ncu of the hi-only correction product (k_umma2_h3m<true, EPI_BASIS>) in a c3 step.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02bh; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_umma2_h3m' -c 2 \
  -o /tmp/h3m python bench.py --steps 1 --warmup 0 --e2e-steps 1 --no-cpu-baseline > $O/ncu.log 2>&1
ncu -i /tmp/h3m.ncu-rep --page source --csv --kernel-name regex:k_umma2_h3m 2>/dev/null | gzip > $O/h3m_source.csv.gz
ncu -i /tmp/h3m.ncu-rep --page details --csv 2>/dev/null | grep -i "stall\|warp cycles\|issue" | head -80 > $O/h3m_details.txt
