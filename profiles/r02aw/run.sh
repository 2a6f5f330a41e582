#!/bin/bash
# c4 per-kernel step list (18 ms of its 55 ms step carry no ProfScope class).
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02aw; mkdir -p $O
timeout 600 python tools/timeline.py --config c4 --steps 2 --warmup 2 --top 12 --json $O/timeline_c4.json --list $O/step_c4.txt > $O/timeline_c4.log 2>&1
