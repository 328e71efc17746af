#!/bin/bash
# launch list at 99.99% (escape path); K1b occupancy
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for sp in 0.862 0.5; do timeout 300 python tools/k1_time.py $sp 2>&1 | tail -1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_9999.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --sparsity 0.9999 > /dev/null 2>&1
python tools/launches.py gpurun_out/r2_launches_9999.csv | grep -v "at::\|synth"
