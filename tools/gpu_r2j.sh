#!/bin/bash
# per-kernel launch list of the 7B step (ncu, gpu__time_duration only)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/r2_launch_bench.log 2>&1
echo rc=$?
python tools/launches.py gpurun_out/r2_launches.csv 2>&1 | tail -40
