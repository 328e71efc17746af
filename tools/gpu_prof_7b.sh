#!/bin/bash
# 7B 99% launch list (eager) + full ncu captures of F1s, F5 and k2_emit with SASS source pages
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r3_launches_7b.csv $B > /dev/null 2>&1
python tools/launches.py gpurun_out/r3_launches_7b.csv | grep -v "at::\|synth"
for k in "f_stream" "k2_emit"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 2 -o gpurun_out/r3_$k $B > /dev/null 2>&1; echo "$k rc=$?"
  ncu -i gpurun_out/r3_$k.ncu-rep --page details > gpurun_out/r3_$k.details.txt 2>&1
  ncu -i gpurun_out/r3_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/r3_$k.sass.csv 2>&1
done
ls -la gpurun_out/r3_*
