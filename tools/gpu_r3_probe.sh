#!/bin/bash
# apply range experiment (arall: 1024-entry ranges at every size) + C1 launch lists (graph replay)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for lib in "" "$PWD/variants/arall.so"; do
  for w in qwen2.5-7b qwen2.5-1.5b; do
    PULSE_LIB=$lib timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib##*/}', '$w', d['ms_per_step'], d['phases']['apply'], d['verified'])"
  done
done
timeout 600 python bench.py --workload c1 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', d['ms_per_step'], d['phases'], d['verified'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_launches_c1_graph.csv python bench.py --workload c1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launches.py gpurun_out/r3_launches_c1_graph.csv | grep -v "at::\|synth"
