#!/bin/bash
# configs: C1 / C2 bench lines (both arms), C1 launch list, e2e stage laps, upscale + helpers tests
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_host_api.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
for w in c1 qwen2.5-1.5b; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 3 > gpurun_out/r2_cfg_$w.json 2> gpurun_out/r2_cfg_$w.err
  echo "$w rc=$?"; tail -1 gpurun_out/r2_cfg_$w.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['phases'], d['e2e']['value'], d['cpu_baseline']['value'], d['parity_vs_reference'], d['verified'])"
  timeout 600 python bench.py --impl reference --workload $w --steps 3 --warmup 1 > gpurun_out/r2_cfg_${w}_ref.json 2>/dev/null; tail -c 200 gpurun_out/r2_cfg_${w}_ref.json
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c1.csv python bench.py --workload c1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
python tools/launches.py gpurun_out/r2_launches_c1.csv | grep -v "at::\|synth"
PULSE_TIMING=1 timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline 2> gpurun_out/r2_e2e_timing.err > gpurun_out/r2_e2e_timing.json
grep "pulse timing\|\[pulse" gpurun_out/r2_e2e_timing.err | tail -40
