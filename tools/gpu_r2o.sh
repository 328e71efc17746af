#!/bin/bash
# K2 1024-entry ranges, parallel helpers, experiment 4: tests + sweep benches
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_device.py tests/test_parity_configs.py tests/test_host_api.py tests/test_resident.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_pt_o.log 2>&1
tail -3 gpurun_out/r2_pt_o.log
PULSE_K1_EXPERIMENT=4 timeout 300 python tools/k1_time.py 0.99 2>&1 | tail -1
for sp in 0.99 0.9999; do timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --sparsity $sp 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sp', d['ms_per_step'], d['value'], d['phases'], d['verified'])"; done
