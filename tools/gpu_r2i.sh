#!/bin/bash
# apply F5 (index, value) pairs + unstage without shuffles: correctness + bench
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_device.py tests/test_parity_configs.py tests/test_host_api.py tests/test_resident.py tests/test_fuzz_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_pt_f5.log 2>&1
tail -3 gpurun_out/r2_pt_f5.log
for r in 0 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --repr $r 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('repr $r', d['ms_per_step'], d['value'], d['phases'], d['verified'])"; done
