#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_device.py tests/test_parity_configs.py tests/test_host_api.py tests/test_resident.py tests/test_fuzz_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_pt_q.log 2>&1
tail -3 gpurun_out/r2_pt_q.log
for w in c1 qwen2.5-1.5b qwen2.5-7b; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['ms_per_step'], d['value'], d['phases'], d['verified'])"; done
timeout 600 python bench.py --sparsity 0.999 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('0.999', d['ms_per_step'], d['value'], d['phases'], d['verified'])"
