#!/bin/bash
# K1b pipelined + dense2 defer threshold; apply 32-bit COO scan + cp.async without cvta: tests + sweep + bench
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_device.py tests/test_parity_configs.py tests/test_fuzz_parity.py tests/test_host_api.py tests/test_resident.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_pt_m.log 2>&1
tail -3 gpurun_out/r2_pt_m.log
for sp in 0.99 0.97 0.95 0.9 0.862 0.5; do timeout 300 python tools/k1_time.py $sp 2>&1 | tail -1; done | tee gpurun_out/r2_k1_m.txt
for sp in 0.99 0.999 0.9999 0.9; do timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --sparsity $sp 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sp', d['ms_per_step'], d['value'], d['phases'], d['verified'])"; done
