#!/bin/bash
# K1 two-shape staging (sparse 5x5 / dense 3x4): correctness + timing + bench
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_device.py tests/test_parity_configs.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_pt_k1cfg.log 2>&1
tail -3 gpurun_out/r2_pt_k1cfg.log
for shape in sparse dense; do for sp in 0.99 0.999 0.9999 0.95 0.9; do PULSE_K1_SHAPE=$shape timeout 300 python tools/k1_time.py $sp 2>&1 | tail -1 | sed "s/^/$shape /"; done; done | tee gpurun_out/r2_k1cfg_time.txt
for sp in 0.99 0.9; do timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --sparsity $sp 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sp', d['ms_per_step'], d['value'], d['phases'], d['verified'])"; done
