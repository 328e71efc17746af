#!/bin/bash
# K1 bitmap staging, batched flush re-reads, L2 hints: correctness + timing
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_device.py tests/test_parity_configs.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_pt_k1v2.log 2>&1
tail -3 gpurun_out/r2_pt_k1v2.log
for h in 1 0; do for sp in 0.99 0.999 0.9999 0.9 0.95; do PULSE_K1_L2HINT=$h timeout 300 python tools/k1_time.py $sp 2>&1 | tail -1 | sed "s/^/hint=$h /"; done; done | tee gpurun_out/r2_k1v2_time.txt
for x in 2 1; do PULSE_K1_EXPERIMENT=$x timeout 300 python tools/k1_time.py 0.99 2>&1 | tail -1; done | tee -a gpurun_out/r2_k1v2_time.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['phases'], d['verified'])"
