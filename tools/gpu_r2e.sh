#!/bin/bash
# K1 bitmap staging: correctness + timing + attribution
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_device.py tests/test_parity_configs.py tests/test_host_api.py tests/test_resident.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_pt_k1v2.log 2>&1
tail -15 gpurun_out/r2_pt_k1v2.log
for sp in 0.99 0.999 0.9999 0.9 0.95; do timeout 300 python tools/k1_time.py $sp 2>&1 | tail -1; done | tee gpurun_out/r2_k1v2_time.txt
for x in 2 3 1; do PULSE_K1_EXPERIMENT=$x timeout 300 python tools/k1_time.py 0.99 2>&1 | tail -1; done | tee -a gpurun_out/r2_k1v2_time.txt
for x in 2 3; do PULSE_K1_EXPERIMENT=$x timeout 300 python tools/k1_time.py 0.9 2>&1 | tail -1; done | tee -a gpurun_out/r2_k1v2_time.txt
