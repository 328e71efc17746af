#!/bin/bash
# K1 deferral (count-only tickets written by K1b): correctness + density sweep
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_device.py tests/test_parity_configs.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_pt_defer.log 2>&1
tail -3 gpurun_out/r2_pt_defer.log
for shape in auto sparse dense dense2; do for sp in 0.99 0.97 0.95 0.9 0.862 0.5; do
  if [ $shape = auto ]; then e=""; else e="PULSE_K1_SHAPE=$shape"; fi
  env $e timeout 300 python tools/k1_time.py $sp 2>&1 | tail -1 | sed "s/^/$shape /"; done; done | tee gpurun_out/r2_k1_defer.txt
