#!/bin/bash
# K1 staging-shape variants + failing tests re-run + ncu source captures
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_device.py tests/test_parity_configs.py tests/test_fuzz_parity.py -m gpu -q -p no:cacheprovider > gpurun_out/r2_pt_fix.log 2>&1
tail -8 gpurun_out/r2_pt_fix.log
for v in base s4b4 s4b4s s3b4 s3b5; do
  lib=""; [ "$v" != base ] && lib="PULSE_LIB=$PWD/variants/$v.so"
  for sp in 0.99 0.9 0.999; do
    env $lib timeout 300 python tools/k1_time.py $sp 2>&1 | tail -1 | sed "s/^/$v: /"
  done
done | tee gpurun_out/r2_k1_variants2.txt
./tools/_bin/bw_probe | tee gpurun_out/r2_bw_probe.txt
