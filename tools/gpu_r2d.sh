#!/bin/bash
# K1 staging variants round 2 + ncu source captures of k1_tma, k2_emit, f_stream
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in base s4b4s s4b5 s4b6 s5b4 s5b5 s3b6; do
  lib=""; [ "$v" != base ] && lib="PULSE_LIB=$PWD/variants/$v.so"
  for sp in 0.99 0.999 0.9999 0.9; do
    env $lib timeout 300 python tools/k1_time.py $sp 2>&1 | tail -1 | sed "s/^/$v: /"
  done
done | tee gpurun_out/r2_k1_variants3.txt
timeout 600 ncu --set full --import-source on -k k1_tma --launch-skip 2 --launch-count 1 -f -o gpurun_out/r2_k1 python tools/k1_time.py 0.99 > gpurun_out/r2_ncu_k1.log 2>&1
echo "ncu k1 rc=$?"
timeout 900 ncu --set full --import-source on -k regex:"f_stream|k2_emit" --launch-skip 9 --launch-count 3 -f -o gpurun_out/r2_k2_apply python bench.py --steps 2 --warmup 3 --no-graph --no-e2e --no-cpu-baseline > gpurun_out/r2_ncu_k2a.log 2>&1
echo "ncu k2/apply rc=$?"
ls -la gpurun_out/*.ncu-rep
