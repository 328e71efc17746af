#!/bin/bash
# dense K1 shapes (records only vs element mode) at 90/95/97%
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for v in base d3b3r2k d2b3r2k d2b4r1k d2b4el; do
  lib=""; [ "$v" != base ] && lib="PULSE_LIB=$PWD/variants/$v.so"
  for sp in 0.9 0.95 0.97; do env $lib PULSE_K1_SHAPE=dense timeout 300 python tools/k1_time.py $sp 2>&1 | tail -1 | sed "s/^/$v: /"; done
done | tee gpurun_out/r2_k1_dense.txt
timeout 900 ncu --set full --import-source on -k regex:"k2_emit|f_stream" --launch-skip 8 --launch-count 4 -f -o gpurun_out/r2_k2f5 python bench.py --steps 2 --warmup 3 --no-graph --no-e2e --no-cpu-baseline > gpurun_out/r2_ncu_k2f5.log 2>&1
echo "ncu rc=$?"
