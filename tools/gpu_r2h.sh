#!/bin/bash
# more sparse K1 shapes; attribution at the new default; ncu source capture of the optimistic k2_emit
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in base s5b6 s6b4 s5b7 s6b5; do
  lib=""; [ "$v" != base ] && lib="PULSE_LIB=$PWD/variants/$v.so"
  for sp in 0.99 0.999; do env $lib PULSE_K1_SHAPE=sparse timeout 300 python tools/k1_time.py $sp 2>&1 | tail -1 | sed "s/^/$v: /"; done
done | tee gpurun_out/r2_k1_variants4.txt
for x in 2 3 1; do PULSE_K1_EXPERIMENT=$x timeout 300 python tools/k1_time.py 0.99 2>&1 | tail -1; done | tee gpurun_out/r2_k1_attrib2.txt
timeout 900 ncu --set full --import-source on -k k2_emit --launch-skip 6 --launch-count 1 -f -o gpurun_out/r2_k2 python bench.py --steps 2 --warmup 3 --no-graph --no-e2e --no-cpu-baseline > gpurun_out/r2_ncu_k2.log 2>&1
echo "ncu rc=$?"
