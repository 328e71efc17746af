#!/bin/bash
# round-2 GPU batch: GPU suite per file (timeouts, host-memory watermark), K1 variants
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
: > gpurun_out/r2_pytest_gpu.log
for f in tests/test_*.py; do
  echo "== $f" >> gpurun_out/r2_pytest_gpu.log
  ( peak=0; while true; do u=$(free -m | awk 'NR==2{print $3}'); [ "$u" -gt "$peak" ] && peak=$u && echo $peak > gpurun_out/r2_mem_peak; sleep 1; done ) &
  mon=$!
  start=$(date +%s)
  timeout 900 python -m pytest $f -m gpu -q -p no:cacheprovider -x > gpurun_out/r2_pt_one.log 2>&1
  rc=$?
  kill $mon 2>/dev/null; wait $mon 2>/dev/null
  echo "rc=$rc secs=$(( $(date +%s) - start )) host_mem_peak_mb=$(cat gpurun_out/r2_mem_peak)" >> gpurun_out/r2_pytest_gpu.log
  tail -15 gpurun_out/r2_pt_one.log >> gpurun_out/r2_pytest_gpu.log
  cp gpurun_out/r2_pt_one.log "gpurun_out/r2_pt_$(basename $f .py).log"
done
grep -E "^==|rc=|passed|failed|error" gpurun_out/r2_pytest_gpu.log
for v in base s5 s6 s5b2; do
  lib=""; [ "$v" != base ] && lib="PULSE_LIB=$PWD/variants/$v.so"
  for sp in 0.99 0.9; do
    env $lib timeout 300 python tools/k1_time.py $sp 2>&1 | tail -1 | sed "s/^/$v: /"
  done
done | tee gpurun_out/r2_k1_variants.txt
for x in 0 2 3 1; do PULSE_K1_EXPERIMENT=$x timeout 300 python tools/k1_time.py 0.99 2>&1 | tail -1; done | tee gpurun_out/r2_k1_attrib.txt
