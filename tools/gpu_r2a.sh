#!/bin/bash
# round-2 GPU batch: full GPU suite (parity at configs, fuzz), sanitizers, bench
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu.log
tail -30 gpurun_out/r2_pytest_gpu.log
for tool in memcheck synccheck racecheck; do
  extra=""; [ "$tool" != memcheck ] && extra="--small"
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize.py $extra > gpurun_out/r2_sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/r2_sanitize_$tool.log
  tail -5 gpurun_out/r2_sanitize_$tool.log
done
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
tail -c 4000 gpurun_out/r2_bench.json
