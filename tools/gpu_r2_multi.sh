#!/bin/bash
# round-2 multi-GPU on one box (run with gpurun --gpus N): bench both arms at N=1..G,
# NCCL gather check against the reference, pytest multi-GPU test
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
G=$(nvidia-smi -L | wc -l); echo "GPUs: $G"
for N in 1 2 4 8; do
  [ $N -gt $G ] && break
  if [ $N = 1 ]; then run="python"; else run="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2970$N"; fi
  timeout 900 $run bench.py --gpus $N --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_scale_n$N.json 2> gpurun_out/r2_scale_n$N.err
  echo "bench N=$N rc=$?"; tail -1 gpurun_out/r2_scale_n$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['ms_per_step'], d['value'], d.get('e2e',{}).get('value'), d['verified'])"
  timeout 600 $run bench.py --impl reference --gpus $N --steps 3 --warmup 1 > gpurun_out/r2_scale_ref_n$N.json 2> gpurun_out/r2_scale_ref_n$N.err
  echo "ref N=$N rc=$?"; tail -c 300 gpurun_out/r2_scale_ref_n$N.json
done
for N in 2 4; do
  [ $N -gt $G ] && break
  run="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2971$N"
  timeout 900 $run tools/check_shard.py qwen2.5-7b > gpurun_out/r2_gather_7b_n$N.log 2>&1
  echo "check_shard 7B N=$N rc=$?"; grep -E "repr|CHECK|check" gpurun_out/r2_gather_7b_n$N.log
done
timeout 900 python -m pytest tests/test_multi_gpu.py -m gpu -q -p no:cacheprovider 2>&1 | tail -3
