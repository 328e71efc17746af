#!/bin/bash
# A/B of library variants at N = 1, 2, 4 (run with gpurun --gpus 4): bench.py lines (no e2e / cpu baseline)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
G=$(nvidia-smi -L | wc -l)
for round in 1 2; do
for v in ${VARIANTS:-cur}; do
  for N in ${NS:-1 2 4}; do
    [ $N -gt $G ] && continue
    if [ $N = 1 ]; then run="python"; else run="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2975$N"; fi
    PULSE_LIB=$PWD/variants/$v.so timeout 600 $run bench.py --gpus $N --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases']; print('$v', 'N=$N', d['ms_per_step'], d['value'], 'k1', p['k1_scan']['ms'], 'k2', p['k2_emit']['ms'], 'apply', p['apply']['ms'], d['verified'])"
  done
done
done
