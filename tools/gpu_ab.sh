#!/bin/bash
# A/B of library variants on the bench (apply phase + step), 2 rounds each, interleaved
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for round in 1 2; do
for v in ${VARIANTS:-head}; do
  for w in ${WORKLOADS:-qwen2.5-7b c1}; do
    PULSE_LIB=$PWD/variants/$v.so timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $EXTRA 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases']; print('$v', '$w', d['ms_per_step'], 'k1', p['k1_scan']['ms'], 'k2', p['k2_emit']['ms'], 'apply', p['apply']['ms'], d['verified'])"
  done
done
done
