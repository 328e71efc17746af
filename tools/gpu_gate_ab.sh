# A/B of the conditional-node gating at N=4 (two runs each)
run="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561"
for i in 1 2; do
  for g in 0 1; do
    PULSE_NO_GRAPH_GATE=$g timeout 600 $run bench.py --gpus 4 --no-cpu-baseline --no-e2e > gpurun_out/ab_g${g}_$i.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/ab_g${g}_$i.json').read().strip().split(chr(10))[-1]); print('nogate=$g', d['ms_per_step'], d['value'], d['encode_ms'], d['apply_ms'], d['phases']['k2_emit']['ms'])"
  done
done
