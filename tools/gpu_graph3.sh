run="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29691"
for g in "" "--no-graph" "" "--no-graph"; do
  timeout 180 $run bench.py --gpus 2 --no-cpu-baseline --no-e2e --repr 0 $g 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['config']['launch'], d['encode_ms'], d['apply_ms'])"
done
