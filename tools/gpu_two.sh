tag=$1
bash tools/gpu_round.sh $tag
run="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531"
for r in 0 1 2; do
  timeout 600 $run bench.py --gpus 2 --no-cpu-baseline --no-e2e --repr $r > gpurun_out/${tag}_n2_r$r.json 2> gpurun_out/${tag}_n2_r$r.err
  echo "N=2 repr $r rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/${tag}_n2_r$r.json').read().strip().split(chr(10))[-1]); print(d['ms_per_step'], d['value'], d['encode_ms'], d['apply_ms'], d['verified'])"
done
timeout 900 $run tools/check_shard.py qwen2.5-7b > gpurun_out/${tag}_shard_n2.log 2>&1; echo "check_shard rc=$?"; tail -2 gpurun_out/${tag}_shard_n2.log
