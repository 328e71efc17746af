# Sharded bench at N=2 (all representations) and N=4, plus the 2-rank byte-identity check.
tag=$1
for n in 2 4; do
  run="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n"
  reprs="0 1 2"; [ $n = 4 ] && reprs="0"
  for r in $reprs; do
    timeout 600 $run bench.py --gpus $n --no-cpu-baseline --no-e2e --repr $r > gpurun_out/${tag}_n${n}_r$r.json 2> gpurun_out/${tag}_n${n}_r$r.err
    echo "N=$n repr $r rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/${tag}_n${n}_r$r.json').read().strip().split(chr(10))[-1]); print(d['ms_per_step'], d['value'], d['encode_ms'], d['apply_ms'], d['verified'])"
  done
done
run="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541"
timeout 900 $run tools/check_shard.py qwen2.5-7b > gpurun_out/${tag}_shard_n2.log 2>&1; echo "check_shard rc=$?"; tail -2 gpurun_out/${tag}_shard_n2.log
