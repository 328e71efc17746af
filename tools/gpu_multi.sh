# Multi-GPU validation on one box: bench (with e2e), sharded byte identity,
# reference arm under torchrun, and the 32B multi-step config.
tag=$1
for N in 2 4; do
  run="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N"
  timeout 900 $run bench.py --gpus $N --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_n$N.json 2> gpurun_out/${tag}_bench_n$N.err
  echo "bench N=$N rc=$?"; tail -c 600 gpurun_out/${tag}_bench_n$N.json
  timeout 600 $run bench.py --impl reference --gpus $N --steps 3 --warmup 1 > gpurun_out/${tag}_ref_n$N.json 2> gpurun_out/${tag}_ref_n$N.err
  echo "ref N=$N rc=$?"
  timeout 900 $run tools/check_shard.py qwen2.5-7b > gpurun_out/${tag}_shard_n$N.log 2>&1
  echo "check_shard N=$N rc=$?"; tail -3 gpurun_out/${tag}_shard_n$N.log
done
run="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29520"
timeout 1200 $run tools/multistep.py --workload qwen2.5-32b --k 1 4 16 > gpurun_out/${tag}_multistep_32b_n4.jsonl 2> gpurun_out/${tag}_multistep_32b_n4.err
echo "multistep 32B N=4 rc=$?"; cat gpurun_out/${tag}_multistep_32b_n4.jsonl
