# C4 (BASELINE configs[3]): 32B shape sharded over 4 GPUs, multi-step patches k = 1/4/16; and the
# 32B bench step at N=4
run="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571"
timeout 1500 $run tools/multistep.py --workload qwen2.5-32b --k 1 4 16 > gpurun_out/c4_multistep_32b_n4.jsonl 2> gpurun_out/c4_multistep_32b_n4.err
echo "multistep rc=$?"; cut -c1-400 gpurun_out/c4_multistep_32b_n4.jsonl; tail -3 gpurun_out/c4_multistep_32b_n4.err
timeout 900 $run bench.py --gpus 4 --workload qwen2.5-32b --no-cpu-baseline --no-e2e > gpurun_out/c4_bench_32b_n4.json 2> gpurun_out/c4_bench_32b_n4.err
echo "bench rc=$?"; tail -1 gpurun_out/c4_bench_32b_n4.json | cut -c1-300
