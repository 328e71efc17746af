# tests, then the bench at N=1, 2, 4 on one 4-GPU box (two N=4 runs)
tag=${1:-sc}
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${tag}_n1.json 2>/dev/null
for n in 2 4 4; do
  run="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$n"
  timeout 600 $run bench.py --gpus $n --no-cpu-baseline --no-e2e > gpurun_out/${tag}_n${n}_$RANDOM.json 2>/dev/null
done
for f in gpurun_out/${tag}_n*.json; do python -c "import json; d=json.loads(open('$f').read().strip().split(chr(10))[-1]); print('$f', d['n_gpus'], d['ms_per_step'], d['value'], d['encode_ms'], d['apply_ms'], d['phases']['k2_emit']['ms'], d['verified'])"; done
