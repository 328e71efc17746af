# Final confirmation on a 4-GPU box: all representations at N=1, the sparsity sweep, and N=2 / N=4.
tag=${1:-fin}
for r in 0 1 2; do
  CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e --repr $r > gpurun_out/${tag}_n1_r$r.json 2>/dev/null
done
for sp in 0.9 0.999 0.9999; do
  CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --sparsity $sp > gpurun_out/${tag}_sweep_$sp.json 2>/dev/null
done
for n in 2 2 4 4; do
  run="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2959$n"
  timeout 600 $run bench.py --gpus $n --no-cpu-baseline --no-e2e > gpurun_out/${tag}_n${n}_$RANDOM.json 2>/dev/null
done
for f in gpurun_out/${tag}_*.json; do python -c "import json; d=json.loads(open('$f').read().strip().split(chr(10))[-1]); print('$f', d['n_gpus'], d['config']['representation'], d['config']['sparsity'], d['ms_per_step'], d['value'], d['frac_of_hbm'], d['apply_ms'], d['verified'])"; done
