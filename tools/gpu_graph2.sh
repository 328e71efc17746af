tag=$1
run="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29681"
for r in 0 2; do
  timeout 180 $run bench.py --gpus 2 --no-cpu-baseline --no-e2e --repr $r > gpurun_out/${tag}_n2_r$r.json 2> gpurun_out/${tag}_n2_r$r.err; echo "N=2 r$r rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/${tag}_n2_r$r.json').read().strip().split(chr(10))[-1]); print(d['ms_per_step'], d['value'], d['config']['launch'], d['verified'])"; grep -i "graph capture" gpurun_out/${tag}_n2_r$r.err | head -2
done
