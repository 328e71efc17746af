tag=$1
for wl in c1 qwen2.5-7b; do
  for g in "" "--no-graph"; do
    timeout 300 python bench.py --workload $wl --no-cpu-baseline --no-e2e $g > gpurun_out/${tag}_$wl$g.json 2> gpurun_out/${tag}_$wl$g.err; echo "$wl $g rc=$?"
    python -c "import json; d=json.loads(open('gpurun_out/${tag}_$wl$g.json').read().strip().split(chr(10))[-1]); print(d['ms_per_step'], d['value'], d['config']['launch'], d['verified'])"; tail -2 gpurun_out/${tag}_$wl$g.err
  done
done
run="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29671"
for r in 0 2; do
  timeout 600 $run bench.py --gpus 2 --no-cpu-baseline --no-e2e --repr $r > gpurun_out/${tag}_n2_r$r.json 2> gpurun_out/${tag}_n2_r$r.err; echo "N=2 r$r rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/${tag}_n2_r$r.json').read().strip().split(chr(10))[-1]); print(d['ms_per_step'], d['value'], d['config']['launch'], d['verified'])"; grep -i "graph\|error" gpurun_out/${tag}_n2_r$r.err | head -3
done
