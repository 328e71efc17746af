# Scaling run: bench at N = each argument (one box), no e2e/cpu legs.
tag=$1; shift
for N in "$@"; do
  if [ "$N" = 1 ]; then run="python"; else run="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N"; fi
  timeout 600 $run bench.py --gpus $N --no-cpu-baseline --no-e2e > gpurun_out/${tag}_n$N.json 2> gpurun_out/${tag}_n$N.err
  echo "N=$N rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/${tag}_n$N.json').read().strip().split(chr(10))[-1]); print(d['n_gpus'], d['ms_per_step'], d['value'], d['encode_ms'], d['apply_ms'], d['verified'])"
done
