# What the driver runs at N=2: both arms, default flags.
run="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29701"
timeout 900 $run bench.py --impl reference --gpus 2 --steps 10 --warmup 3 > gpurun_out/dl_ref.json 2> gpurun_out/dl_ref.err; echo "ref rc=$?"; cat gpurun_out/dl_ref.json | cut -c1-200
timeout 1200 $run bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/dl_pulse.json 2> gpurun_out/dl_pulse.err; echo "pulse rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/dl_pulse.json').read().strip().split(chr(10))[-1]); print(d['value'], d['ms_per_step'], d['config']['launch'], d['e2e']['value'], d['cpu_baseline']['value'], d['verified'])"
grep -c '^{' gpurun_out/dl_pulse.json
