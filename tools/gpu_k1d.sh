timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for s in 0.9 0.99; do timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 --sparsity $s > gpurun_out/k1d_$s.json 2>&1; echo "$s rc=$?"; tail -1 gpurun_out/k1d_$s.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['encode_ms'], d['apply_ms'], d['frac_of_hbm'], d['verified'])"; done
