# K1 element-mode staging A/B: cooperative (default build) vs per-lane loop (variant), plus GPU tests
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for sp in 0.9 0.95 0.99; do
  timeout 300 python tools/k1_time.py $sp 2>&1 | tail -1 | sed 's/^/coop: /'
  PULSE_LIB=$PWD/paper_2602_03839_b200/libpulse_variant_loop.so timeout 300 python tools/k1_time.py $sp 2>&1 | tail -1 | sed 's/^/loop: /'
done
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 --sparsity 0.9 > gpurun_out/k1ab_09.json 2>/dev/null; tail -1 gpurun_out/k1ab_09.json | cut -c1-400
