# tests + 7B and 1.5B bench lines + launch lists (quick A/B after a kernel change)
tag=${1:-q}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for wl in qwen2.5-7b qwen2.5-1.5b; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline --no-e2e > gpurun_out/${tag}_$wl.json 2>/dev/null; echo "$wl rc=$?"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/${tag}_${wl}_launches.csv python bench.py --workload $wl --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
done
