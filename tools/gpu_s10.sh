timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s10_bench.json 2>gpurun_out/s10_bench.err; echo "bench rc=$?"
timeout 300 python tools/pcie_bw.py > gpurun_out/s10_pcie.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/s10_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1; echo rc=$?
