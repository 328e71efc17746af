timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/s8_bench.json 2>gpurun_out/s8_bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/s8_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_emit -s 4 -c 1 -o gpurun_out/s8_k2emit python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1; echo "full rc=$?"
ncu -i gpurun_out/s8_k2emit.ncu-rep --page details --csv > gpurun_out/s8_k2emit.details.csv 2>&1
ncu -i gpurun_out/s8_k2emit.ncu-rep --page source --csv --print-source sass > gpurun_out/s8_k2emit.sass.csv 2>&1
