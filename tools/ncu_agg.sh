B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:f_stream -s 2 -c 1 -o gpurun_out/agg $B > /dev/null 2>&1; echo "rc=$?"
ncu -i gpurun_out/agg.ncu-rep --page source --csv --print-source sass > gpurun_out/agg.sass.csv 2>&1
ncu -i gpurun_out/agg.ncu-rep --page details > gpurun_out/agg.details.txt 2>&1
