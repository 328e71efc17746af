# Full ncu captures of the apply kernels (f_pass agg / apply / restore) of the 7B bench step, plus source pages.
tag=$1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:f_pass -s 6 -c 2 -o gpurun_out/${tag}_fpass $B > gpurun_out/${tag}_fpass.log 2>&1; echo "fpass rc=$?"
ncu -i gpurun_out/${tag}_fpass.ncu-rep --page details --csv > gpurun_out/${tag}_fpass.details.csv 2>&1
ncu -i gpurun_out/${tag}_fpass.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_fpass.sass.csv 2>&1
