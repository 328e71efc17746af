# Full ncu capture of K1 at 90% sparsity (the dense end of the C5 sweep) + source page.
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --sparsity 0.9"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_tma -s 3 -c 1 -o gpurun_out/k1d $B > gpurun_out/k1d.log 2>&1; echo "rc=$?"
ncu -i gpurun_out/k1d.ncu-rep --page details > gpurun_out/k1d.details.txt 2>&1
ncu -i gpurun_out/k1d.ncu-rep --page source --csv --print-source sass > gpurun_out/k1d.sass.csv 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/k1d_launches.csv $B > /dev/null 2>&1
