# Full ncu captures of the apply + K2 kernels of the 7B bench step (one launch each), plus source pages.
tag=$1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
for k in "f_pass<0, 3>" "f_pass<0, 0>" "k2_emit"; do
  n=$(echo "$k" | tr -dc 'a-z0-9')
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$k" -s 2 -c 1 -o gpurun_out/${tag}_$n $B > gpurun_out/${tag}_$n.log 2>&1; echo "$n rc=$?"
  ncu -i gpurun_out/${tag}_$n.ncu-rep --page details --csv > gpurun_out/${tag}_$n.details.csv 2>&1
  ncu -i gpurun_out/${tag}_$n.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_$n.sass.csv 2>&1
done
ls -la gpurun_out/
