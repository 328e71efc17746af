# Round refresh: full bench (e2e + cpu baseline), reference arm, launch list, full ncu captures of
# K1 (k1_tma), K2 (k2_emit) and the apply streaming passes (f_stream), host CPU info.
tag=$1
lscpu > gpurun_out/${tag}_lscpu.txt 2>&1; grep -o -m1 'sha_ni' /proc/cpuinfo >> gpurun_out/${tag}_lscpu.txt
openssl speed -elapsed -evp sha256 -bytes 16384 -seconds 2 > gpurun_out/${tag}_openssl.txt 2>&1
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err; echo "ref rc=$?"
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv $B > /dev/null 2>&1; echo "list rc=$?"
B1="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_tma -s 3 -c 1 -o gpurun_out/${tag}_k1 $B1 > /dev/null 2>&1; echo "k1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_emit -s 4 -c 1 -o gpurun_out/${tag}_k2 $B1 > /dev/null 2>&1; echo "k2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:f_stream -s 4 -c 2 -o gpurun_out/${tag}_apply $B1 > /dev/null 2>&1; echo "apply rc=$?"
for k in k1 k2 apply; do
  ncu -i gpurun_out/${tag}_$k.ncu-rep --page details --csv > gpurun_out/${tag}_$k.details.csv 2>&1
  ncu -i gpurun_out/${tag}_$k.ncu-rep --page details > gpurun_out/${tag}_$k.details.txt 2>&1
  ncu -i gpurun_out/${tag}_$k.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/${tag}_$k.raw.csv 2>&1
done
