# Round refresh: full bench (e2e + cpu baseline), reference arm, launch list, K1 full profile, host CPU info.
tag=$1
lscpu > gpurun_out/${tag}_lscpu.txt 2>&1; grep -o -m1 'sha_ni' /proc/cpuinfo >> gpurun_out/${tag}_lscpu.txt
openssl speed -elapsed -evp sha256 -bytes 16384 -seconds 2 > gpurun_out/${tag}_openssl.txt 2>&1
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_tma -s 3 -c 1 -o gpurun_out/${tag}_k1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "k1 rc=$?"
