#!/bin/bash
# Round-2 final single-GPU evidence: bench (e2e + cpu baseline + reference parity), reference arm,
# int32 / FLAT lines, density sweep, C1 / C2 lines, launch list (time + DRAM bytes), full ncu
# captures of k1_tma / k2_emit / the apply streaming passes.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
t=${TAG:-r2f}
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/${t}_bench.json 2> gpurun_out/${t}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/${t}_bench_ref.json 2> gpurun_out/${t}_bench_ref.err; echo "ref rc=$?"
for r in 1 2; do
  timeout 600 python bench.py --repr $r --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${t}_repr$r.json 2>/dev/null; echo "repr $r rc=$?"
done
for sp in 0.9 0.95 0.999 0.9999; do
  timeout 600 python bench.py --sparsity $sp --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${t}_sweep_$sp.json 2>/dev/null; echo "sweep $sp rc=$?"
done
for w in c1 qwen2.5-1.5b; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 3 > gpurun_out/${t}_cfg_$w.json 2>/dev/null; echo "cfg $w rc=$?"
  timeout 600 python bench.py --impl reference --workload $w --steps 3 --warmup 1 > gpurun_out/${t}_cfg_${w}_ref.json 2>/dev/null
done
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/${t}_launches.csv $B > /dev/null 2>&1; echo "list rc=$?"
B1="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_tma -s 3 -c 1 -o gpurun_out/${t}_k1 $B1 > /dev/null 2>&1; echo "k1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_emit -s 6 -c 1 -o gpurun_out/${t}_k2 $B1 > /dev/null 2>&1; echo "k2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:f_stream -s 6 -c 2 -o gpurun_out/${t}_apply $B1 > /dev/null 2>&1; echo "apply rc=$?"
for k in k1 k2 apply; do
  ncu -i gpurun_out/${t}_$k.ncu-rep --page details > gpurun_out/${t}_$k.details.txt 2>&1
  ncu -i gpurun_out/${t}_$k.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/${t}_$k.raw.csv 2>&1
done
rm -f gpurun_out/${t}_*.ncu-rep
ls gpurun_out/${t}_*
