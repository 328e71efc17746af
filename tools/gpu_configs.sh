# BASELINE configs[0..1] (C1: 16M single tensor, C2: Qwen2.5-1.5B shape) on one GPU, with e2e and the reference arm.
tag=$1
for wl in c1 qwen2.5-1.5b; do
  timeout 600 python bench.py --workload $wl > gpurun_out/${tag}_$wl.json 2> gpurun_out/${tag}_$wl.err; echo "$wl rc=$?"
  timeout 600 python bench.py --workload $wl --impl reference > gpurun_out/${tag}_${wl}_ref.json 2> gpurun_out/${tag}_${wl}_ref.err; echo "$wl ref rc=$?"
done
