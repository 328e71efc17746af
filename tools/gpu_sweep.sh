# Sparsity sweep and multi-step patches (C4) on one GPU.
tag=$1
for s in 0.9 0.99 0.999 0.9999; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 --sparsity $s > gpurun_out/${tag}_sweep_$s.json 2> gpurun_out/${tag}_sweep_$s.err
  echo "sparsity $s rc=$?"
done
timeout 900 python tools/multistep.py --workload qwen2.5-7b --k 1 4 16 > gpurun_out/${tag}_multistep_7b.jsonl 2> gpurun_out/${tag}_multistep_7b.err
echo "multistep rc=$?"
