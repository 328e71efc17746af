#!/bin/bash
# full-size byte parity vs the reference (oracle/_ref) on one GPU: 7B headline (all representations,
# N=1 and N=8 sections), 7B 99.99% (escapes, N=8), 32B sharded over 8 with k = 1/4/16
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nproc; free -g | head -2
#timeout 1500 python tools/parity_full.py --workload qwen2.5-7b --ranks 1 --threads 1 --out gpurun_out/r2_parity_7b_n1.jsonl 2>&1 | tail -3 | cut -c1-400
#timeout 1500 python tools/parity_full.py --workload qwen2.5-7b --ranks 8 --threads 3 --out gpurun_out/r2_parity_7b_n8.jsonl 2>&1 | tail -3 | cut -c1-400
#timeout 1500 python tools/parity_full.py --workload qwen2.5-7b --ranks 8 --sparsity 0.9999 --threads 3 --out gpurun_out/r2_parity_7b_9999_n8.jsonl 2>&1 | tail -3 | cut -c1-400
timeout 3000 python tools/parity_full.py --workload qwen2.5-32b --ranks 8 --k 1,4,16 --reprs 0,1,2 --threads 2 --out gpurun_out/r2_parity_32b_n8.jsonl > gpurun_out/r2_parity_32b.log 2>&1; tail -30 gpurun_out/r2_parity_32b.log | cut -c1-400
