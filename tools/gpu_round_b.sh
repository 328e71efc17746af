# Round-1b confirmation on a 2-GPU box: the driver's N=2 both-arm run, then single-GPU configs
# (C1, C2 with e2e and the reference arm), the sparsity sweep (C5) and multi-step patches (C4).
bash tools/gpu_driverlike.sh
export CUDA_VISIBLE_DEVICES=0
bash tools/gpu_configs.sh rb
bash tools/gpu_sweep.sh rb
