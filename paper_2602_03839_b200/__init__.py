"""B200-native PULSE (Patch Updates via Lossless Sparse Encoding) hot path.

encode (bitwise diff of two bf16 snapshots -> compacted, delta-coded patch) and
apply (scatter a patch into resident weights), bit-identical to the reference
CPU encoder/decoder (arxiv 2602.03839), as sm_100a CUDA kernels behind a C ABI
(include/pulse_cuda.h).  `device` drives snapshots resident in HBM, `host`
mirrors the reference's host-buffer API, `shard` is the multi-GPU driver.
"""
__all__ = ["device", "host", "shapes", "shard"]
