#!/bin/bash
# Build and run the tcgen05 descriptor probe over its layout hypotheses (GPU box).
cd "$(dirname "$0")"
nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/tc_probe probe.cu || exit 1
p() { timeout 20 /tmp/tc_probe "$@" 2>&1 | tail -1; }
p bf16 128 16 64 0 24 0      # K-major A and B (verified layout)
p tf32 128 16 64 0 24 0
p bf16 64 16 64 0 24 0       # M = 64: where do the rows land?
p bf16 64 64 64 0 24 0
p bf16 128 32 64 0 24 1      # MN-major B, both stride assignments
p bf16 128 32 64 1 24 1
p bf16 64 160 64 0 24 1
p bf16 64 160 64 1 24 1
p bf16 128 256 64 0 24 0     # widest N
p bf16 128 32 64 0 24 0 256  # strides apart: which field strides along K
p bf16 128 32 64 1 24 0 256
p bf16 128 32 64 0 24 1 256
p bf16 128 32 64 1 24 1 256
p tf32 128 32 64 0 24 0 256
