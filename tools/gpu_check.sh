#!/bin/bash
# quick GPU smoke of the kernels, staged so that a hang in one stage does not hide the others
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m paper_2504_16214_b200._build
for k in "dequant" "route" "permute" "gather" "gemm or linear" "layer"; do
  echo "=== $k"
  timeout 240 python -m pytest tests/test_gpu_moe.py -x -q -k "$k" 2>&1 | tail -25
done
