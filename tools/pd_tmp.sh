python -m paper_2504_16214_b200._build >/dev/null 2>&1
timeout 200 python -m pytest tests/test_gpu_moe.py -q -x -k "fused_gather" 2>&1 | tail -2
W4A16_FUSED_GATHER=1 timeout 300 python -m pytest tests/test_gpu_moe.py -q 2>&1 | tail -1
for fg in 1 0 1 0; do echo "== FUSED_GATHER=$fg"; W4A16_FUSED_GATHER=$fg timeout 200 python tools/layer_sweep.py --model ds --tokens 1,16,64,256,1024 2>&1 | tail -5 | cut -c1-100
W4A16_FUSED_GATHER=$fg timeout 200 python tools/gemm_sweep.py --tokens 8192 --reps 5 2>&1 | tail -1 | cut -c1-300; done
