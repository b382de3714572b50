python -m paper_2504_16214_b200._build >/dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_moe.py -q -x 2>&1 | tail -1
python tools/gemm_sweep.py --tokens 1,16,64,256,8192 --reps 10 2>&1 | tail -5 | cut -c1-400
python tools/layer_sweep.py 2>&1 | tail -12
