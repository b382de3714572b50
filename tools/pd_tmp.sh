python -m paper_2504_16214_b200._build >/dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_moe.py -q -x 2>&1 | tail -1
python tools/gemm_sweep.py --tokens 2048,8192 --reps 5 2>&1 | tail -2 | cut -c1-400
python tools/gemm_sweep.py --model mixtral --tokens 8192 --reps 5 | tail -1
W4A16_TRACE=1 python -m paper_2504_16214_b200._build >/dev/null 2>&1
for w in gate_up down; do echo "=== $w"; timeout 120 python tools/trace_gemm.py --which $w --ntok 128 --experts 64 --per-expert 256 2>&1 | grep -A2 "stage period\|prefill tiles\|per 16-token" | cut -c1-150; done
