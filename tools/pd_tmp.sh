python -m paper_2504_16214_b200._build >/dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_moe.py -q -x 2>&1 | tail -1
W4A16_PREFILL_PAIR=1 timeout 300 python -m pytest tests/test_gpu_moe.py -q -x -k "gemm or layer" 2>&1 | tail -1
python tools/gemm_sweep.py --tokens 2048,8192 --reps 5 2>&1 | tail -2 | cut -c1-400
W4A16_PREFILL_PAIR=1 python tools/gemm_sweep.py --tokens 2048,8192 --reps 5 2>&1 | tail -2 | cut -c1-400
python tools/gemm_sweep.py --model mixtral --tokens 8192 --reps 5 | tail -1
python tools/clock_probe.py
W4A16_TRACE=1 python -m paper_2504_16214_b200._build >/dev/null 2>&1
for pr in 0 1; do echo "=== pair $pr"; W4A16_PREFILL_PAIR=$pr timeout 120 python tools/trace_gemm.py --which gate_up --ntok 128 --experts 64 --per-expert 256 2>&1 | grep -v "^    [0-9]\|epi:\|epi_done\|first 12\|per 16\|^    \[" | cut -c1-150; done
