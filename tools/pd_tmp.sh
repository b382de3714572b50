python -m paper_2504_16214_b200._build >/dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_moe.py -q -x 2>&1 | tail -1
W4A16_PREFILL_PAIR=1 W4A16_PAIR=1 timeout 300 python -m pytest tests/test_gpu_moe.py -q -x -k "gemm or layer" 2>&1 | tail -1
timeout 300 python tools/gemm_sweep.py --tokens 1,16,64,256,8192 --reps 10 2>&1 | tail -5 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['T'], d['ms'], round(d['total_ms'],4), d['gate_up_GBs'], d['down_GBs'], d['gate_up_TFs'], d['down_TFs'])"
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-sweep 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['latency_ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['kernel_ms'])"
timeout 300 python tools/layer_sweep.py 2>&1 | tail -12
