python -m paper_2504_16214_b200._build >/dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_moe.py -q -x 2>&1 | tail -1
W4A16_DECODE_NPAIR=0 timeout 300 python -m pytest tests/test_gpu_moe.py -q -x -k "gemm or layer or forward" 2>&1 | tail -1
for np_ in 1 0 1 0; do
echo "== DECODE_NPAIR=$np_"
W4A16_DECODE_NPAIR=$np_ timeout 200 python tools/gemm_sweep.py --tokens 1,16,64,256 --reps 10 2>&1 | tail -4 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['T'], d['ms']['gemm_down'], d['down_GBs'], round(d['total_ms'],4))"
W4A16_DECODE_NPAIR=$np_ timeout 200 python tools/gemm_sweep.py --model qwen3 --tokens 16,64 --reps 10 2>&1 | tail -2 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('qwen3', d['T'], d['ms']['gemm_down'], d['down_GBs'])"
done
