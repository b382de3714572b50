for d in 1 0 1 0; do
W4A16_DUAL=$d python -m paper_2504_16214_b200._build >/dev/null 2>&1
echo "== DUAL=$d"
timeout 200 python tools/gemm_sweep.py --tokens 2048,8192 --reps 8 2>&1 | tail -2 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['T'], d['ms']['gemm_gate_up'], d['ms']['gemm_down'], d['gate_up_TFs'], d['down_TFs'])"
timeout 200 python tools/gemm_sweep.py --model mixtral --tokens 1024,8192 --reps 5 2>&1 | tail -2 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('mixtral', d['T'], d['ms']['gemm_gate_up'], d['ms']['gemm_down'], d['gate_up_TFs'], d['down_TFs'])"
done
