python -m paper_2504_16214_b200._build >/dev/null 2>&1
for sp in 0 2 3 4; do
 if [ $sp = 0 ]; then unset W4A16_SPLITS; else export W4A16_SPLITS=$sp; fi
 echo "== splits $sp"; timeout 100 python tools/gemm_sweep.py --tokens 1,4 --reps 20 2>&1 | tail -2 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['T'], d['ms'], round(d['total_ms'],4))"
 timeout 100 python tools/layer_sweep.py 2>&1 | grep '"T": 1,' | head -3
done
