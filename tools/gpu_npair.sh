python -m paper_2504_16214_b200._build
for rep in 1 2; do for v in 128 32 64; do
  echo -n "NPAIR_MIN_NTOK=$v: "; W4A16_NPAIR_MIN_NTOK=$v python tools/layer_sweep.py --model qwen3,ds,mixtral --tokens 256,1024 --reps 30 2>&1 | grep '"T"' | python -c "
import sys, json
print(' '.join(f\"{d['model'][:3]}T{d['T']} {d['ms']*1e3:.1f}\" for d in map(json.loads, sys.stdin)))"
done; done
