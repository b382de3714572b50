python -m paper_2504_16214_b200._build
for gu in 0 2 4 7 8 14; do for dn in 0 2 3 4; do
  echo -n "gu=$gu dn=$dn: "; W4A16_SPLITS_GU=$gu W4A16_SPLITS_DN=$dn python tools/layer_sweep.py --model ds --tokens 1,4 --reps 30 2>&1 | grep '"T"' | python -c "
import sys, json
print(' '.join(f\"T{d['T']} {d['ms']*1e3:.1f}us\" for d in map(json.loads, sys.stdin)))"
done; done
