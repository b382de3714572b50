# same-box A/B of runtime knobs on the small-batch layers only (DS-R1 T=1/4/16, Qwen3 T=1/16, Mixtral T=1/16)
python -m paper_2504_16214_b200._build > /dev/null
for rep in 1 2; do
  for cfg in "$@"; do
    ( export $cfg; echo "== $cfg rep $rep"
      python tools/layer_sweep.py --model ds --tokens 1,4,16 --reps 40 2>&1 | grep '"T"' | python -c "
import sys, json
for l in sys.stdin: d=json.loads(l); print('  ds T', d['T'], d['ms'], d['hbm_frac'])"
      python tools/layer_sweep.py --model qwen3,mixtral --tokens 1,16 --reps 40 2>&1 | grep '"T"' | python -c "
import sys, json
for l in sys.stdin: d=json.loads(l); print('  ', d['model'], 'T', d['T'], d['ms'], d['hbm_frac'])" )
  done
done
