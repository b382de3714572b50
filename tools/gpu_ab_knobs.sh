# A/B of compile-time knobs on the layer sweep: each line "NAME=VALUE ..." is one build
sweep() {
  python tools/layer_sweep.py --model ds --tokens 1,16,64,256 --reps 30 2>&1 | grep '"T"' | python -c "
import sys, json
for l in sys.stdin: d=json.loads(l); print('  ds T', d['T'], d['ms'], d['hbm_frac'])"
  python tools/layer_sweep.py --model qwen3,mixtral --tokens 16,256 --reps 30 2>&1 | grep '"T"' | python -c "
import sys, json
for l in sys.stdin: d=json.loads(l); print('  ', d['model'], 'T', d['T'], d['ms'], d['hbm_frac'])"
}
for rep in 1 2; do
  for cfg in "$@"; do
    env $cfg python -m paper_2504_16214_b200._build > /dev/null
    echo "== $cfg rep $rep"
    sweep
  done
done
