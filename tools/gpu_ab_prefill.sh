# same-box A/B of runtime knobs on the prefill layers: DS-R1 T=2048/4096/8192 + the other configs
python -m paper_2504_16214_b200._build > /dev/null
for rep in 1 2; do
  for cfg in "$@"; do
    ( export $cfg; echo "== $cfg rep $rep"
      python tools/layer_sweep.py --model ds --tokens 2048,4096,8192 --reps 5 2>&1 | grep '"T"' | python -c "
import sys, json
for l in sys.stdin: d=json.loads(l); print('  ds T', d['T'], d['ms'], d['tc_frac'])"
      python tools/other_configs_probe.py 2>&1 | grep -E "mixtral|qwen3|llama" )
  done
done
