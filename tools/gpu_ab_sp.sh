# A/B of the small prefill-tile TMEM split (W4A16_SP_*): token-tile probe + other configs + DS sweep
for rep in 1 2; do
for cfg in "$@"; do
  ( export $cfg; python -m paper_2504_16214_b200._build > /dev/null; echo "== $cfg rep $rep"
    python tools/ntok_probe.py qwen3:256,mixtral:64,mixtral:128,ds:512,ds:1024,qwen3:512 2>&1 | grep picked
    python tools/other_configs_probe.py 2>&1 | grep -E "qwen3|mixtral|llama"
    python tools/layer_sweep.py --model ds --tokens 1024,2048,4096 --reps 10 2>&1 | grep '"T"' | python -c "
import sys, json
for l in sys.stdin: d=json.loads(l); print('  ds T', d['T'], d['ms'], d['tc_frac'])" )
done; done
last="${@: -1}"
( export $last; python -m paper_2504_16214_b200._build > /dev/null; timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1 )
