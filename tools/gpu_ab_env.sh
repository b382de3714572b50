# same-box A/B of runtime environment knobs (no rebuild): layer prefix + other configs + DS sweep.
# usage: bash tools/gpu_ab_env.sh "KNOB=V ..." "KNOB=V ..."
python -m paper_2504_16214_b200._build > /dev/null
for rep in 1 2; do
  for cfg in "$@"; do
    ( export $cfg; echo "== $cfg rep $rep"
      python tools/layer_prefix.py ds 1 qwen3 16 2>&1 | grep -E "gate_up|down|combine"
      python tools/other_configs_probe.py 2>&1 | grep -v Warning
      python tools/layer_sweep.py --model ds --tokens 1,16,64,256 --reps 30 2>&1 | grep '"T"' | python -c "
import sys, json
for l in sys.stdin: d=json.loads(l); print('  ds T', d['T'], d['ms'], d['hbm_frac'], d['tc_frac'])" )
  done
done
