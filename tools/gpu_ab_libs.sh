# same-box A/B of prebuilt libraries (ab_libs/libw4a16moe_<name>.so): layer prefix + DS-R1 sweep
for rep in 1 2; do
  for name in "$@"; do
    cp ab_libs/libw4a16moe_$name.so paper_2504_16214_b200/lib/libw4a16moe.so
    echo "== $name rep $rep"
    python tools/layer_prefix.py ds 1 qwen3 16 qwen3 256 2>&1 | grep -E "gate_up|down|combine"
    python tools/other_configs_probe.py 2>&1 | grep -v Warning
    python tools/layer_sweep.py --model ds --tokens 1,16,64,256 --reps 30 2>&1 | grep '"T"' | python -c "
import sys, json
for l in sys.stdin: d=json.loads(l); print('  ds T', d['T'], d['ms'], d['hbm_frac'])"
  done
done
