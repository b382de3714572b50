# same-box A/B of build / runtime knobs: DS-R1 layer sweep + bench.py's other_configs. Each argument is
# one "KNOB=V ..." set, exported for both the build and the runs; the LAST set also runs the GPU tests.
sweep() {
  python tools/layer_sweep.py --model ds --tokens 1,16,64,256 --reps 30 2>&1 | grep '"T"' | python -c "
import sys, json
for l in sys.stdin: d=json.loads(l); print('  ds T', d['T'], d['ms'], d['hbm_frac'])"
  python tools/other_configs_probe.py 2>&1 | grep -v Warning
}
last="${@: -1}"
( export $last; python -m paper_2504_16214_b200._build > /dev/null
  echo "== tests with $last"
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3 )
for rep in 1 2; do
  for cfg in "$@"; do
    ( export $cfg; python -m paper_2504_16214_b200._build > /dev/null; echo "== $cfg rep $rep"; sweep )
  done
done
