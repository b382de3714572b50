# A/B: decode accumulator ring 2 (default) vs 4 (W4A16_DECODE_ACC4=1)
sweep() {
  python tools/layer_sweep.py --model ds --tokens 1,16,64,256 --reps 30 2>&1 | grep '"T"' | python -c "
import sys, json
for l in sys.stdin: d=json.loads(l); print('  ds T', d['T'], d['ms'], d['hbm_frac'])"
  python tools/layer_sweep.py --model qwen3,mixtral --tokens 16,256 --reps 30 2>&1 | grep '"T"' | python -c "
import sys, json
for l in sys.stdin: d=json.loads(l); print('  ', d['model'], 'T', d['T'], d['ms'], d['hbm_frac'])"
}
for rep in 1 2; do
  for v in 0 1; do
    W4A16_DECODE_ACC4=$v python -m paper_2504_16214_b200._build > /dev/null
    echo "== DECODE_ACC4=$v rep $rep"
    if [ $rep = 1 ] && [ $v = 1 ]; then
      timeout 600 python -m pytest tests/test_gpu_moe.py tests/test_gpu_shapes.py -x -q -p no:cacheprovider 2>&1 | tail -2
    fi
    sweep
  done
done
