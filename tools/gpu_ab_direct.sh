python -m paper_2504_16214_b200._build
timeout 600 python -m pytest tests/test_gpu_moe.py tests/test_gpu_shapes.py -x -q -p no:cacheprovider -k "gemm or layer or gate_up or deepseek or qwen or mixtral" 2>&1 | tail -2
for rep in 1 2; do
for d in 0 4; do
  echo "== W4A16_DIRECT_ROWS=$d"
  W4A16_DIRECT_ROWS=$d python tools/layer_sweep.py --model ds --tokens 1,16,64 --reps 30 2>&1 | grep '"T"' | python -c "
import sys, json
for l in sys.stdin: d=json.loads(l); print('  T', d['T'], d['ms'], d['hbm_frac'])"
  W4A16_DIRECT_ROWS=$d python tools/layer_sweep.py --model qwen3,mixtral --tokens 16 --reps 30 2>&1 | grep '"T"' | python -c "
import sys, json
for l in sys.stdin: d=json.loads(l); print('  ', d['model'], 'T', d['T'], d['ms'], d['hbm_frac'])"
done; done
