python -m paper_2504_16214_b200._build
timeout 600 python -m pytest tests/test_gpu_moe.py -x -q -p no:cacheprovider -k "splitk or gemm" 2>&1 | tail -1
for rep in 1 2; do
for cfg in "W4A16_SPLITS_GU=1 W4A16_SPLITS_DN=1" "W4A16_SPLITS_GU=0" "W4A16_SPLITS_GU=4"; do
  echo "== $cfg"
  env $cfg python tools/layer_sweep.py --model ds --tokens 1,2,4,8,16 --reps 30 2>&1 | grep '"T"' | python -c "
import sys, json
print(' '.join(f\"T{d['T']} {d['ms']*1e3:.1f}\" for d in map(json.loads, sys.stdin)))"
  env $cfg python tools/layer_sweep.py --model qwen3,mixtral --tokens 1,16 --reps 30 2>&1 | grep '"T"' | python -c "
import sys, json
print(' '.join(f\"{d['model'][:3]}T{d['T']} {d['ms']*1e3:.1f}\" for d in map(json.loads, sys.stdin)))"
done; done
