python -m paper_2504_16214_b200._build
timeout 600 python -m pytest tests/test_gpu_moe.py -x -q -p no:cacheprovider -k "gemm or layer or gate_up" 2>&1 | tail -2
echo "== new epilogue"; python tools/layer_sweep.py --model ds --tokens 1,16,64,256 --reps 30 2>&1 | grep '"T"'
python tools/layer_sweep.py --model qwen3,mixtral --tokens 16,256 --reps 30 2>&1 | grep '"T"'
W4A16_TRACE=1 python -m paper_2504_16214_b200._build
for args in "--which gate_up --experts 8 --per-expert 1" "--which down --experts 224 --per-expert 2"; do
  echo "=== $args"; timeout 120 python tools/trace_gemm.py $args 2>&1 | grep -v "^    [0-9]" | head -18
done
