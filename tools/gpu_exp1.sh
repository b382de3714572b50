python -m paper_2504_16214_b200._build
echo "== A default"; python tools/layer_sweep.py --model ds --tokens 1,16,64 --reps 20 2>&1 | grep '"T"'
python tools/layer_sweep.py --model qwen3 --tokens 16,256 --reps 20 2>&1 | grep '"T"'
echo "== C prefill-mode GEMMs at 16 tokens"; W4A16_DECODE_MAX_NTOK=0 python tools/layer_sweep.py --model ds --tokens 1,16,64 --reps 20 2>&1 | grep '"T"'
W4A16_KSPLIT=0 python -m paper_2504_16214_b200._build
echo "== B KSPLIT=0 (4 accumulator stages)"; python tools/layer_sweep.py --model ds --tokens 1,16,64 --reps 20 2>&1 | grep '"T"'
python tools/layer_sweep.py --model qwen3 --tokens 16,256 --reps 20 2>&1 | grep '"T"'
W4A16_KSPLIT=0 W4A16_TRACE=1 python -m paper_2504_16214_b200._build
for args in "--which gate_up --experts 8 --per-expert 1" "--which down --experts 224 --per-expert 2"; do
  echo "=== KSPLIT=0 $args"; timeout 120 python tools/trace_gemm.py $args 2>&1 | grep -v "^    [0-9]" | head -20
done
