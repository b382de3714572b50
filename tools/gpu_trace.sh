W4A16_TRACE=1 python -m paper_2504_16214_b200._build
for args in "--which gate_up --experts 8 --per-expert 1" "--which gate_up --experts 224 --per-expert 2" "--which down --experts 8 --per-expert 1" "--which down --experts 224 --per-expert 2"; do
  echo "=== $args"; timeout 120 python tools/trace_gemm.py $args 2>&1 | grep -v "^    [0-9]"
done
