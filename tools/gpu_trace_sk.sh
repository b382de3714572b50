W4A16_TRACE=1 python -m paper_2504_16214_b200._build > /dev/null
for sk in 0 1; do
  for cta in 0 100; do
    echo "=== STREAMK=$sk cta $cta"
    W4A16_STREAMK=$sk timeout 120 python tools/trace_gemm.py --which down --experts 8 --per-expert 1 --cta $cta --dump 2>&1 | cat
    W4A16_STREAMK=$sk timeout 120 python tools/trace_gemm.py --which down --experts 1 --per-expert 1 --nk 14336,4096 --cta $cta --dump 2>&1 | grep -E "CTA entry|stream-K piece|warp arr"
  done
done
