# decode stage timelines (trace build) for TMEM A-slot counts 2 (default) and 3
for cfg in "W4A16_DECODE_NUMA=2" "W4A16_DECODE_NUMA=3 W4A16_DECODE_MAXACC=4"; do
  ( export $cfg W4A16_TRACE=1; python -m paper_2504_16214_b200._build > /dev/null
    for w in "gate_up --experts 8 --per-expert 1" "gate_up --experts 224 --per-expert 2"; do
      echo "=== $cfg $w"; timeout 120 python tools/trace_gemm.py --which $w 2>&1 | grep -v "^    [0-9]"
    done )
done
