#!/bin/bash
# A/B of env knobs on one box: bench value (T=64 decode step) per setting, twice each
python -m paper_2504_16214_b200._build >/dev/null 2>&1
for rep in 1 2; do
for cfg in "W4A16_FUSED_OSUM=1 W4A16_DECODE_NPAIR=1" "W4A16_FUSED_OSUM=0 W4A16_DECODE_NPAIR=1" "W4A16_FUSED_OSUM=0 W4A16_DECODE_NPAIR=0" "W4A16_FUSED_OSUM=1 W4A16_DECODE_NPAIR=0"; do
  env $cfg timeout 200 python bench.py --steps 30 --warmup 5 --no-cpu --no-sweep 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['ms_per_step'], d['e2e']['value'], {k: round(v,4) for k,v in d['kernel_ms'].items() if 'gemm' in k or 'sums' in k})"
done; done
