#!/bin/bash
# tests + bench (no ncu)
mkdir -p gpurun_out
python -m paper_2504_16214_b200._build
timeout 600 python -m pytest tests/test_gpu_moe.py -x -q 2>&1 | tail -4
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print({k:d[k] for k in ('value','ms_per_step','tflops','hbm_frac','gpu_launches')})
print('roofline',d['roofline']['achieved'],d['roofline']['frac'],'kernel_ms',d['kernel_ms'])
print('clocks',d['clocks']); print('e2e',d['e2e']['value'])
for r in d['sweep']: print(r)
PY
tail -3 gpurun_out/bench.err
