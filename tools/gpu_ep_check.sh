mkdir -p gpurun_out
python -m paper_2504_16214_b200._build
timeout 900 python -m pytest tests/test_gpu_moe.py -x -q -p no:cacheprovider -k "ep_nccl or raw_awq or c_abi or gather_combine or moe_layer or empty" > gpurun_out/t_ep.log 2>&1; echo "ep tests rc=$?"; tail -15 gpurun_out/t_ep.log
timeout 900 python -m pytest tests/test_gpu_shapes.py -x -q -p no:cacheprovider -k "outliers or deepseek" > gpurun_out/t_shapes.log 2>&1; echo "shape tests rc=$?"; tail -5 gpurun_out/t_shapes.log
timeout 900 python bench.py --steps 20 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench2.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench2.json").read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value","ms_per_step","e2e","ep_world1","check")})
PY
