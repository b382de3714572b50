python -m paper_2504_16214_b200._build >/dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_moe.py -q 2>&1 | tail -1
for mp in 4096 0 4096 0; do echo "== MAX_PAIRS=$mp"; W4A16_ROUTE_PERMUTE_MAX_PAIRS=$mp timeout 200 python tools/layer_sweep.py --model ds,qwen3 --tokens 1,4,16,64,256 2>&1 | tail -10 | cut -c1-110; done
