# small-kernel iteration: their GPU tests, then the per-kernel layer prefix at small batches
python -m paper_2504_16214_b200._build > /dev/null
timeout 600 python -m pytest tests/test_gpu_moe.py -x -q -p no:cacheprovider -k "gather or combine or sums or permute or route or layer" 2>&1 | tail -2
python tools/layer_prefix.py ds 1 ds 16 qwen3 16 qwen3 256
