python -m paper_2504_16214_b200._build
python tools/layer_prefix.py ds 1 ds 4 ds 16 qwen3 16 qwen3 256 2>&1
W4A16_NO_PDL=1 python tools/layer_prefix.py ds 1 2>&1 | sed 's/^/NOPDL /'
