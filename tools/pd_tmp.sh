python -m paper_2504_16214_b200._build >/dev/null 2>&1
W4A16_FUSED_OSUM=1 timeout 300 python -m pytest tests/test_gpu_moe.py -q -x -k "layer or graph or pipeline" 2>&1 | tail -1
for f in 1 0 1 0; do echo "== FUSED_OSUM=$f"; W4A16_FUSED_OSUM=$f timeout 200 python tools/layer_sweep.py 2>&1 | grep '"ds"' | head -5; done
