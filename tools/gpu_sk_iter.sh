# stream-K iteration: CTA timelines (trace build) of the DS-R1 T=1 down GEMM, then the single-GEMM probe
bash tools/gpu_trace_sk.sh 2>&1 | grep -E "===|tile starts|stream-K piece|warp arrivals|CTA entry"
python -m paper_2504_16214_b200._build > /dev/null
python tools/sk_probe.py
