#!/bin/bash
# tests + bench + launch list + full ncu capture of the two grouped-GEMM launches of one step
mkdir -p gpurun_out
python -m paper_2504_16214_b200._build
timeout 600 python -m pytest tests/test_gpu_moe.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python tools/summarize_bench.py gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 400 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:w4a16_moe_gemm -c 2 \
   -o gpurun_out/prof_gemm -f python bench.py --steps 1 --warmup 1 --no-sweep --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
