#!/bin/bash
# tests + bench + launch list of the timed steps + one ncu --set full capture per grouped GEMM
# usage: bash tools/gpu_prof.sh [tokens]   (each ncu run bounded by its own timeout)
T=${1:-64}
mkdir -p gpurun_out
python -m paper_2504_16214_b200._build
timeout 600 python -m pytest tests/test_gpu_moe.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --tokens $T > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python tools/summarize_bench.py gpurun_out/bench.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 400 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --tokens $T > /dev/null 2>&1; echo "ncu launches rc=$?"
for skip in 0 1; do
  timeout 420 ncu --set full --clock-control none --import-source on -k regex:w4a16_moe_gemm -s $skip -c 1 \
     -o gpurun_out/prof_gemm$skip -f python bench.py --steps 1 --warmup 0 --no-sweep --no-cpu --tokens $T > gpurun_out/ncu_full$skip.log 2>&1
  echo "ncu full $skip rc=$?"; tail -2 gpurun_out/ncu_full$skip.log
done
# prefill: one 128-token gate/up launch (64 experts x 256 rows, full tiles)
timeout 420 ncu --set full --clock-control none --import-source on -k regex:w4a16_moe_gemm -s 2 -c 1 \
   -o gpurun_out/prof_prefill -f python tools/prof_one.py --which gate_up --experts 64 --per-expert 256 --ntok 128 --reps 3 --sums 0 \
   > gpurun_out/ncu_prefill.log 2>&1
echo "ncu prefill rc=$?"; tail -2 gpurun_out/ncu_prefill.log
