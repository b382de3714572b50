mkdir -p gpurun_out
python -m paper_2504_16214_b200._build
python tools/layer_sweep.py --model ds --tokens 1,4,16 --reps 20 > gpurun_out/sweep_ds.txt 2>&1
python tools/layer_sweep.py --model qwen3 --tokens 16,256 --reps 20 > gpurun_out/sweep_q.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/small_launches.csv python tools/small_probe.py ds:1,ds:16,qwen3:256,llama:1 > gpurun_out/small_probe.log 2>&1; echo "ncu rc=$?"
cat gpurun_out/sweep_ds.txt gpurun_out/sweep_q.txt
