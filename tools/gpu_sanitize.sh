python -m paper_2504_16214_b200._build
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_moe.py -x -q -p no:cacheprovider -k "gemm or layer or gate_up" 2>&1 | tail -2
python tools/layer_sweep.py --model ds --tokens 1,64 --reps 30 2>&1 | grep '"T"'
for tool in memcheck synccheck racecheck initcheck; do
  CUDA_MODULE_LOADING=EAGER timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_all.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitizer_$tool.log
done
