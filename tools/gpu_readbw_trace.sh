python tools/read_bw.py
bash tools/gpu_trace.sh
