mkdir -p gpurun_out
python -m paper_2504_16214_b200._build
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest2.log 2>&1; echo "gpu tests rc=$?"; tail -8 gpurun_out/gputest2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke2.log
