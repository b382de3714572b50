mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_final.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/gputest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_final.json").read().strip().splitlines()[-1])
print({k: d.get(k) for k in ("value", "ms_per_step", "hbm_frac", "gpu_launches")})
print("roofline", d["roofline"]["achieved"], d["roofline"]["frac"], "e2e", d["e2e"]["value"], "ep1", d["ep_world1"])
print("check", d["check"]); print("clocks", d["clocks"])
print("sweep", d["sweep_ds_r1"]["tokens"], d["sweep_ds_r1"]["hbm_frac"], d["sweep_ds_r1"]["tc_frac"])
PY
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref.json
