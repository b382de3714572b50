W4A16_TRACE=1 python -m paper_2504_16214_b200._build
python - <<'PY'
import sys
sys.argv = ["x", "--which", "down", "--experts", "224", "--per-expert", "2"]
src = open("tools/trace_gemm.py").read()
src = src.replace('''for i in range(lo, lo + 12):
    print("   ", i, " ".join(f"{EV[e][:10]}={t[e][i]}" for e in (0, 1, 2, 3, 4, 5, 7, 8)))''', '''for i in range(lo + 2, lo + 36):
    print("   ", i, " ".join(f"{EV[e][:7]}={t[e][i] - t[4][i]}" for e in (3, 5, 6, 7, 8)), "ready_gap", t[4][i] - t[4][i - 1],
          "epi_full_ok - prev epi_done", t[6][i] - t[8][i - 1], "tilestart-prev_done", t[9][i] - t[8][i - 1], "arrive_cost", t[22][i-1] - t[8][i-1], "full_ok-prev_end", t[6][i] - t[22][i-1])''')
exec(compile(src, "trace_gemm.py", "exec"))
PY
