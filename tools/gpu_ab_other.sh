# same-box A/B of build knobs on bench.py's other_configs: each argument is one "NAME=VALUE ..." build
for rep in 1 2; do
  for cfg in "$@"; do
    env $cfg python -m paper_2504_16214_b200._build > /dev/null
    echo "== $cfg rep $rep"
    python tools/other_configs_probe.py 2>&1 | grep -v Warning
  done
done
