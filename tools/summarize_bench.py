import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value', 'ms_per_step', 'tflops', 'hbm_frac', 'gpu_launches')})
r = d['roofline']
print('roofline', r['achieved'], r['frac'], 'kernel_ms', d['kernel_ms'])
print('clocks', d['clocks'], 'e2e', d['e2e']['value'])
for s in d.get('sweep', []):
    print(s)
