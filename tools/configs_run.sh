# every bench config on one GPU (device-resident value only): one JSON line each
mkdir -p gpurun_out
for c in cfg1 cfg3m1 cfg3m4 cfg3m8 cfg3m16 cfg4; do
  timeout 900 python bench.py --config $c --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{' | python -c "
import json, sys
d = json.loads(sys.stdin.read())
print('$c', round(d['value'] / 1e9, 2), 'G tuples/s', round(d['ms_per_step'], 2), 'ms/step', 'roofline frac', round(d['roofline']['frac'], 3), 'result', d.get('result', {}).get('matches_golden', d.get('result')))"
done
